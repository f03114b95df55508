// pf_dual.cuh — explicit local dual operators, device side.
//
// k_dual_root: per subdomain, the root front of the bordered partial
// factorisation (pf_dual.hpp) — m = nB + nM, column-major, lower triangle —
//   [[ S    . ]
//    [ G_B  0 ]]
// becomes
//   Sd = G_B S G_B^T              (Dirichlet preconditioner share),
//   F  = G_B S_reg^{-1} G_B^T      (F-apply share; S_reg: fixing dofs -> identity)
// by: symmetrising S; Sd column by column through T = S G_B^T[:, j] (G_B is a
// few entries per multiplier); fixing rows/columns to identity; a blocked
// right-looking LDL^T of the nB B-pivots (16-column panels factored in place,
// the trailing update reading the panel from shared memory with a padded
// stride) whose trailing multiplier block is -F.  One CTA per subdomain;
// setup only.
//
// k_local_gemv / k_local_reduce: the per-iteration apply y = sum_s Op_s x_s
// (one CTA per subdomain, a warp per row of the dense symmetric operator,
// x_s staged in shared memory), then each multiplier sums its (one or two)
// subdomain contributions in a fixed order.
#pragma once

#include <cuda_runtime.h>

namespace pf {
namespace dev {

struct DualSet {
  const int* prob;                 // this launch's problems
  const int* prob_type;
  const long long* prob_fbase;     // front base in F (chunk buffer)
  const long long* type_rootoff;   // root front offset inside a problem's fronts
  const int *type_nB, *type_nM;
  const int *type_gptr, *type_gidx;  // per type: base into g_ptr (nM+1) / g_b
  const int *g_ptr, *g_b;
  const int *type_fix, *type_nfix, *fixpos;
  const double* Gv;
  const long long* prob_gval;
  const long long* prob_op;        // output offset (nM*nM) of Fop / Sop
  double* F;
  double* Fop;
  double* Sop;
  int* err;
};

constexpr int kDualPW = 16;   // panel width of the root factorisation
constexpr int kDualLd = 17;   // padded row stride of the staged panel

__global__ void __launch_bounds__(512) k_dual_root(DualSet S) {
  extern __shared__ double sm_d[];
  const int p = S.prob[blockIdx.x];
  const int t = S.prob_type[p];
  const int nB = S.type_nB[t], nM = S.type_nM[t], m = nB + nM;
  double* Fr = S.F + S.prob_fbase[p] + S.type_rootoff[t];
  const int* gp = S.g_ptr + S.type_gptr[t];
  const int* gb = S.g_b + S.type_gidx[t];
  const double* gv = S.Gv + S.prob_gval[p];
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  auto at = [&](int i, int j) -> double& { return Fr[i + (long long)j * m]; };
  // 1. S block full (upper from lower)
  for (int j = warp; j < nB; j += nw)
    for (int i = lane; i < j; i += 32) at(i, j) = at(j, i);
  __syncthreads();
  // 2. Sd = G S G^T, one multiplier column j at a time: T = S G^T e_j (smem)
  double* T = sm_d;
  double* Sd = S.Sop + S.prob_op[p];
  for (int j = 0; j < nM; ++j) {
    for (int b = tid; b < nB; b += nth) {
      double v = 0.0;
      for (int q = gp[j]; q < gp[j + 1]; ++q) v += gv[q] * at(b, gb[q]);
      T[b] = v;
    }
    __syncthreads();
    for (int i = tid; i < nM; i += nth) {
      double v = 0.0;
      for (int q = gp[i]; q < gp[i + 1]; ++q) v += gv[q] * T[gb[q]];
      Sd[(long long)i * nM + j] = v;
    }
    __syncthreads();
  }
  // 3. regularise the fixing dofs (floating subdomains): rows/columns -> identity
  const int* fx = S.fixpos + S.type_fix[t];
  for (int q = 0; q < S.type_nfix[t]; ++q) {
    const int f = fx[q];
    for (int i = tid; i < m; i += nth) {
      if (i > f) at(i, f) = 0.0;
      if (i < f) at(f, i) = 0.0;
    }
    __syncthreads();
    if (tid == 0) at(f, f) = 1.0;
    __syncthreads();
  }
  // 4. LDL^T of the nB B-pivots; the trailing multiplier block becomes -F
  double* Lp = sm_d;  // staged panel rows (padded stride)
  __shared__ double Dk[kDualPW];
  for (int p0 = 0; p0 < nB; p0 += kDualPW) {
    const int pw = min(kDualPW, nB - p0);
    for (int j = p0; j < p0 + pw; ++j) {
      const double d = at(j, j);
      if (!(d != 0.0) || !isfinite(d)) {
        if (tid == 0) atomicExch(S.err, 1);
        return;
      }
      const double inv = 1.0 / d;
      for (int c = j + 1 + warp; c < p0 + pw; c += nw) {
        const double lc = at(c, j) * inv;
        for (int i = c + lane; i < m; i += 32) at(i, c) -= at(i, j) * lc;
      }
      __syncthreads();
      for (int i = j + 1 + tid; i < m; i += nth) at(i, j) *= inv;
      __syncthreads();
    }
    const int r0 = p0 + pw;
    const int nr = m - r0;
    for (int e = tid; e < nr * kDualPW; e += nth) {
      const int r = e / kDualPW, k = e - r * kDualPW;
      Lp[r * kDualLd + k] = k < pw ? at(r0 + r, p0 + k) : 0.0;
    }
    if (tid < kDualPW) Dk[tid] = tid < pw ? at(p0 + tid, p0 + tid) : 0.0;
    __syncthreads();
    for (int c = r0 + warp; c < m; c += nw) {
      double w[kDualPW];
#pragma unroll
      for (int k = 0; k < kDualPW; ++k) w[k] = Dk[k] * Lp[(c - r0) * kDualLd + k];
      for (int i = c + lane; i < m; i += 32) {
        const double* li = Lp + (i - r0) * kDualLd;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < kDualPW; k += 2) a0 += li[k] * w[k], a1 += li[k + 1] * w[k + 1];
        at(i, c) -= a0 + a1;
      }
    }
    __syncthreads();
  }
  // 5. F = -(trailing multiplier block), full symmetric row-major
  double* Fo = S.Fop + S.prob_op[p];
  for (int e = tid; e < nM * nM; e += nth) {
    const int i = e / nM, j = e - i * nM;
    Fo[e] = -(i >= j ? at(nB + i, nB + j) : at(nB + j, nB + i));
  }
}

/// Y[yoff_s + i] = sum_j Op_s[i][j] x[xoff_s + j]  (x already gathered per subdomain)
__global__ void __launch_bounds__(256) k_local_gemv(int nsub, const int* __restrict__ nloc,
                                                    const long long* __restrict__ loff,
                                                    const long long* __restrict__ opoff,
                                                    const double* __restrict__ Op,
                                                    const double* __restrict__ xloc, double* __restrict__ Y) {
  extern __shared__ double xs[];
  const int s = blockIdx.x;
  if (s >= nsub) return;
  const int n = nloc[s];
  const double* x = xloc + loff[s];
  for (int j = threadIdx.x; j < n; j += blockDim.x) xs[j] = x[j];
  __syncthreads();
  const double* A = Op + opoff[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw) {
    const double* a = A + (long long)i * n;
    double v = 0.0;
    for (int j = lane; j < n; j += 32) v += a[j] * xs[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) Y[loff[s] + i] = v;
  }
}

/// xloc[k] = x[lam[k]] for every (subdomain, local multiplier) slot
__global__ void k_local_gather(long long n, const int* __restrict__ lam, const double* __restrict__ x,
                               double* __restrict__ xloc) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) xloc[k] = x[lam[k]];
}

/// y[i] = alpha * sum over the multiplier's slots (fixed order) of Y
__global__ void k_local_reduce(int n, const int* __restrict__ ptr, const long long* __restrict__ slot,
                               const double* __restrict__ Y, double* __restrict__ y, double alpha) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) v += Y[slot[q]];
  y[i] = alpha * v;
}

}  // namespace dev
}  // namespace pf
