// pf_kernels.cuh — sm_100a kernels of the FETI engine.
//
// Hot path (per Krylov iteration): the batched supernodal LDL^T sweeps
// (k_sweep, pf_sweep.cuh) over every subdomain factor, the
// gather G^T lambda and scatter G x around them, the Dirichlet
// preconditioner SpMVs, the coarse projector and deterministic Krylov
// vector ops.  All fp64, all reductions in fixed order (bitwise repeatable).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pf {
namespace dev {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Batched supernodal solve data (concatenated over symbolic types)
// ---------------------------------------------------------------------------
struct TypeDesc {
  int n, nsn, ntask;
  int sn_base, task_base;            // into sn_* / task_* arrays
  long long row_base, cb_base;       // into slot / cb_rows
  long long fold_base, foldidx_base; // into fold_ptr (n+1 per type) / fold_idx
  long long slot_base;               // into slots (uint16, per-supernode lists padded to 8)
};

/// One work item of a sweep level, flattened on the host so a warp starts
/// its task with a single 80-byte broadcast load instead of a chain of
/// dependent lookups (problem -> type -> task -> ...).
struct __align__(16) WorkRec {
  long long lofs;   // value stream of the task: offset into L (doubles)
  long long xofs;   // problem offset into X / D (prob_x)
  long long cbofs;  // problem offset into CB (prob_cb)
  int c0, nct, cbo, cbl;
  int sn, nsn;      // first supernode (global index into sn_meta), count
  int lbytes;       // value stream bytes
  int slot_base;    // type's slot table base (uint16 elements)
  int fold_base, foldidx_base, cb_base;  // type bases of fold_ptr / fold_idx / cb_rows
  int pad;
};

struct SolveSet {
  const TypeDesc* types;
  const int *sn_col0, *sn_ncol, *sn_nrow;
  const long long *sn_rowoff, *sn_valoff;  // relative to the type's row/value base
  const int* slot;
  const int *task_sn0, *task_sn1, *task_c0, *task_c1, *task_cboff, *task_cblen;
  const int* cb_rows;                      // relative to type cb_base
  const int* fold_ptr;                     // per type: n+1 entries at fold_base (relative to foldidx_base)
  const int* fold_idx;                     // cb indices (relative to the problem's cb region)
  const int2* sn_meta;                     // per supernode: ncol | nrow << 16, slot offset (type-relative)
  const uint16_t* slots;                   // per supernode row -> workspace slot
  const long long* task_lbeg;              // task value stream start (type-relative, even)
  const int* task_lbytes;                  // task value stream length (bytes)
  // problems
  int nprob;
  const int* prob_type;
  const long long *prob_lval, *prob_x, *prob_cb;
  // work list of one level: (problem, type-relative task)
  int nwork;
  const int *work_prob, *work_task;
  const WorkRec* work;
  // data
  const double* L;
  const double* D;
  double* X;
  double* CB;
  int nrhs;         // 1 or 2 right-hand sides (second at X + x_stride)
  long long x_stride, cb_stride;
};

__device__ __forceinline__ long long col_off(int j, int m) {
  return (long long)j * (m - 1) - (long long)j * (j - 1) / 2;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

/// lanes l ends with the sum over all 32 lanes of acc[l % PW]
template <int PW>
__device__ __forceinline__ double transpose_reduce(double (&acc)[PW], int lane) {
#pragma unroll
  for (int off = PW / 2; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      const double send = upper ? acc[k] : acc[k + off];
      const double keep = upper ? acc[k + off] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  double v = acc[0];
#pragma unroll
  for (int off = PW; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];  // fixed order
  return s;
}

// ---------------------------------------------------------------------------
// Sparse gather / scatter / SpMV helpers (row-parallel, fixed summation order)
// ---------------------------------------------------------------------------

/// X[rows[i]] (=|+=) alpha * sum_q val[q] * x[idx[q]]
__global__ void k_gather(int nrows, const int* rows, const int* ptr, const int* idx, const double* val,
                         const double* x, double* X, double alpha, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s += val[q] * x[idx[q]];
  if (accumulate)
    X[rows[i]] += alpha * s;
  else
    X[rows[i]] = alpha * s;
}

/// y[i] = beta*y[i] + alpha*(sum over segment 1 + sum over segment 2)
/// (two subdomain segments per multiplier row, split at mid[i]).
__global__ void k_spmv2(int nrows, const int* ptr, const int* mid, const int* idx, const double* val,
                        const double* X, double* y, double alpha, double beta, const double* sub) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s1 = 0.0, s2 = 0.0;
  for (int q = ptr[i]; q < mid[i]; ++q) s1 += val[q] * X[idx[q]];
  for (int q = mid[i]; q < ptr[i + 1]; ++q) s2 += val[q] * X[idx[q]];
  double v = alpha * (s1 + s2);
  if (sub) v -= sub[i];
  y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + v;
}

/// plain CSR SpMV y = alpha*A x + beta*y
__global__ void k_spmv(int nrows, const int* ptr, const int* idx, const double* val, const double* x, double* y,
                       double alpha, double beta) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s += val[q] * x[idx[q]];
  y[i] = (beta == 0.0 ? 0.0 : beta * y[i]) + alpha * s;
}

/// indexed SpMV with values fetched from another array: y[rows_out[i]] = sum val[vpos[q]] * x[idx[q]]
__global__ void k_spmv_ind(int nrows, const int* ptr, const long long* vpos, const long long* idx,
                           const double* val, const double* x, double* y, const long long* rows_out,
                           const double* ysub, double alpha) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  double s = 0.0;
  for (int q = ptr[i]; q < ptr[i + 1]; ++q) s += val[vpos[q]] * x[idx[q]];
  const long long o = rows_out[i];
  y[o] = (ysub ? ysub[i] : 0.0) + alpha * s;
}

/// permute in: X[xo + pos] = src[so + perm[pos]] (per problem, one block-stride loop)
__global__ void k_perm_in(int nprob, const long long* prob_x, const long long* prob_src, const int* prob_n,
                          const long long* prob_perm, const int* perm, const double* src, double* X, int stride) {
  const int p = blockIdx.y;
  if (p >= nprob) return;
  const int n = prob_n[p];
  const int* pm = perm + prob_perm[p];
  const double* s = src + prob_src[p];
  double* x = X + prob_x[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[(long long)i * stride] = s[pm[i]];
}

/// permute out: dst[so + perm[pos]] = X[xo + pos]
__global__ void k_perm_out(int nprob, const long long* prob_x, const long long* prob_dst, const int* prob_n,
                           const long long* prob_perm, const int* perm, const double* X, double* dst, int stride) {
  const int p = blockIdx.y;
  if (p >= nprob) return;
  const int n = prob_n[p];
  const int* pm = perm + prob_perm[p];
  double* d = dst + prob_dst[p];
  const double* x = X + prob_x[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d[pm[i]] = x[(long long)i * stride];
}

__global__ void k_zero_idx(int n, const long long* idx, double* X) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) X[idx[i]] = 0.0;
}

// ---------------------------------------------------------------------------
// Deterministic reductions and Krylov vector kernels
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 296;  // 2 x 148 SMs, fixed for determinism
constexpr int kRedThreads = 256;

/// partial[b] = sum over the block's fixed grid-stride range of a[i]*b[i]
__global__ void k_dot_partial(int n, const double* a, const double* b, double* partial) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += a[i] * b[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

/// out[slot] = sum of partials (single block, fixed order)
__global__ void k_dot_final(int nparts, const double* partial, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partial[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_axpby(int n, double a, const double* x, double b, double* y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}

/// y = x + coef*y with coef = num/den read from device scalars (PCG p-update)
__global__ void k_xpay_dev(int n, const double* x, double* y, const double* num, const double* den) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double c = *num / *den;
  if (i < n) y[i] = x[i] + c * y[i];
}

/// y += sgn*(num/den)*x  (device scalars)
__global__ void k_axpy_dev(int n, double sgn, const double* num, const double* den, const double* x, double* y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double c = sgn * (*num / *den);
  if (i < n) y[i] += c * x[i];
}

/// SQMR step: given scalars, update d, lambda.  sc: [rho, sigma, tau, theta, theta_old, c]
__global__ void k_sqmr_dx(int n, const double* sc, const double* q, double* d, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double alpha = sc[0] / sc[1];
  const double c2 = sc[5] * sc[5];
  const double dn = c2 * sc[4] * sc[4] * d[i] + c2 * alpha * q[i];
  d[i] = dn;
  x[i] += dn;
}

// ---------------------------------------------------------------------------
// Krylov scalars on the device (only the status word crosses to the host):
// single-thread kernels between the dot products update them; the vector
// kernels read their coefficients from device memory.
// status[0]: 0 running, 1 converged, >= 2 breakdown code; status[1]: iterations
// ---------------------------------------------------------------------------
enum : int {
  KS_RHO = 32, KS_SIGMA, KS_A, KS_RR, KS_THETA, KS_THOLD, KS_C, KS_TAU, KS_T0, KS_RHON, KS_B, KS_REL,
  KS_RZ, KS_PKP, KS_PP, KS_RZN, KS_D0
};
enum : int { KST_RUN = 0, KST_CONV = 1, KST_SIGMA = 2, KST_RHO = 3, KST_PKP = 4, KST_RZ = 5 };

/// y += sgn * (*coef) * x
__global__ void k_axpy_s(int n, const double* coef, double sgn, const double* x, double* y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double c = sgn * *coef;
  if (i < n) y[i] += c * x[i];
}
/// y = x + (*coef) * y
__global__ void k_xpay_s(int n, const double* x, double* y, const double* coef) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double c = *coef;
  if (i < n) y[i] = x[i] + c * y[i];
}
/// SQMR: d = c^2 theta_old^2 d + c^2 a q; x += d
__global__ void k_sqmr_dx_s(int n, const double* sc, const double* q, double* d, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double c2 = sc[KS_C] * sc[KS_C];
  const double dn = c2 * sc[KS_THOLD] * sc[KS_THOLD] * d[i] + c2 * sc[KS_A] * q[i];
  d[i] = dn;
  x[i] += dn;
}
__global__ void k_ks_sqmr_init(double* sc, int* status) {
  const double t0 = sqrt(sc[KS_RR]);
  sc[KS_T0] = t0, sc[KS_TAU] = t0, sc[KS_THETA] = 0.0, sc[KS_REL] = 1.0;
  status[0] = (t0 == 0.0 || !(t0 > 0.0)) ? KST_CONV : KST_RUN, status[1] = 0;
  if (status[0] == KST_CONV) sc[KS_REL] = 0.0;
}
__global__ void k_ks_sqmr_a(double* sc, int* status) {
  const double sigma = sc[KS_SIGMA];
  if (sigma == 0.0 || !isfinite(sigma)) status[0] = KST_SIGMA;
  sc[KS_A] = sc[KS_RHO] / sigma;
}
__global__ void k_ks_sqmr_tau(double* sc, int* status, double tol) {
  const double rn = sqrt(sc[KS_RR]);
  const double th_old = sc[KS_THETA];
  const double theta = rn / sc[KS_TAU];
  const double c = 1.0 / sqrt(1.0 + theta * theta);
  const double tau = sc[KS_TAU] * theta * c;
  sc[KS_THOLD] = th_old, sc[KS_THETA] = theta, sc[KS_C] = c, sc[KS_TAU] = tau;
  sc[KS_REL] = tau / sc[KS_T0];  // quasi-residual tau_k <= tol ||r0|| (oracle rule)
  status[1] += 1;
  if (status[0] == KST_RUN && tau <= tol * sc[KS_T0]) status[0] = KST_CONV;
}
__global__ void k_ks_sqmr_b(double* sc, int* status) {
  if (sc[KS_RHO] == 0.0 && status[0] == KST_RUN) status[0] = KST_RHO;
  sc[KS_B] = sc[KS_RHON] / sc[KS_RHO];
  sc[KS_RHO] = sc[KS_RHON];
}
__global__ void k_ks_pcg_init(double* sc, int* status) {
  const double d0 = sqrt(fmax(sc[KS_RZ], 0.0));
  sc[KS_D0] = d0, sc[KS_REL] = 1.0;
  status[0] = (d0 == 0.0 || !(d0 > 0.0)) ? KST_CONV : KST_RUN, status[1] = 0;
  if (status[0] == KST_CONV) sc[KS_REL] = 0.0;
}
__global__ void k_ks_pcg_alpha(double* sc, int* status) {
  if (sc[KS_PKP] <= 1e-14 * sc[KS_PP]) status[0] = KST_PKP;
  sc[KS_A] = sc[KS_RZ] / sc[KS_PKP];
}
__global__ void k_ks_pcg_beta(double* sc, int* status, double tol) {
  const double rzn = sc[KS_RZN];
  const double delta = sqrt(fmax(rzn, 0.0));
  sc[KS_REL] = delta / sc[KS_D0];
  status[1] += 1;
  if (status[0] != KST_RUN) return;
  if (delta <= tol * sc[KS_D0]) {
    status[0] = KST_CONV;
    return;
  }
  if (rzn <= 0.0) status[0] = KST_RZ;
  sc[KS_B] = rzn / sc[KS_RZ];
  sc[KS_RZ] = rzn;
}

// ---------------------------------------------------------------------------
// Coarse space: dense symmetric GEMV  y = A x  (nc x nc, row-major)
// ---------------------------------------------------------------------------
__global__ void k_dense_gemv(int n, const double* A, const double* x, double* y) {
  __shared__ double red[32];
  const int i = blockIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s += A[(size_t)i * n + j] * x[j];
  s = block_sum(s, red);
  if (threadIdx.x == 0) y[i] = s;
}

/// y = A x for a dense row-major n x n A: a warp per row (16-byte loads when
/// the rows are 16-byte aligned, four loads in flight per lane), x staged in
/// shared memory; grid-stride over rows.  Coarse projector (G_c^T G_c)^{-1}.
__global__ void __launch_bounds__(256) k_dense_gemv_w(int n, const double* __restrict__ A,
                                                      const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec = (n & 1) == 0 && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  for (int row = blockIdx.x * 8 + warp; row < n; row += gridDim.x * 8) {
    const double* a = A + (size_t)row * n;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (vec) {
      const double2* a2 = reinterpret_cast<const double2*>(a);
      const int n2 = n >> 1;
      int j = lane;
      for (; j + 32 < n2; j += 64) {
        const double2 u = __ldg(a2 + j), v = __ldg(a2 + j + 32);
        s0 += u.x * xs[2 * j], s1 += u.y * xs[2 * j + 1];
        s2 += v.x * xs[2 * j + 64], s3 += v.y * xs[2 * j + 65];
      }
      if (j < n2) {
        const double2 u = __ldg(a2 + j);
        s0 += u.x * xs[2 * j], s1 += u.y * xs[2 * j + 1];
      }
    } else {
      for (int j = lane; j < n; j += 32) s0 += __ldg(a + j) * xs[j];
    }
    const double s = warp_sum((s0 + s2) + (s1 + s3));
    if (lane == 0) y[row] = s;
  }
}

/// CSR SpMV with a warp per row (long rows: G_c^T, ~400 entries per coarse
/// mode); y = alpha*A x + beta*y, fixed summation order.
__global__ void __launch_bounds__(256) k_spmv_warp(int nrows, const int* __restrict__ ptr,
                                                   const int* __restrict__ idx, const double* __restrict__ val,
                                                   const double* __restrict__ x, double* y, double alpha,
                                                   double beta) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= nrows) return;
  double s = 0.0;
  for (int q = ptr[row] + lane; q < ptr[row + 1]; q += 32) s += val[q] * x[idx[q]];
  s = warp_sum(s);
  if (lane == 0) y[row] = (beta == 0.0 ? 0.0 : beta * y[row]) + alpha * s;
}

/// Dense top of a single-problem sweep, pass 1: y = X[c0..c0+n) + folded
/// child contributions (fixed order).
/// Only contributions of the sparse levels (CB index < cb_top) count: the
/// top tasks' own couplings are inside W.
__global__ void k_dense_top_gather(int n, int c0, int cb_top, const int* __restrict__ fold_ptr,
                                   const int* __restrict__ fold_idx, const double* __restrict__ CB, const double* X,
                                   double* y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = X[c0 + i];
  for (int q = fold_ptr[c0 + i]; q < fold_ptr[c0 + i + 1]; ++q) {
    const int f = fold_idx[q];
    if (f < cb_top) v += CB[f];
  }
  y[i] = v;
}

/// pass 2: X[c0 + i] = sum_j W[i][j] y[j] (W = inverse of the top Schur
/// complement), one warp per row, y staged in shared memory.
__global__ void __launch_bounds__(256) k_dense_top_gemv(int n, int c0, const double* __restrict__ W,
                                                        const double* __restrict__ y, double* X) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int row = blockIdx.x * 8 + warp; row < n; row += gridDim.x * 8) {
    const double* w = W + (size_t)row * n;
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s += w[j] * ys[j];
    s = warp_sum(s);
    if (lane == 0) X[c0 + row] = s;
  }
}

/// Sparse levels of a single-problem system as dense per-task operators (one
/// CTA of four warps per task; operator column-major so a fixed input index
/// is a coalesced column):
/// mode 0 (forward): in = X[c0..c0+nct) + child contributions (fold lists,
///                   staged in parallel, summed per column in fixed order),
///                   out = [X[c0..); CB[cbo..cbo+cbl)]
/// mode 1 (backward): in = [X[c0..); X[cb_rows]] (ancestor values, final),
///                   out = X[c0..c0+nct).
__global__ void __launch_bounds__(128) k_dense_task(int t0, int mode, const int* __restrict__ c0,
                                                    const int* __restrict__ nct, const int* __restrict__ cbo,
                                                    const int* __restrict__ cbl, const long long* __restrict__ toff,
                                                    const double* __restrict__ T, const int* __restrict__ fold_ptr,
                                                    const int* __restrict__ fold_idx, const int* __restrict__ cb_rows,
                                                    double* X, double* CB) {
  constexpr int kFold = 1024;  // fold entries staged per task (longer lists use the serial path)
  __shared__ double in[128], fv[kFold];
  __shared__ int fp[129];
  const int q = t0 + blockIdx.x;
  const int n = nct[q], nb = cbl[q], nw = n + nb, c = c0[q];
  const int ni = mode == 0 ? n : nw, no = mode == 0 ? nw : n;
  if (mode == 0) {
    for (int i = threadIdx.x; i <= n; i += blockDim.x) fp[i] = fold_ptr[c + i];
    __syncthreads();
    const int f0 = fp[0], nf = fp[n] - f0;
    const bool staged = nf <= kFold;
    if (staged) {
      for (int f = threadIdx.x; f < nf; f += blockDim.x) fv[f] = CB[fold_idx[f0 + f]];
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double v = X[c + i];
      if (staged)
        for (int f = fp[i]; f < fp[i + 1]; ++f) v += fv[f - f0];  // fixed order
      else
        for (int f = fp[i]; f < fp[i + 1]; ++f) v += CB[fold_idx[f]];
      in[i] = v;
    }
  } else {
    for (int i = threadIdx.x; i < nw; i += blockDim.x) in[i] = i < n ? X[c + i] : X[cb_rows[cbo[q] + i - n]];
  }
  __syncthreads();  // every input staged before any output overwrites X
  const double* A = T + toff[q];
  for (int r = threadIdx.x; r < no; r += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = 0;
    for (; j + 4 <= ni; j += 4) {
      const double v0 = A[(long long)j * no + r], v1 = A[(long long)(j + 1) * no + r];
      const double v2 = A[(long long)(j + 2) * no + r], v3 = A[(long long)(j + 3) * no + r];
      a0 += v0 * in[j], a1 += v1 * in[j + 1], a2 += v2 * in[j + 2], a3 += v3 * in[j + 3];
    }
    for (; j < ni; ++j) a0 += A[(long long)j * no + r] * in[j];
    const double v = (a0 + a1) + (a2 + a3);
    if (r < n) X[c + r] = v;
    else CB[cbo[q] + r - n] = v;
  }
}

}  // namespace dev
}  // namespace pf
