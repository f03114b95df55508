// pf_iface.cuh — device side of the sparse direct interface solve
// (pf_iface.hpp: nested dissection of the multipliers over the subdomain grid).
//
// Per front R = [sep | bdry] the factorisation keeps two dense row-major
// operators (block LDL^T with the pivot block inverted explicitly, so the
// solve is GEMVs only — no triangular dependency chains):
//   T = A21 A11^{-1}            (nbdry x nsep)        forward : c_bdry -= T c_sep
//   M = [A11^{-1} | -T^T]       (nsep x (nsep+nbdry)) backward: x_sep = M [c_sep ; x_bdry]
// Every value is read once per solve: the solve is HBM-bound at
// 8 B x sum_R nsep (nsep + 2 nbdry).  One launch per tree depth and direction
// handles all fronts of that depth.
//
// Determinism: a boundary multiplier of R is also a boundary multiplier of at
// most one other front of the same depth (the rectangle on the other side of
// its interface), so forward updates go to two accumulators u0 / u1 chosen by
// the side of the interface R lies on: one writer per entry and launch, and
// c = (b + u0) + u1 is summed in that order.
#pragma once

#include <cuda_runtime.h>

#include "pf_kernels.cuh"

namespace pf {
namespace dev {

struct IfaceFrontDev {
  long long offM, offT, offI;  // into M, T (doubles) and idx / side
  int nsep, nbdry, ldM, ldT;
};

struct IfaceSolve {
  const IfaceFrontDev* fronts;
  const int2* work;            // per CTA: (front, first row)
  const int* idx;
  const unsigned char* side;   // per idx entry (separator entries unused)
  const double* M;
  const double* T;
  const double* b;             // right-hand side (read only)
  double* u0;
  double* u1;                  // forward accumulators
  double* x;                   // solution
};

constexpr int kIfChunk = 4096, kIfThreads = 256;

/// One depth of the forward (MODE 0) or backward (MODE 1) pass.  A group of LPR
/// lanes owns RPG rows of its front and walks them together (RPG x 2 16-byte
/// loads in flight per lane); the input vector is staged in shared memory in
/// chunks of kIfChunk entries through the front's index list.
template <int MODE, int LPR, int RPG>
__global__ void __launch_bounds__(kIfThreads) k_iface_gemv(IfaceSolve S, int work0) {
  __shared__ __align__(16) double xs[kIfChunk];
  constexpr int G = kIfThreads / LPR;  // row groups per CTA
  const int2 w = S.work[work0 + blockIdx.x];
  const IfaceFrontDev F = S.fronts[w.x];
  const int ncols = MODE ? F.nsep + F.nbdry : F.nsep;
  const int nrows = MODE ? F.nsep : F.nbdry;
  const long long ld = MODE ? F.ldM : F.ldT;
  const double* A = MODE ? S.M + F.offM : S.T + F.offT;
  const int* idx = S.idx + F.offI;
  const int g = threadIdx.x / LPR, l = threadIdx.x % LPR;
  int row[RPG];
  const double2* a2[RPG];
  double acc[RPG];
#pragma unroll
  for (int q = 0; q < RPG; ++q) {
    row[q] = w.y + g + q * G;
    // rows past the end read row 0 of the front (valid memory), their sums are dropped
    a2[q] = reinterpret_cast<const double2*>(A + (row[q] < nrows ? row[q] : 0) * ld);
    acc[q] = 0.0;
  }
  if (kPdlEarly) pdl_trigger();
  pdl_wait();
  for (int c0 = 0; c0 < ncols; c0 += kIfChunk) {
    const int cn = min(kIfChunk, ncols - c0);
    __syncthreads();
    for (int k = threadIdx.x; k < cn + (cn & 1); k += kIfThreads) {
      double v = 0.0;
      if (k < cn) {
        const int i = idx[c0 + k];
        v = (!MODE || c0 + k < F.nsep) ? (S.b[i] + S.u0[i]) + S.u1[i] : S.x[i];
      }
      xs[k] = v;
    }
    __syncthreads();
    const int npair = (cn + 1) >> 1, pb = c0 >> 1;
    double s0[RPG], s1[RPG];
#pragma unroll
    for (int q = 0; q < RPG; ++q) s0[q] = s1[q] = 0.0;
    int p = l;
    for (; p + LPR < npair; p += 2 * LPR) {
      double2 v[RPG][2];
#pragma unroll
      for (int q = 0; q < RPG; ++q) v[q][0] = __ldcs(a2[q] + pb + p), v[q][1] = __ldcs(a2[q] + pb + p + LPR);
      const double2 xa = *reinterpret_cast<const double2*>(xs + 2 * p);
      const double2 xb = *reinterpret_cast<const double2*>(xs + 2 * (p + LPR));
#pragma unroll
      for (int q = 0; q < RPG; ++q) {
        s0[q] += v[q][0].x * xa.x, s1[q] += v[q][0].y * xa.y;
        s0[q] += v[q][1].x * xb.x, s1[q] += v[q][1].y * xb.y;
      }
    }
    if (p < npair) {
      const double2 xa = *reinterpret_cast<const double2*>(xs + 2 * p);
#pragma unroll
      for (int q = 0; q < RPG; ++q) {
        const double2 v = __ldcs(a2[q] + pb + p);
        s0[q] += v.x * xa.x, s1[q] += v.y * xa.y;
      }
    }
#pragma unroll
    for (int q = 0; q < RPG; ++q) acc[q] += s0[q] + s1[q];
  }
#pragma unroll
  for (int q = 0; q < RPG; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0 && row[q] < nrows) {
      if (MODE) {
        S.x[idx[row[q]]] = v;
      } else {
        const int k = F.nsep + row[q];
        double* u = S.side[F.offI + k] ? S.u1 : S.u0;
        u[idx[k]] -= v;
      }
    }
  }
}

/// Extend-add of a child's Schur complement (lower triangle of the mc x mc
/// block at C, leading dimension ldc) into the parent front A (m x m, lower
/// triangle): A[max(pi,pj), min(pi,pj)] += C[i, j], i >= j, p = map.  rowmajor:
/// C holds a subdomain's F_s row-major (entry (i, j) at i ldc + j).
__global__ void k_iface_extend_add(int mc, const double* __restrict__ C, long long ldc, int rowmajor,
                                   const int* __restrict__ map, double* A, long long m) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)mc * mc) return;
  const int i = (int)(q % mc), j = (int)(q / mc);
  if (i < j) return;
  const int pi = map[i], pj = map[j];
  if (pi < 0 || pj < 0) return;
  const double v = rowmajor ? C[(long long)i * ldc + j] : C[i + (long long)j * ldc];
  A[(long long)max(pi, pj) + (long long)min(pi, pj) * m] += v;
}

/// Mirror the lower triangle of the leading ns x ns block of A (ld m) into the
/// packed P (ld ns), both triangles.
__global__ void k_iface_copy_sym(int ns, const double* __restrict__ A, long long m, double* P) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)ns * ns) return;
  const int i = (int)(q % ns), j = (int)(q / ns);
  P[q] = i >= j ? A[i + (long long)j * m] : A[j + (long long)i * m];
}

/// Front storage from X = A11^{-1} (ns x ns, column-major, symmetric) and
/// Tc = A21 A11^{-1} (nb x ns, column-major): M row r = [X(:, r) ; -Tc(:, r)],
/// T row j = Tc(j, :).
__global__ void k_iface_store(int ns, int nb, const double* __restrict__ X, const double* __restrict__ Tc, double* M,
                              int ldM, double* T, int ldT) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nM = (long long)ns * (ns + nb);
  if (q < nM) {
    const int k = (int)(q % (ns + nb)), r = (int)(q / (ns + nb));
    M[(long long)r * ldM + k] = k < ns ? X[k + (long long)r * ns] : -Tc[(k - ns) + (long long)r * nb];
  } else if (q < nM + (long long)nb * ns) {
    const long long t = q - nM;
    const int j = (int)(t % nb), r = (int)(t / nb);  // coalesced read of Tc
    T[(long long)j * ldT + r] = Tc[t];
  }
}

/// Multi-right-hand-side solves (setup of the coarse border, W = F^{-1} G_c):
/// rows idx[0..r) of the column-major n x k matrix C gathered into the dense
/// r x k block G (ld r); with C2 given, rows >= r1 come from C2 instead.
__global__ void k_iface_rows_gather(int r, int k, const int* __restrict__ idx, const double* __restrict__ C,
                                    const double* __restrict__ C2, int r1, long long n, double* __restrict__ G) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)r * k) return;
  const int i = (int)(q % r);
  const long long j = q / r;
  G[q] = (C2 && i >= r1 ? C2 : C)[idx[i] + j * n];
}
/// C[idx[i], j] = G[i, j] (sub = 0) or C[idx[i], j] -= G[i, j] (sub = 1); the
/// rows of one front are distinct, fronts are processed one after the other
__global__ void k_iface_rows_scatter(int r, int k, const int* __restrict__ idx, const double* __restrict__ G, int sub,
                                     long long n, double* C) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)r * k) return;
  const int i = (int)(q % r);
  const long long j = q / r;
  double* c = C + idx[i] + j * n;
  *c = sub ? *c - G[q] : G[q];
}

/// Y[i * ld + c] = X[i + c * n] (column-major n x nc -> row-major with ld)
__global__ void k_iface_to_rows(int n, int nc, const double* __restrict__ X, double* Y, long long ld) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)n * nc) return;
  const int i = (int)(q % n), c = (int)(q / n);
  Y[(long long)i * ld + c] = X[q];
}

}  // namespace dev
}  // namespace pf
