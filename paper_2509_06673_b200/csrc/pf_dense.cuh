// pf_dense.cuh — dense FP64 linear algebra on the tensor cores (north-star
// item 2 / SURVEY 2.2 "dense Cholesky of G^T G on DMMA"): a tiled DGEMM on
// mma.sync.m8n8k4.f64 and the blocked Cholesky + explicit inverse of the
// coarse matrix G_c^T G_c built from it (setup, once per run).
//
// Layout: column-major, leading dimensions in elements.  Every kernel sums in
// a fixed order (deterministic).
#pragma once

#include <cuda_runtime.h>

namespace pf {
namespace dev {

constexpr int kDgM = 64, kDgN = 64, kDgK = 16, kDgThreads = 256, kDgLd = kDgK + 4;

/// C = beta C + alpha opA(A) opB(B), C M x N, K inner.
/// opA(i,k) = TA ? A[k + i lda] : A[i + k lda];  opB(k,j) = TB ? B[j + k ldb] : B[k + j ldb].
/// lower: CTA tiles strictly above the diagonal are skipped (SYRK-style
/// updates of a lower triangle).  ktri: opA(i,k) = 0 for k < i and
/// opB(k,j) = 0 for k < j (lower-triangular Y in Y^T Y): the K loop of a tile
/// starts at max(row0, col0), below which every product vanishes.
/// 64x64 tile per 256-thread CTA; warp w: rows 16 (w % 4) .. +16, columns
/// 32 (w / 4) .. +32 as 2 x 4 m8n8k4 tiles; K chunks of 16 staged in shared
/// memory (rows of 20 doubles: conflict-free fragment loads), the next chunk
/// prefetched into registers while the current one is multiplied.
template <bool TA, bool TB>
__global__ void __launch_bounds__(kDgThreads) k_dgemm(int M, int N, int K, double alpha, const double* __restrict__ A,
                                                     int lda, const double* __restrict__ B, int ldb, double beta,
                                                     double* C, int ldc, int lower, int ktri) {
  __shared__ __align__(16) double As[kDgM][kDgLd];
  __shared__ __align__(16) double Bs[kDgN][kDgLd];
  const int r0 = blockIdx.x * kDgM, c0 = blockIdx.y * kDgN;
  if (lower && r0 + kDgM <= c0) return;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int wr = (wp & 3) * 16, wc = (wp >> 2) * 32;
  const int kbeg = ktri ? (max(r0, c0) / kDgK) * kDgK : 0;
  // loader: 4 elements of A and 4 of B per thread per chunk
  double ra[4], rb[4];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + kDgThreads * e;
      // A tile 64 x 16: coalesced along i (column-major) or along k (transposed)
      const int ai = TA ? idx / kDgK : idx % kDgM, ak = TA ? idx % kDgK : idx / kDgM;
      const int gi = r0 + ai, gk = k0 + ak;
      ra[e] = (gi < M && gk < K) ? (TA ? A[gk + (long long)gi * lda] : A[gi + (long long)gk * lda]) : 0.0;
      // B tile 16 x 64 (k x j): coalesced along k (column-major) or along j (transposed)
      const int bj = TB ? idx % kDgN : idx / kDgK, bk = TB ? idx / kDgN : idx % kDgK;
      const int gj = c0 + bj, gk2 = k0 + bk;
      rb[e] = (gj < N && gk2 < K) ? (TB ? B[gj + (long long)gk2 * ldb] : B[gk2 + (long long)gj * ldb]) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + kDgThreads * e;
      const int ai = TA ? idx / kDgK : idx % kDgM, ak = TA ? idx % kDgK : idx / kDgM;
      As[ai][ak] = ra[e];
      const int bj = TB ? idx % kDgN : idx / kDgK, bk = TB ? idx / kDgN : idx % kDgK;
      Bs[bj][bk] = rb[e];
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (kbeg < K) load(kbeg);
  for (int k0 = kbeg; k0 < K; k0 += kDgK) {
    __syncthreads();  // the previous chunk's fragments are consumed
    store();
    __syncthreads();
    if (k0 + kDgK < K) load(k0 + kDgK);  // in flight during the MMAs below
#pragma unroll
    for (int k4 = 0; k4 < kDgK; k4 += 4) {
      const int kk = k4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[wr + i * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[wc + j * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1])
                       : "d"(af[i]), "d"(bf[j]));
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + wr + i * 8 + (lane >> 2), c = c0 + wc + j * 8 + (lane & 3) * 2 + h;
        if (r >= M || c >= N || (lower && r < c)) continue;
        double* cp = C + r + (long long)c * ldc;
        *cp = (beta == 0.0 ? 0.0 : beta * *cp) + alpha * acc[i][j][h];
      }
}

/// Diagonal block of the blocked Cholesky: A[k0:k0+nb, k0:k0+nb] = L L^T in
/// place (lower), and Linv = L^{-1} (nb x nb, column-major, ld nb; zero above
/// the diagonal).  One CTA; the block staged in shared memory.
/// With `sg` (signed Cholesky of a symmetric quasi-definite matrix, A = L S L^T
/// with S = diag(sg) of +-1, no pivoting): the pivot's sign goes to sg[k0 + j],
/// l_jj = sqrt(|d_j|), l_ij = r_ij / (s_j l_jj); a pivot below pivmin fails.
constexpr int kChNb = 64;
__global__ void __launch_bounds__(256) k_potrf_diag(int n, double* A, int lda, int k0, double* Linv, int* err,
                                                    int* sg = nullptr, double pivmin = 0.0) {
  __shared__ double S[kChNb][kChNb + 1];
  __shared__ double sj[kChNb];
  const int nb = min(kChNb, n - k0), tid = threadIdx.x;
  for (int q = tid; q < nb * nb; q += blockDim.x) {
    const int i = q % nb, j = q / nb;
    S[i][j] = i >= j ? A[(k0 + i) + (long long)(k0 + j) * lda] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = S[j][j];
    const double sgn = sg ? (d < 0.0 ? -1.0 : 1.0) : 1.0;
    if (sg ? !(fabs(d) > pivmin) : !(d > 0.0)) {
      if (tid == 0) atomicExch(err, 1 + k0 + j);
      return;
    }
    const double s = sqrt(fabs(d));
    __syncthreads();
    if (tid == 0) S[j][j] = s, sj[j] = sgn;
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) S[i][j] /= sgn * s;
    __syncthreads();
    // right-looking update of the remaining lower triangle
    for (int q = tid; q < (nb - j - 1) * (nb - j - 1); q += blockDim.x) {
      const int i = j + 1 + q % (nb - j - 1), c = j + 1 + q / (nb - j - 1);
      if (i >= c) S[i][c] -= sgn * S[i][j] * S[c][j];
    }
    __syncthreads();
  }
  for (int q = tid; q < nb * nb; q += blockDim.x) {
    const int i = q % nb, j = q / nb;
    if (i >= j) A[(k0 + i) + (long long)(k0 + j) * lda] = S[i][j];
  }
  if (sg)
    for (int j = tid; j < nb; j += blockDim.x) sg[k0 + j] = sj[j] < 0.0 ? -1 : 1;
  // L^{-1}: thread per column, forward substitution (column j of the inverse)
  for (int j = tid; j < nb; j += blockDim.x) {
    double x[kChNb];
    for (int i = 0; i < nb; ++i) {
      double v = i == j ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) v -= S[i][k] * x[k];
      x[i] = i < j ? 0.0 : v / S[i][i];
    }
    for (int i = 0; i < nb; ++i) Linv[i + (long long)j * kChNb] = i < j ? 0.0 : x[i];
  }
}

/// signed Cholesky helpers: T = P (copy, m x kb, ld_t = m) and P[:, j] *= sg[j]
/// (the panel becomes L21 = A21 L11^{-T} S11; T keeps A21 L11^{-T} = L21 S11
/// for the trailing update A22 -= L21 T^T)
__global__ void k_panel_signs(int m, int kb, double* P, int ldp, double* T, const int* __restrict__ sg) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)m * kb) return;
  const int i = (int)(q % m), j = (int)(q / m);
  const double v = P[i + (long long)j * ldp];
  T[i + (long long)j * m] = v;
  P[i + (long long)j * ldp] = sg[j] < 0 ? -v : v;
}

/// D[i + j ld] = sg[i] * Y[i + j ld] (rows scaled by the pivot signs: S Y)
__global__ void k_scale_rows(int n, const double* __restrict__ Y, double* D, int ld, const int* __restrict__ sg) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)n * n) return;
  const int i = (int)(q % n);
  const long long j = q / n;
  const double v = Y[i + j * ld];
  D[i + j * ld] = sg[i] < 0 ? -v : v;
}

/// T[:, c0 + i] += e_i for i < nb (rows 0..nb of a block row): the identity
/// block of E_i - L_{i,<i} Y_{<i}
__global__ void k_add_identity(double* T, int ldt, int c0, int nb) {
  const int i = threadIdx.x;
  if (i < nb) T[i + (long long)(c0 + i) * ldt] += 1.0;
}

/// copy a nb x N block row (ld_src) into rows [r0, r0 + nb) of Y (ld_y)
__global__ void k_copy_rows(int nb, int N, const double* S, int lds, double* Y, int ldy, int r0) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)nb * N) return;
  const int i = (int)(q % nb), j = (int)(q / nb);
  Y[(r0 + i) + (long long)j * ldy] = S[i + (long long)j * lds];
}


// ---------------------------------------------------------------------------
// Direct interface solve (the GPU analogue of MonolithicSolver, feti.hpp:313-440)
// ---------------------------------------------------------------------------
/// F[g_i, g_j] += F_s[i][j] for every owned subdomain (CTA per subdomain; F_s
/// row-major n_s x n_s at op[s], local multiplier g = lam[loff[s] + i], < 0:
/// padding).  An entry of F receives at most two contributions (the multipliers
/// of one interface lie in its two subdomains; two distinct interfaces share at
/// most one), and (0 + a) + b == (0 + b) + a in IEEE arithmetic, so the atomic
/// sums are deterministic.  F column-major n x n (symmetric).
__global__ void k_dense_assemble(int np, const int* __restrict__ nloc, const long long* __restrict__ op,
                                 const double* __restrict__ Fs, const long long* __restrict__ loff,
                                 const int* __restrict__ lam, double* F, int n) {
  const int s = blockIdx.x, m = nloc[s];
  const double* A = Fs + op[s];
  const int* g = lam + loff[s];
  for (long long q = threadIdx.x; q < (long long)m * m; q += blockDim.x) {
    const int i = (int)(q / m), j = (int)(q % m);
    const int gi = g[i], gj = g[j];
    if (gi >= 0 && gj >= 0) atomicAdd(F + (long long)gi + (long long)gj * n, A[q]);
  }
}

/// G dense (n x nc, column-major, zeroed) from the CSR of G^T: column c = row c
__global__ void k_csr_rows_to_cols(int nc, const int* __restrict__ ptr, const int* __restrict__ idx,
                                   const double* __restrict__ val, double* G, int n) {
  const int c = blockIdx.x;
  for (int q = ptr[c] + threadIdx.x; q < ptr[c + 1]; q += blockDim.x) G[idx[q] + (long long)c * n] = val[q];
}

/// Z row-major with ld: Z[i * ld + n + c] = Yc[i + c * n] (the coarse columns
/// of the augmented solution operator [Z | Y_c])
__global__ void k_aug_coarse(int n, int nc, const double* __restrict__ Yc, double* Z, long long ld) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)n * nc) return;
  const int i = (int)(q % n), c = (int)(q / n);
  Z[(long long)i * ld + n + c] = Yc[q];
}

/// y = A x for a row-major M x N A (ld even: 16-byte rows) too wide for x to
/// sit in shared memory whole: x staged in chunks of kGvChunk, a warp per two
/// rows (16-byte loads, eight in flight per lane and row), partial sums in a
/// fixed lane order and a warp tree: deterministic.  HBM-bound: 8 B per
/// matrix value, each read once.
constexpr int kGvChunk = 4096, kGvRows = 2, kGvWarps = 8;
__global__ void __launch_bounds__(32 * kGvWarps) k_gemv_rows(int M, int N, const double* __restrict__ A,
                                                            long long ld, const double* __restrict__ x,
                                                            double* __restrict__ y) {
  __shared__ __align__(16) double xs[kGvChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r0 = (blockIdx.x * kGvWarps + warp) * kGvRows;
  double acc[kGvRows];
#pragma unroll
  for (int r = 0; r < kGvRows; ++r) acc[r] = 0.0;
  for (int c0 = 0; c0 < N; c0 += kGvChunk) {
    const int cn = min(kGvChunk, N - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += blockDim.x) xs[i] = x[c0 + i];
    __syncthreads();
    const int npair = cn >> 1;
#pragma unroll
    for (int r = 0; r < kGvRows; ++r) {
      const int row = r0 + r;
      if (row >= M) continue;
      const double2* a2 = reinterpret_cast<const double2*>(A + (long long)row * ld + c0);
      double s0 = 0.0, s1 = 0.0;
      int p = lane;
      for (; p + 7 * 32 < npair; p += 8 * 32) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(a2 + p + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = 2 * (p + 32 * u);
          s0 += v[u].x * xs[c];
          s1 += v[u].y * xs[c + 1];
        }
      }
      for (; p < npair; p += 32) {
        const double2 v = __ldcs(a2 + p);
        s0 += v.x * xs[2 * p];
        s1 += v.y * xs[2 * p + 1];
      }
      if ((cn & 1) && lane == 0) s0 += A[(long long)row * ld + c0 + cn - 1] * xs[cn - 1];
      acc[r] += s0 + s1;
    }
  }
#pragma unroll
  for (int r = 0; r < kGvRows; ++r) {
    double v = acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && r0 + r < M) y[r0 + r] = v;
  }
}

}  // namespace dev
}  // namespace pf
