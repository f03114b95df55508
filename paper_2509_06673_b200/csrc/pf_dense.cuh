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
constexpr int kChNb = 64;
__global__ void __launch_bounds__(256) k_potrf_diag(int n, double* A, int lda, int k0, double* Linv, int* err) {
  __shared__ double S[kChNb][kChNb + 1];
  const int nb = min(kChNb, n - k0), tid = threadIdx.x;
  for (int q = tid; q < nb * nb; q += blockDim.x) {
    const int i = q % nb, j = q / nb;
    S[i][j] = i >= j ? A[(k0 + i) + (long long)(k0 + j) * lda] : 0.0;
  }
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    const double d = S[j][j];
    if (!(d > 0.0)) {
      if (tid == 0) atomicExch(err, 1);
      return;
    }
    const double s = sqrt(d);
    __syncthreads();
    if (tid == 0) S[j][j] = s;
    for (int i = j + 1 + tid; i < nb; i += blockDim.x) S[i][j] /= s;
    __syncthreads();
    // right-looking update of the remaining lower triangle
    for (int q = tid; q < (nb - j - 1) * (nb - j - 1); q += blockDim.x) {
      const int i = j + 1 + q % (nb - j - 1), c = j + 1 + q / (nb - j - 1);
      if (i >= c) S[i][c] -= S[i][j] * S[c][j];
    }
    __syncthreads();
  }
  for (int q = tid; q < nb * nb; q += blockDim.x) {
    const int i = q % nb, j = q / nb;
    if (i >= j) A[(k0 + i) + (long long)(k0 + j) * lda] = S[i][j];
  }
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

}  // namespace dev
}  // namespace pf
