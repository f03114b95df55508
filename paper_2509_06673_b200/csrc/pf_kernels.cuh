// pf_kernels.cuh — sm_100a kernels of the FETI engine.
//
// Hot path (per Krylov iteration): the batched supernodal LDL^T sweeps
// (k_leaf_fwd / k_top / k_leaf_bwd) over every subdomain factor, the
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
  int n, nsn, ntask, top_sn0, top_c0;
  int sn_base, task_base, fold_base;  // into sn_* / task_* / fold_ptr arrays
  long long row_base, cb_base;        // into rows(slot) / cb_rows + fold_idx
};

struct SolveSet {
  const TypeDesc* types;
  const int *sn_col0, *sn_ncol, *sn_nrow;
  const long long *sn_rowoff, *sn_valoff;  // relative to the type's row/value base
  const int* slot;
  const int *task_sn0, *task_sn1, *task_c0, *task_c1, *task_cboff, *task_cblen;
  const int* cb_rows;                      // relative to type cb_base
  const int* fold_ptr;                     // per type: n_top+1 entries (relative), at fold_base
  const int* fold_idx;                     // cb slot indices (relative to the problem's cb region)
  // problems
  int nprob;
  const int* prob_type;
  const long long *prob_lval, *prob_x, *prob_cb;
  // leaf work list
  int nwork;
  const int *work_prob, *work_task;
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

/// Leaf forward sweep + diagonal scaling: one warp per (problem, task).
/// Workspace per warp in shared memory: task columns then contribution rows.
__global__ void k_leaf_fwd(SolveSet S, int ws_max) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * (blockDim.x >> 5) + wib;
  if (w >= S.nwork) return;
  double* ws = smem + (size_t)wib * ws_max;
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nc_task = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const double* L = S.L + S.prob_lval[p];
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride;
    for (int i = lane; i < nc_task; i += kWarp) ws[i] = X[c0 + i];
    for (int i = lane; i < cbl; i += kWarp) ws[nc_task + i] = 0.0;
    __syncwarp();
    for (int k = S.task_sn0[t]; k < S.task_sn1[t]; ++k) {
      const int sk = T.sn_base + k;
      const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
      const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
      const double* V = L + S.sn_valoff[sk];
      for (int j = 0; j < nc; ++j) {
        const double xj = ws[sl[j]];
        const double* col = V + col_off(j, m) - (j + 1);
        for (int i = j + 1 + lane; i < m; i += kWarp) ws[sl[i]] -= col[i] * xj;
        __syncwarp();
      }
    }
    const double* Dp = S.D + S.prob_x[p];
    for (int i = lane; i < nc_task; i += kWarp) X[c0 + i] = ws[i] / Dp[c0 + i];
    double* CB = S.CB + S.prob_cb[p] + r * S.cb_stride + cbo;
    for (int i = lane; i < cbl; i += kWarp) CB[i] = ws[nc_task + i];
    __syncwarp();
  }
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

/// Top part: fold contributions, forward, diagonal, backward. One CTA per problem.
__global__ void k_top(SolveSet S, int in_smem) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  const int p = blockIdx.x;
  if (p >= S.nprob) return;
  const TypeDesc T = S.types[S.prob_type[p]];
  const int ntop = T.n - T.top_c0;
  if (ntop == 0) return;
  const double* L = S.L + S.prob_lval[p];
  const double* Dp = S.D + S.prob_x[p] + T.top_c0;
  const int* fp = S.fold_ptr + T.fold_base;
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride + T.top_c0;
    double* ws = in_smem ? smem : X;  // large top parts work in place in global memory (L2)
    const double* CB = S.CB + S.prob_cb[p] + r * S.cb_stride;
    for (int i = threadIdx.x; i < ntop; i += blockDim.x) {
      double v = X[i];
      for (int q = fp[i]; q < fp[i + 1]; ++q) v += CB[S.fold_idx[T.cb_base + q]];
      ws[i] = v;
    }
    __syncthreads();
    for (int k = T.top_sn0; k < T.nsn; ++k) {
      const int sk = T.sn_base + k;
      const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
      const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
      const double* V = L + S.sn_valoff[sk];
      for (int j = 0; j < nc; ++j) {
        const double xj = ws[sl[j]];
        const double* col = V + col_off(j, m) - (j + 1);
        for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) ws[sl[i]] -= col[i] * xj;
        __syncthreads();
      }
    }
    for (int i = threadIdx.x; i < ntop; i += blockDim.x) ws[i] /= Dp[i];
    __syncthreads();
    for (int k = T.nsn - 1; k >= T.top_sn0; --k) {
      const int sk = T.sn_base + k;
      const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
      const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
      const double* V = L + S.sn_valoff[sk];
      for (int j = nc - 1; j >= 0; --j) {
        const double* col = V + col_off(j, m) - (j + 1);
        double acc = 0.0;
        for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) acc += col[i] * ws[sl[i]];
        const double s = block_sum(acc, red);
        if (threadIdx.x == 0) ws[sl[j]] -= s;
        __syncthreads();
      }
    }
    if (in_smem)
      for (int i = threadIdx.x; i < ntop; i += blockDim.x) X[i] = ws[i];
    __syncthreads();
  }
}

/// Leaf backward sweep: one warp per (problem, task); ancestors read from X.
__global__ void k_leaf_bwd(SolveSet S, int ws_max) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * (blockDim.x >> 5) + wib;
  if (w >= S.nwork) return;
  double* ws = smem + (size_t)wib * ws_max;
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nc_task = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const int* cbr = S.cb_rows + T.cb_base + cbo;
  const double* L = S.L + S.prob_lval[p];
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride;
    for (int i = lane; i < nc_task; i += kWarp) ws[i] = X[c0 + i];
    for (int i = lane; i < cbl; i += kWarp) ws[nc_task + i] = X[cbr[i]];
    __syncwarp();
    for (int k = S.task_sn1[t] - 1; k >= S.task_sn0[t]; --k) {
      const int sk = T.sn_base + k;
      const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
      const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
      const double* V = L + S.sn_valoff[sk];
      for (int j = nc - 1; j >= 0; --j) {
        const double* col = V + col_off(j, m) - (j + 1);
        double acc = 0.0;
        for (int i = j + 1 + lane; i < m; i += kWarp) acc += col[i] * ws[sl[i]];
        acc = warp_sum(acc);
        if (lane == 0) ws[sl[j]] -= acc;
        __syncwarp();
      }
    }
    for (int i = lane; i < nc_task; i += kWarp) X[c0 + i] = ws[i];
    __syncwarp();
  }
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
                          const long long* prob_perm, const int* perm, const double* src, double* X,
                          const double* bias, double bscale) {
  const int p = blockIdx.y;
  if (p >= nprob) return;
  const int n = prob_n[p];
  const int* pm = perm + prob_perm[p];
  const double* s = src + prob_src[p];
  double* x = X + prob_x[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = s[pm[i]];
  (void)bias, (void)bscale;
}

/// permute out: dst[so + perm[pos]] = X[xo + pos]
__global__ void k_perm_out(int nprob, const long long* prob_x, const long long* prob_dst, const int* prob_n,
                           const long long* prob_perm, const int* perm, const double* X, double* dst) {
  const int p = blockIdx.y;
  if (p >= nprob) return;
  const int n = prob_n[p];
  const int* pm = perm + prob_perm[p];
  double* d = dst + prob_dst[p];
  const double* x = X + prob_x[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[pm[i]] = x[i];
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

}  // namespace dev
}  // namespace pf
