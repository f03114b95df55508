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
  int n, nsn, ntask;
  int sn_base, task_base;            // into sn_* / task_* arrays
  long long row_base, cb_base;       // into slot / cb_rows
  long long fold_base, foldidx_base; // into fold_ptr (n+1 per type) / fold_idx
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
  // problems
  int nprob;
  const int* prob_type;
  const long long *prob_lval, *prob_x, *prob_cb;
  // work list of one level: (problem, type-relative task)
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

// ---------------------------------------------------------------------------
// Panel primitives.  A supernode (nc columns, m rows, packed strict-lower
// trapezoid, column-major) is processed in panels of up to 32 columns:
//   forward : 32x32 unit-lower triangle by one warp with shuffles, then the
//             rows below the panel updated with coalesced column reads;
//   backward: rows below the panel reduced into 32 partial sums (warp
//             transpose-reduction, 31 shuffles), then the transposed triangle.
// All loads of a panel's off-diagonal block are independent of x, so they
// are issued back to back (memory-level parallelism), and there is no
// per-column barrier.
// ---------------------------------------------------------------------------

__device__ __forceinline__ double Lval(const double* V, int m, int i, int j) {  // L(i, j), i > j
  return V[col_off(j, m) + (i - j - 1)];
}

/// lane l ends with sum over lanes of acc[l] (acc fully unrolled in registers)
__device__ __forceinline__ double transpose_reduce32(double (&acc)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      const double send = upper ? acc[k] : acc[k + off];
      const double keep = upper ? acc[k + off] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return acc[0];
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

/// Forward elimination of one panel [p0, p0+pw) of a supernode (pw <= PW).
template <int PW>
__device__ __forceinline__ void warp_fwd_panel(const double* __restrict__ V, const int* __restrict__ sl, int m, int p0,
                                               int pw, double* ws, double* xp, int lane) {
  int cb[PW];  // offsets inside one supernode fit in 32 bits
#pragma unroll
  for (int j = 0; j < PW; ++j) cb[j] = j < pw ? (int)(col_off(p0 + j, m) - (p0 + j) - 1) : 0;
  double xi = lane < pw ? ws[sl[p0 + lane]] : 0.0;
  double lrow[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) lrow[j] = (j < pw && lane > j && lane < pw) ? V[cb[j] + p0 + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < PW; ++j) xi -= lrow[j] * __shfl_sync(0xffffffffu, xi, j);
  if (lane < pw) ws[sl[p0 + lane]] = xi;
  if (lane < PW) xp[lane] = xi;
  __syncwarp();
  for (int r = p0 + pw + lane; r < m; r += 32) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < PW; ++j)
      if (j < pw) acc += V[cb[j] + r] * xp[j];
    ws[sl[r]] -= acc;
  }
  __syncwarp();
}

/// Warp forward elimination of one supernode on workspace ws (slots sl).
__device__ __forceinline__ void warp_fwd_sn(const double* __restrict__ V, const int* __restrict__ sl, int nc, int m,
                                            double* ws, double* xp, int lane) {
  for (int p0 = 0; p0 < nc; p0 += 32) {
    const int pw = min(32, nc - p0);
    if (pw <= 4) warp_fwd_panel<4>(V, sl, m, p0, pw, ws, xp, lane);
    else if (pw <= 8) warp_fwd_panel<8>(V, sl, m, p0, pw, ws, xp, lane);
    else if (pw <= 16) warp_fwd_panel<16>(V, sl, m, p0, pw, ws, xp, lane);
    else warp_fwd_panel<32>(V, sl, m, p0, pw, ws, xp, lane);
  }
}

constexpr int kBw = 16;  // CTA backward panel width (register budget)

/// Backward substitution of one panel [p0, p0+pw) (rows below final in ws).
template <int PW>
__device__ __forceinline__ void warp_bwd_panel(const double* __restrict__ V, const int* __restrict__ sl, int m, int p0,
                                               int pw, double* ws, int lane) {
  int cb[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) cb[j] = j < pw ? (int)(col_off(p0 + j, m) - (p0 + j) - 1) : 0;
  double acc[PW];
#pragma unroll
  for (int j = 0; j < PW; ++j) acc[j] = 0.0;
  for (int r = p0 + pw + lane; r < m; r += 32) {
    const double xr = ws[sl[r]];
#pragma unroll
    for (int j = 0; j < PW; ++j)
      if (j < pw) acc[j] += V[cb[j] + r] * xr;
  }
  const double t = transpose_reduce<PW>(acc, lane);
  const int li = lane % PW;
  double xi = (lane < PW && li < pw) ? ws[sl[p0 + li]] - t : 0.0;
  const long long mycb = lane < pw ? col_off(p0 + lane, m) - (p0 + lane) - 1 : 0;
  double lcol[PW];
#pragma unroll
  for (int k = 0; k < PW; ++k) lcol[k] = (k < pw && k > lane && lane < pw) ? V[mycb + p0 + k] : 0.0;
#pragma unroll
  for (int k = PW - 1; k >= 0; --k) xi -= lcol[k] * __shfl_sync(0xffffffffu, xi, k);
  if (lane < pw) ws[sl[p0 + lane]] = xi;
  __syncwarp();
}

/// Warp backward substitution of one supernode (ancestor rows final in ws).
__device__ __forceinline__ void warp_bwd_sn(const double* __restrict__ V, const int* __restrict__ sl, int nc, int m,
                                            double* ws, int lane) {
  const int np = (nc + kBw - 1) / kBw;
  for (int pi = np - 1; pi >= 0; --pi) {
    const int p0 = pi * kBw, pw = min(kBw, nc - p0);
    if (pw <= 4) warp_bwd_panel<4>(V, sl, m, p0, pw, ws, lane);
    else if (pw <= 8) warp_bwd_panel<8>(V, sl, m, p0, pw, ws, lane);
    else warp_bwd_panel<16>(V, sl, m, p0, pw, ws, lane);
  }
}

// ---------------------------------------------------------------------------
// Async staging of a warp task's packed factor values (cp.async, 16-byte
// pieces, double-buffered chunks of whole supernodes).
// ---------------------------------------------------------------------------
constexpr int kStage = 512;  // doubles per stage buffer (+2 alignment slack)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

/// Forward chunk: supernodes [k, ke) with values <= kStage (or one oversized supernode).
__device__ __forceinline__ int chunk_fwd_end(const SolveSet& S, const TypeDesc& T, int k, int kend) {
  const long long v0 = S.sn_valoff[T.sn_base + k];
  int e = k + 1;
  while (e < kend && S.sn_valoff[T.sn_base + e + 1] - v0 <= kStage) ++e;
  return e;
}
/// Backward chunk: supernodes [kb, k) ending at k.
__device__ __forceinline__ int chunk_bwd_begin(const SolveSet& S, const TypeDesc& T, int k, int kbeg) {
  const long long v1 = S.sn_valoff[T.sn_base + k];
  int b = k - 1;
  while (b > kbeg && v1 - S.sn_valoff[T.sn_base + b - 1] <= kStage) --b;
  return b;
}

/// Issue the copy of values [v0, v1) (doubles, relative to L) into buf; returns
/// the offset (0/1 double) of v0 inside buf, or -1 when the range is oversized.
__device__ __forceinline__ int stage_issue(const double* L, long long v0, long long v1, double* buf, int lane) {
  if (v1 - v0 > kStage) return -1;
  const double* g = L + v0;
  const int shift = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
  const double* ga = g - shift;
  const int n16 = (int)((v1 - v0 + shift + 1) >> 1);
  for (int i = lane; i < n16; i += 32) cp_async16(buf + 2 * i, ga + 2 * i);
  return shift;
}

/// Leaf forward sweep + diagonal scaling: one warp per (problem, task).
/// Shared memory per warp: [xp 32][workspace ws_max][2 stage buffers].
__global__ void __launch_bounds__(128, 3) k_leaf_fwd(SolveSet S, int ws_max) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * (blockDim.x >> 5) + wib;
  if (w >= S.nwork) return;
  double* xp = smem + (size_t)wib * (ws_max + 32 + 2 * (kStage + 2));
  double* ws = xp + 32;
  double* stg[2] = {ws + ws_max, ws + ws_max + kStage + 2};
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nc_task = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const int sn0 = S.task_sn0[t], sn1 = S.task_sn1[t];
  const double* L = S.L + S.prob_lval[p];
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride;
    int kc = sn0, kn = chunk_fwd_end(S, T, kc, sn1), buf = 0;
    int sh = stage_issue(L, S.sn_valoff[T.sn_base + kc], S.sn_valoff[T.sn_base + kn], stg[0], lane);
    cp_async_commit();
    {
      const int* fp = S.fold_ptr + T.fold_base;
      const int* fi = S.fold_idx + T.foldidx_base;
      const double* CBp = S.CB + S.prob_cb[p] + r * S.cb_stride;
      for (int i = lane; i < nc_task; i += kWarp) {
        double v = X[c0 + i];
        for (int q = fp[c0 + i]; q < fp[c0 + i + 1]; ++q) v += CBp[fi[q]];  // child contributions, fixed order
        ws[i] = v;
      }
    }
    for (int i = lane; i < cbl; i += kWarp) ws[nc_task + i] = 0.0;
    while (kc < sn1) {
      const int kn2 = kn < sn1 ? chunk_fwd_end(S, T, kn, sn1) : kn;
      int sh2 = 0;
      if (kn < sn1) sh2 = stage_issue(L, S.sn_valoff[T.sn_base + kn], S.sn_valoff[T.sn_base + kn2], stg[buf ^ 1], lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const long long vb = S.sn_valoff[T.sn_base + kc];
      for (int k = kc; k < kn; ++k) {
        const int sk = T.sn_base + k;
        const double* V = sh >= 0 ? stg[buf] + sh + (S.sn_valoff[sk] - vb) : L + S.sn_valoff[sk];
        warp_fwd_sn(V, S.slot + T.row_base + S.sn_rowoff[sk], S.sn_ncol[sk], S.sn_nrow[sk], ws, xp, lane);
      }
      __syncwarp();
      kc = kn, kn = kn2, sh = sh2, buf ^= 1;
    }
    cp_async_wait<0>();
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

constexpr int kTopThreads = 256;

/// CTA task workspace: task columns (smem or in place in X) and the task's
/// contribution rows (smem or in place in its CB region).
struct CtaWs {
  double* col;
  double* cb;
  int nct;
  __device__ __forceinline__ double& operator[](int s) const { return s < nct ? col[s] : cb[s - nct]; }
};

/// mode 0: forward (fold, eliminate, scale, emit contributions)
/// mode 1: root (fold, forward, scale, backward)
/// mode 2: backward (ancestors final in X)
__device__ void cta_task(const SolveSet& S, int p, int tt, int mode, int in_smem, double* smem, double (*red)[32],
                         double* xp, long long* coff) {
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + tt;
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nct = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const double* L = S.L + S.prob_lval[p];
  const int* fp = S.fold_ptr + T.fold_base;
  const int* fi = S.fold_idx + T.foldidx_base;
  const int* cbr = S.cb_rows + T.cb_base + cbo;
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride;
    double* CBp = S.CB + S.prob_cb[p] + r * S.cb_stride;
    CtaWs ws{in_smem ? smem : X + c0, in_smem ? smem + nct : CBp + cbo, nct};
    if (mode != 2) {
      for (int i = threadIdx.x; i < nct; i += blockDim.x) {
        double v = X[c0 + i];
        for (int q = fp[c0 + i]; q < fp[c0 + i + 1]; ++q) v += CBp[fi[q]];
        ws.col[i] = v;
      }
      for (int i = threadIdx.x; i < cbl; i += blockDim.x) ws.cb[i] = 0.0;
    } else {
      if (in_smem)
        for (int i = threadIdx.x; i < nct; i += blockDim.x) ws.col[i] = X[c0 + i];
      for (int i = threadIdx.x; i < cbl; i += blockDim.x) ws.cb[i] = X[cbr[i]];
    }
    __syncthreads();
    if (mode != 2) {
      for (int k = S.task_sn0[t]; k < S.task_sn1[t]; ++k) {
        const int sk = T.sn_base + k;
        const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
        const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
        const double* V = L + S.sn_valoff[sk];
        for (int p0 = 0; p0 < nc; p0 += 32) {
          const int pw = min(32, nc - p0);
          if (wid == 0) {
            double xi = lane < pw ? ws[sl[p0 + lane]] : 0.0;
            double lrow[32];
#pragma unroll
            for (int j = 0; j < 32; ++j)
              lrow[j] = (j < pw && lane > j && lane < pw) ? __ldg(V + col_off(p0 + j, m) + (p0 + lane - p0 - j - 1)) : 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j) xi -= lrow[j] * __shfl_sync(0xffffffffu, xi, j);
            if (lane < pw) ws[sl[p0 + lane]] = xi;
            xp[lane] = xi;
            coff[lane] = lane < pw ? col_off(p0 + lane, m) - (p0 + lane) - 1 : 0;
          }
          __syncthreads();
          for (int rr = p0 + pw + threadIdx.x; rr < m; rr += blockDim.x) {
            double v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = j < pw ? __ldg(V + coff[j] + rr) : 0.0;
            double acc = 0.0;
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += v[j] * xp[j];
            ws[sl[rr]] -= acc;
          }
          __syncthreads();
        }
      }
      const double* Dp = S.D + S.prob_x[p] + c0;
      for (int i = threadIdx.x; i < nct; i += blockDim.x) ws.col[i] /= Dp[i];
      __syncthreads();
    }
    if (mode != 0) {
      for (int k = S.task_sn1[t] - 1; k >= S.task_sn0[t]; --k) {
        const int sk = T.sn_base + k;
        const int nc = S.sn_ncol[sk], m = S.sn_nrow[sk];
        const int* sl = S.slot + T.row_base + S.sn_rowoff[sk];
        const double* V = L + S.sn_valoff[sk];
        const int np = (nc + kBw - 1) / kBw;
        for (int pi = np - 1; pi >= 0; --pi) {
          const int p0 = pi * kBw, pw = min(kBw, nc - p0);
          double acc[kBw];
#pragma unroll
          for (int j = 0; j < kBw; ++j) acc[j] = 0.0;
          long long cb[kBw];
#pragma unroll
          for (int j = 0; j < kBw; ++j) cb[j] = j < pw ? col_off(p0 + j, m) - (p0 + j) - 1 : 0;
          for (int rr = p0 + pw + threadIdx.x; rr < m; rr += blockDim.x) {
            const double xr = ws[sl[rr]];
#pragma unroll
            for (int j = 0; j < kBw; ++j)
              if (j < pw) acc[j] += __ldg(V + cb[j] + rr) * xr;
          }
          const double tw = transpose_reduce<kBw>(acc, lane);
          if (lane < 16) red[wid][lane] = tw;
          __syncthreads();
          if (wid == 0) {
            double tsum = 0.0;
            for (int w2 = 0; w2 < nwarp; ++w2) tsum += red[w2][lane & 15];  // fixed order
            double xi = lane < pw ? ws[sl[p0 + lane]] - tsum : 0.0;
            double lcol[kBw];
#pragma unroll
            for (int kk = 0; kk < kBw; ++kk) lcol[kk] = (kk < pw && kk > lane) ? Lval(V, m, p0 + kk, p0 + lane) : 0.0;
#pragma unroll
            for (int kk = kBw - 1; kk >= 0; --kk) xi -= lcol[kk] * __shfl_sync(0xffffffffu, xi, kk);
            if (lane < pw) ws[sl[p0 + lane]] = xi;
          }
          __syncthreads();
        }
      }
    }
    if (in_smem) {
      for (int i = threadIdx.x; i < nct; i += blockDim.x) X[c0 + i] = ws.col[i];
      if (mode == 0)
        for (int i = threadIdx.x; i < cbl; i += blockDim.x) CBp[cbo + i] = ws.cb[i];
    }
    __syncthreads();
  }
}

/// One CTA per (problem, task) of a level; mode as in cta_task.
__global__ void __launch_bounds__(kTopThreads) k_cta_level(SolveSet S, int mode, int in_smem) {
  extern __shared__ double smem[];
  __shared__ double xp[32];
  __shared__ long long coff[32];
  __shared__ double red[kTopThreads / 32][32];
  const int w = blockIdx.x;
  if (w >= S.nwork) return;
  cta_task(S, S.work_prob[w], S.work_task[w], mode, in_smem, smem, red, xp, coff);
}

/// Leaf backward sweep: one warp per (problem, task); ancestors read from X;
/// factor values staged backwards in chunks.
__global__ void __launch_bounds__(128, 3) k_leaf_bwd(SolveSet S, int ws_max) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * (blockDim.x >> 5) + wib;
  if (w >= S.nwork) return;
  double* ws = smem + (size_t)wib * (ws_max + 32 + 2 * (kStage + 2)) + 32;
  double* stg[2] = {ws + ws_max, ws + ws_max + kStage + 2};
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nc_task = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const int sn0 = S.task_sn0[t], sn1 = S.task_sn1[t];
  const int* cbr = S.cb_rows + T.cb_base + cbo;
  const double* L = S.L + S.prob_lval[p];
  for (int r = 0; r < S.nrhs; ++r) {
    double* X = S.X + S.prob_x[p] + r * S.x_stride;
    // chunk [kb, ke) processed in descending supernode order
    int ke = sn1, kb = chunk_bwd_begin(S, T, ke, sn0), buf = 0;
    int sh = stage_issue(L, S.sn_valoff[T.sn_base + kb], S.sn_valoff[T.sn_base + ke], stg[0], lane);
    cp_async_commit();
    for (int i = lane; i < nc_task; i += kWarp) ws[i] = X[c0 + i];
    for (int i = lane; i < cbl; i += kWarp) ws[nc_task + i] = X[cbr[i]];
    while (ke > sn0) {
      const int kb2 = kb > sn0 ? chunk_bwd_begin(S, T, kb, sn0) : kb;
      int sh2 = 0;
      if (kb > sn0) sh2 = stage_issue(L, S.sn_valoff[T.sn_base + kb2], S.sn_valoff[T.sn_base + kb], stg[buf ^ 1], lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const long long vb = S.sn_valoff[T.sn_base + kb];
      for (int k = ke - 1; k >= kb; --k) {
        const int sk = T.sn_base + k;
        const double* V = sh >= 0 ? stg[buf] + sh + (S.sn_valoff[sk] - vb) : L + S.sn_valoff[sk];
        warp_bwd_sn(V, S.slot + T.row_base + S.sn_rowoff[sk], S.sn_ncol[sk], S.sn_nrow[sk], ws, lane);
      }
      __syncwarp();
      ke = kb, kb = kb2, sh = sh2, buf ^= 1;
    }
    cp_async_wait<0>();
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
