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
// k_local_symv / k_local_reduce: the per-iteration apply y = sum_s Op_s x_s
// (one CTA per subdomain over the packed lower tile triangle of the symmetric
// operator, x_s gathered into shared memory), then each multiplier sums its
// (one or two) subdomain contributions in a fixed order.
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
// large root fronts (c3: 64x64-cell P2 subdomains, m ~ 1800) use 8-column
// panels so the staged panel rows fit in shared memory
constexpr int kDualPWs = 8, kDualLds = 9;
constexpr long long kDualSmemMax = 227 * 1024;
/// panel width k_dual_root uses for a root front of order m (0: too large)
__host__ __device__ inline int dual_panel_width(long long m) {
  return 8LL * m * kDualLd <= kDualSmemMax ? kDualPW : (8LL * m * kDualLds <= kDualSmemMax ? kDualPWs : 0);
}

template <int PW>
__global__ void __launch_bounds__(512) k_dual_root(DualSet S) {
  constexpr int LD = PW + 1;
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
  __shared__ double Dk[PW];
  for (int p0 = 0; p0 < nB; p0 += PW) {
    const int pw = min(PW, nB - p0);
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
    for (int e = tid; e < nr * PW; e += nth) {
      const int r = e / PW, k = e - r * PW;
      Lp[r * LD + k] = k < pw ? at(r0 + r, p0 + k) : 0.0;
    }
    if (tid < PW) Dk[tid] = tid < pw ? at(p0 + tid, p0 + tid) : 0.0;
    __syncthreads();
    // trailing update A22 -= L_p D_p L_p^T on the FP64 tensor cores: 8x8
    // output tiles of the lower triangle (I >= J), warp per tile, K = the
    // panel width in m8n8k4 steps (A fragment: L_p row lane/4, column lane%4;
    // B fragment: D_k L_p(c, k) for column lane/4; C: row lane/4, columns
    // 2 (lane%4) + {0,1}); padded panel columns are zero
    {
      const int nt8 = (nr + 7) >> 3;
      const int ntile = nt8 * (nt8 + 1) / 2;
      const int fr = lane >> 2, fk = lane & 3;
      for (int q = warp; q < ntile; q += nw) {
        int I = (int)((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
        while ((I + 1) * (I + 2) / 2 <= q) ++I;
        while (I * (I + 1) / 2 > q) --I;
        const int J = q - I * (I + 1) / 2;
        const int ra = I * 8 + fr, cb = J * 8 + fr;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int k4 = 0; k4 < PW; k4 += 4) {
          const int kk = k4 + fk;
          const double af = ra < nr ? Lp[ra * LD + kk] : 0.0;
          const double bf = cb < nr ? Dk[kk] * Lp[cb * LD + kk] : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c0), "+d"(c1)
                       : "d"(af), "d"(bf));
        }
        const int r = I * 8 + fr, cc = J * 8 + 2 * fk;
        if (r < nr) {
          if (cc < nr && r >= cc) at(r0 + r, r0 + cc) -= c0;
          if (cc + 1 < nr && r >= cc + 1) at(r0 + r, r0 + cc + 1) -= c1;
        }
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

// ---------------------------------------------------------------------------
// Symmetric packed operators: F_s and Sd_s are symmetric, so only the lower
// tile triangle is stored.  32x32 tiles (I >= J) in order k = I(I+1)/2 + J;
// inside a tile, element (row r, column c) sits at double index
// ((c/2)*32 + r)*2 + (c&1): lane r of a warp loads the double2 of columns
// (2cp, 2cp+1) of its row, 512 contiguous bytes per warp-load.  Padding rows
// and columns (>= n) are zero.  Diagonal tiles hold the full symmetric block.
// ---------------------------------------------------------------------------
constexpr int kSymT = 32;

__host__ __device__ inline long long sym_tiles(int n) {
  const long long nt = (n + kSymT - 1) / kSymT;
  return nt * (nt + 1) / 2;
}

/// pack: P_s tiles from the full row-major operator A_s (lower triangle read)
__global__ void k_pack_sym(int nsub, const int* __restrict__ nloc, const long long* __restrict__ full_off,
                           const double* __restrict__ A, const long long* __restrict__ pack_off, double* P) {
  const int s = blockIdx.y;
  if (s >= nsub) return;
  const int n = nloc[s];
  const long long total = sym_tiles(n) * kSymT * kSymT;
  const double* a = A + full_off[s];
  double* p = P + pack_off[s];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(e >> 10), w = (int)(e & 1023);
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= k) ++I;
    const int J = k - I * (I + 1) / 2;
    const int c = ((w >> 6) << 1) | (w & 1), r = (w >> 1) & 31;
    const int i = I * kSymT + r, j = J * kSymT + c;
    p[e] = (i < n && j < n) ? a[(long long)i * n + j] : 0.0;
  }
}

/// Y[loff_s + i] = sum_j Op_s[i][j] x[lam[loff_s + j]] with Op_s symmetric,
/// packed (above).  nsplit CTAs per subdomain; x_s gathered straight from the
/// multiplier vector into shared memory; warp w of CTA h takes tiles
/// w + 8 (h + nsplit m), m = 0, 1, ... and accumulates row sums (T x_J into y_I)
/// and, off the diagonal, column sums (T^T x_I into y_J) into its own shared y
/// buffer in tile order; the buffers are summed in warp order and CTA h writes
/// its partial result into plane h of Y (the planes are summed in plane order
/// by the consumer, like the K-slices of the type GEMM).  Every summation
/// order is fixed (deterministic).  A subdomain's operator is streamed by
/// nsplit SMs at once: with one CTA per subdomain (BASELINE c5: 130 unshared
/// subdomains of 0.65 MB each) the launch reached 3.3 TB/s.
__global__ void __launch_bounds__(256) k_local_symv(int nsub, const int* __restrict__ nloc,
                                                    const long long* __restrict__ loff,
                                                    const long long* __restrict__ opoff,
                                                    const double* __restrict__ Op, const int* __restrict__ lam,
                                                    const double* __restrict__ x, double* __restrict__ Y,
                                                    const int* __restrict__ list, int nsplit,
                                                    long long plane_stride) {
  if (kPdlEarly) pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const int sb = blockIdx.x / nsplit, h = blockIdx.x % nsplit;
  if (sb >= nsub) return;
  const int s = list ? list[sb] : sb;
  const int n = nloc[s], nt = (n + kSymT - 1) / kSymT, np = nt * kSymT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* xs = sm;            // np
  double* yb = sm + np;       // nw x np
  const long long lo = loff[s];
  for (int j = threadIdx.x; j < np; j += blockDim.x) xs[j] = j < n ? x[lam[lo + j]] : 0.0;
  for (int j = threadIdx.x; j < nw * np; j += blockDim.x) yb[j] = 0.0;
  __syncthreads();
  const double2* A = reinterpret_cast<const double2*>(Op + opoff[s]);
  double* my = yb + warp * np;
  const int ntile = nt * (nt + 1) / 2;
  int I = 0, J = 0, k = 0;
  for (int t = warp + nw * h; t < ntile; t += nw * nsplit) {
    while (k < t) {  // advance (I, J) to tile t
      if (++J > I) ++I, J = 0;
      ++k;
    }
    const double2* tp = A + (long long)t * (kSymT * kSymT / 2);
    double2 v[16];
#pragma unroll
    for (int cp = 0; cp < 16; ++cp) v[cp] = __ldg(tp + cp * 32 + lane);
    const double* xj = xs + J * kSymT;
    double r0 = 0.0, r1 = 0.0;
#pragma unroll
    for (int cp = 0; cp < 16; ++cp) r0 += v[cp].x * xj[2 * cp], r1 += v[cp].y * xj[2 * cp + 1];
    my[I * kSymT + lane] += r0 + r1;
    if (I != J) {
      const double xr = xs[I * kSymT + lane];
      double acc[32];
#pragma unroll
      for (int cp = 0; cp < 16; ++cp) acc[2 * cp] = v[cp].x * xr, acc[2 * cp + 1] = v[cp].y * xr;
      my[J * kSymT + lane] += transpose_reduce<32>(acc, lane);
    }
    __syncwarp();
  }
  __syncthreads();
  double* Yh = Y + h * plane_stride;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += yb[w * np + i];
    Yh[lo + i] = v;
  }
}

// ---------------------------------------------------------------------------
// Type-shared operators.  Subdomains of one type (same region, same sides on
// the outer boundary, same interface signs) are translates of each other: on
// a homogeneous material their F_s / Sd_s agree to rounding.  Setup compares
// every owned subdomain's operators with its type's first one
// (k_op_maxdiff); members within 1e-12 (relative, max norm) share it, and the
// apply over all members of a type is one dense product Y_t = Op_t X_t
// (k_type_gemm: n_t x n_t times n_t x m_t) instead of m_t GEMVs.
// ---------------------------------------------------------------------------

/// out[2p] = max_ij |A_p - A_rep(p)|, out[2p+1] = max_ij |A_rep(p)| (full row-major operators)
__global__ void k_op_maxdiff(int np, const int* __restrict__ nloc, const long long* __restrict__ off,
                             const int* __restrict__ rep, const double* __restrict__ A, double* out) {
  __shared__ double rd[32], rm[32];
  const int p = blockIdx.x;
  if (p >= np) return;
  const int n = nloc[p];
  const double* a = A + off[p];
  const double* b = A + off[rep[p]];
  double d = 0.0, m = 0.0;
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    d = fmax(d, fabs(a[e] - b[e]));
    m = fmax(m, fabs(b[e]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) rd[w] = d, rm[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) d = fmax(d, rd[i]), m = fmax(m, rm[i]);
    d = fmax(d, rd[0]), m = fmax(m, rm[0]);
    out[2 * p] = d, out[2 * p + 1] = m;
  }
}

/// xloc[k] = x[lam[k]] for every (subdomain, local multiplier) slot
__global__ void k_local_gather(long long n, const int* __restrict__ lam, const double* __restrict__ x,
                               double* __restrict__ xloc) {
  if (kPdlEarly) pdl_trigger();
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int l = k < n ? lam[k] : 0;  // before the PDL wait (the map is constant)
  pdl_wait();
  if (k < n) xloc[k] = x[l];
}

/// one CTA: rows [r0, r0+32) x member columns [c0, c0+32) of a shared type
struct __align__(16) GemmWork {
  long long aoff;   // operator offset (full n x n, row-major, leading dimension lda)
  int n, r0, c0, ncol;  // ncol: member count of the type (columns)
  int coloff;       // first member in the column list
  short ch0, ch1;   // K-slice: 16-chunks [ch0, ch1); partial written to plane `plane`
  int plane, lda;
};
#ifndef PF_GSTAGES
#define PF_GSTAGES 4
#endif
constexpr int kGM = 32, kGN = 32, kGK = 16, kGThreads = 64, kGStages = PF_GSTAGES, kGLd = 20;

__device__ __forceinline__ void cp_async16_zfill(unsigned dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

/// Y[col_loff[j] + i] = sum_k A_t[i][k] xloc[col_loff[j] + k] on the FP64
/// tensor cores (mma.sync m8n8k4): a 32x32 output tile per 64-thread CTA
/// (each warp 16 rows x 32 columns = 2 x 4 MMA tiles), K in 16-chunks through
/// a 4-stage cp.async ring (16-byte copies: operator rows padded to an even
/// leading dimension, slot ranges even; shared-memory rows of 20 doubles so
/// the fragment loads are conflict-free; out-of-range elements zero-filled).
/// K may be split into slices (planes of Y, summed by k_local_reduce in plane
/// order).  Fixed summation order (deterministic).
__global__ void __launch_bounds__(kGThreads) k_type_gemm(const GemmWork* __restrict__ work,
                                                         const double* __restrict__ A,
                                                         const long long* __restrict__ col_loff,
                                                         const double* __restrict__ xloc, double* __restrict__ Y,
                                                         long long plane_stride) {
  __shared__ __align__(16) double As[kGStages][kGM][kGLd];
  __shared__ __align__(16) double Bs[kGStages][kGN][kGLd];
  if (kPdlEarly) pdl_trigger();
  const GemmWork w = work[blockIdx.x];
  const int tid = threadIdx.x, n = w.n;
  const double* a = A + w.aoff;
  // loader: k pair kp = tid % 8 (16 bytes), rows / columns tid / 8 + 8 m (m < 4)
  const int kp = tid & 7, lr0 = tid >> 3;
  const double* ap[4];
  const double* bp[4];
  bool av[4], bv[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int r = w.r0 + lr0 + 8 * m, cc = w.c0 + lr0 + 8 * m;
    av[m] = r < n, bv[m] = cc < w.ncol;
    ap[m] = a + (long long)(av[m] ? r : 0) * w.lda;
    bp[m] = xloc + (bv[m] ? col_loff[w.coloff + cc] : 0);
  }
  const int c_beg = w.ch0, nch = w.ch1;
  // operator (A) and member-input (B) copies of chunk c; B depends on the
  // predecessor kernel (PDL), A does not
  auto issueA = [&](int c) {
    if (c < nch) {
      const int st = c % kGStages;
      const int k = c * kGK + 2 * kp;
      const int nb = k + 1 < n ? 16 : (k < n ? 8 : 0);  // bytes in range
#pragma unroll
      for (int m = 0; m < 4; ++m)
        cp_async16_zfill((unsigned)__cvta_generic_to_shared(&As[st][lr0 + 8 * m][2 * kp]), ap[m] + (nb ? k : 0),
                         av[m] ? nb : 0);
    }
  };
  auto issueB = [&](int c) {
    if (c < nch) {
      const int st = c % kGStages;
      const int k = c * kGK + 2 * kp;
      const int nb = k + 1 < n ? 16 : (k < n ? 8 : 0);
#pragma unroll
      for (int m = 0; m < 4; ++m)
        cp_async16_zfill((unsigned)__cvta_generic_to_shared(&Bs[st][lr0 + 8 * m][2 * kp]), bp[m] + (nb ? k : 0),
                         bv[m] ? nb : 0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto issue = [&](int c) {
    issueA(c);
    issueB(c);
  };
  // warp wp: rows [16 wp, 16 wp + 16) x 32 columns as 2 x 4 m8n8k4 tiles
  // (A fragment: row lane/4, k lane%4; B fragment: k lane%4, column lane/4;
  //  C: row lane/4, columns 2 (lane%4) + {0,1})
  const int lane = tid & 31, wp = tid >> 5;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // prologue: operator chunks before the PDL wait (they land in the first
  // commit group), member inputs after it
#pragma unroll
  for (int c = 0; c < kGStages - 1; ++c) issueA(c_beg + c);
  pdl_wait();
#pragma unroll
  for (int c = 0; c < kGStages - 1; ++c) issueB(c_beg + c);
  for (int c = c_beg; c < nch; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGStages - 2) : "memory");
    __syncthreads();  // chunk c landed for every thread; chunk c-1's slot is free
    issue(c + kGStages - 1);
    const int st = c % kGStages;
#pragma unroll
    for (int k4 = 0; k4 < kGK; k4 += 4) {
      const int kk = k4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[st][wp * 16 + i * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[st][j * 8 + (lane >> 2)][kk];
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
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cc = w.c0 + j * 8 + (lane & 3) * 2 + h;
      if (cc >= w.ncol) continue;
      const long long yo = col_loff[w.coloff + cc] + w.plane * plane_stride;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = w.r0 + wp * 16 + i * 8 + (lane >> 2);
        if (r < n) Y[yo + r] = acc[i][j][h];
      }
    }
}

/// Explicit back-substitution (per-step, same-type subdomains): for every
/// member j of a type, X[col_out[j] + i] = Yb[col_out[j] + i] -
/// sum_k H_t[i][k] xloc[col_in[j] + k], H_t = K_t^+ G_t^T (dim_t x n_t, row
/// major, built once by the factor sweeps), Yb = K^+ b from the interface
/// right-hand side: x_s = K_s^+ (b_s - G_s^T lambda) without a sweep.  The
/// tile machinery of k_type_gemm below (same fragment layout and cp.async
/// ring); rows bound nr, K bound nk, no K slices.
struct __align__(16) HWork {
  long long aoff;
  int nr, nk, r0, c0, ncol, coloff, lda, pad;
};
/// (k_type_gemm) Y[col_loff[j] + i] = sum_k A_t[i][k] xloc[col_loff[j] + k] on the FP64
/// tensor cores (mma.sync m8n8k4): a 32x32 output tile per 64-thread CTA
/// (each warp 16 rows x 32 columns = 2 x 4 MMA tiles), K in 16-chunks through
/// a 4-stage cp.async ring (16-byte copies: operator rows padded to an even
/// leading dimension, slot ranges even; shared-memory rows of 20 doubles so
/// the fragment loads are conflict-free; out-of-range elements zero-filled).
/// K may be split into slices (planes of Y, summed by k_local_reduce in plane
/// order).  Fixed summation order (deterministic).
__global__ void __launch_bounds__(kGThreads) k_h_gemm(const HWork* __restrict__ work,
                                                         const double* __restrict__ A,
                                                      const long long* __restrict__ col_in,
                                                      const long long* __restrict__ col_out,
                                                      const double* __restrict__ xloc, const double* Yb,
                                                      double* X) {  // Yb may alias X (in place)
  __shared__ __align__(16) double As[kGStages][kGM][kGLd];
  __shared__ __align__(16) double Bs[kGStages][kGN][kGLd];
  if (kPdlEarly) pdl_trigger();
  const HWork w = work[blockIdx.x];
  const int tid = threadIdx.x, n = w.nk;
  const double* a = A + w.aoff;
  // loader: k pair kp = tid % 8 (16 bytes), rows / columns tid / 8 + 8 m (m < 4)
  const int kp = tid & 7, lr0 = tid >> 3;
  const double* ap[4];
  const double* bp[4];
  bool av[4], bv[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int r = w.r0 + lr0 + 8 * m, cc = w.c0 + lr0 + 8 * m;
    av[m] = r < w.nr, bv[m] = cc < w.ncol;
    ap[m] = a + (long long)(av[m] ? r : 0) * w.lda;
    bp[m] = xloc + (bv[m] ? col_in[w.coloff + cc] : 0);
  }
  const int c_beg = 0, nch = (n + kGK - 1) / kGK;
  // operator (A) and member-input (B) copies of chunk c; B depends on the
  // predecessor kernel (PDL), A does not
  auto issueA = [&](int c) {
    if (c < nch) {
      const int st = c % kGStages;
      const int k = c * kGK + 2 * kp;
      const int nb = k + 1 < n ? 16 : (k < n ? 8 : 0);  // bytes in range
#pragma unroll
      for (int m = 0; m < 4; ++m)
        cp_async16_zfill((unsigned)__cvta_generic_to_shared(&As[st][lr0 + 8 * m][2 * kp]), ap[m] + (nb ? k : 0),
                         av[m] ? nb : 0);
    }
  };
  auto issueB = [&](int c) {
    if (c < nch) {
      const int st = c % kGStages;
      const int k = c * kGK + 2 * kp;
      const int nb = k + 1 < n ? 16 : (k < n ? 8 : 0);
#pragma unroll
      for (int m = 0; m < 4; ++m)
        cp_async16_zfill((unsigned)__cvta_generic_to_shared(&Bs[st][lr0 + 8 * m][2 * kp]), bp[m] + (nb ? k : 0),
                         bv[m] ? nb : 0);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto issue = [&](int c) {
    issueA(c);
    issueB(c);
  };
  // warp wp: rows [16 wp, 16 wp + 16) x 32 columns as 2 x 4 m8n8k4 tiles
  // (A fragment: row lane/4, k lane%4; B fragment: k lane%4, column lane/4;
  //  C: row lane/4, columns 2 (lane%4) + {0,1})
  const int lane = tid & 31, wp = tid >> 5;
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // prologue: operator chunks before the PDL wait (they land in the first
  // commit group), member inputs after it
#pragma unroll
  for (int c = 0; c < kGStages - 1; ++c) issueA(c_beg + c);
  pdl_wait();
#pragma unroll
  for (int c = 0; c < kGStages - 1; ++c) issueB(c_beg + c);
  for (int c = c_beg; c < nch; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGStages - 2) : "memory");
    __syncthreads();  // chunk c landed for every thread; chunk c-1's slot is free
    issue(c + kGStages - 1);
    const int st = c % kGStages;
#pragma unroll
    for (int k4 = 0; k4 < kGK; k4 += 4) {
      const int kk = k4 + (lane & 3);
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = As[st][wp * 16 + i * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[st][j * 8 + (lane >> 2)][kk];
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
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cc = w.c0 + j * 8 + (lane & 3) * 2 + h;
      if (cc >= w.ncol) continue;
      const long long yo = col_out[w.coloff + cc];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = w.r0 + wp * 16 + i * 8 + (lane >> 2);
        if (r < w.nr) X[yo + r] = Yb ? Yb[yo + r] - acc[i][j][h] : acc[i][j][h];
      }
    }
}


/// H construction: X[idx[e]] = val[e] (scatter of G_s^T e_j into the natural-order
/// right-hand side, one entry list per round)
__global__ void k_h_scatter(int n, const long long* __restrict__ idx, const double* __restrict__ val, double* T) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) T[idx[e]] = val[e];
}
/// H construction: column j of H_t from a solved subdomain segment of X
struct HCol {
  long long xoff, hoff, htoff;  // X segment; H_t offset + column j; H_t^T offset + row j
  int dim, lda, ldt, pad;
};
__global__ void k_h_extract(const HCol* __restrict__ cols, const double* __restrict__ X, double* __restrict__ H,
                            double* __restrict__ HT) {
  const HCol c = cols[blockIdx.y];
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < c.dim; r += gridDim.x * blockDim.x) {
    const double v = X[c.xoff + r];
    H[c.hoff + (long long)r * c.lda] = v;
    HT[c.htoff + r] = v;
  }
}

/// y[i] = alpha * sum over the multiplier's slots (fixed order) of Y
/// (nks K-slices of the type GEMM: Y holds nks planes of `stride` slots; the
/// planes of a slot are summed in plane order, then the slots in slot order)
__global__ void k_local_reduce(int n, const int* __restrict__ ptr, const long long* __restrict__ slot,
                               const double* __restrict__ Y, double* __restrict__ y, double alpha, int nks,
                               long long stride) {
  if (kPdlEarly) pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // slot lists are constant: loaded before the PDL wait
  const int q0 = i < n ? ptr[i] : 0, q1 = i < n ? ptr[i + 1] : 0;
  const long long s0 = q0 < q1 ? slot[q0] : 0, s1 = q0 + 1 < q1 ? slot[q0 + 1] : 0;
  pdl_wait();
  if (i >= n) return;
  double v = 0.0;
  for (int q = q0; q < q1; ++q) {
    const long long sq = q == q0 ? s0 : (q == q0 + 1 ? s1 : slot[q]);
    double u = Y[sq];
    for (int k = 1; k < nks; ++k) u += Y[sq + k * stride];
    v += u;
  }
  y[i] = alpha * v;
}

}  // namespace dev
}  // namespace pf
