// pf_factor.cuh — device numeric factorisation (north-star item 2): batched
// multifrontal LDL^T of every subdomain saddle K_s and interior block K_II.
//
// One CTA per (subdomain, supernode); all supernodes of one etree height are
// independent and run in one launch.  Each CTA assembles its frontal matrix
// (m x m, column-major, lower triangle) in global memory from the subdomain's
// assembled CSR values (A-scatter map) and the update matrices of its
// children (extend-add, children in fixed order -> deterministic), performs
// the partial LDL^T of its nc pivot columns (no pivoting: the constrained
// saddles are symmetric quasi-definite, SURVEY Fact 6), writes the packed
// strict-lower trapezoid of L and the pivots D, and leaves its trailing Schur
// complement in the front for the parent.
#pragma once

#include <cuda_runtime.h>

#include "pf_layout.hpp"

namespace pf {
namespace dev {

struct MfSet {
  // per supernode (concatenated over types; index sn_base[type] + k)
  const int* type_snbase;
  const int *ncol, *nrow, *col0;
  const long long *valoff, *foff, *rp_beg;
  const int *ch_beg, *ch_cnt, *as_beg, *as_cnt;
  const int *ch_idx, *relpos, *as_kidx, *as_fpos;
  // this launch: (problem, supernode) items
  int nitem;
  const int *it_prob, *it_sn;
  // per problem
  const int* prob_type;
  const long long *prob_kval, *prob_lval, *prob_x, *prob_fbase;
  const double* Kv;
  double* F;
  double* L;
  double* D;
  int* err;
  // bordered dual-operator factorisation (pf_dual.hpp): G values per problem
  // (scatter index -2-g), the root supernode per type (assembled, not
  // factored) and whether the factor is written at all
  const double* Gv = nullptr;
  const long long* prob_gval = nullptr;
  const int* type_stop = nullptr;
  int write_factor = 1;
};

constexpr int kMfPW = 16;  // panel width of the front factorisation

/// F[i][c] -= sum_{k in [p0, pe)} L[i][k] d_k L[c][k] for r0 = pe <= c <= i < m
/// (front column-major, leading dimension m; L columns scaled, d_k on the
/// diagonal): 8x8 tiles of the lower triangle, warp per tile, mma.sync
/// m8n8k4.f64 with the panel read through L1 (A: L rows, B: d_k L(c, k));
/// columns beyond pe contribute zero.  Fixed order per entry (deterministic).
__device__ __forceinline__ void mf_trailing_update(double* Fk, int m, int p0, int pe, int warp, int lane, int nw) {
  const int r0 = pe, nr = m - r0;
  if (nr <= 0) return;
  const int nt8 = (nr + 7) >> 3, ntile = nt8 * (nt8 + 1) / 2;
  const int fr = lane >> 2, fk = lane & 3;
  for (int q = warp; q < ntile; q += nw) {
    int I = (int)((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
    while ((I + 1) * (I + 2) / 2 <= q) ++I;
    while (I * (I + 1) / 2 > q) --I;
    const int J = q - I * (I + 1) / 2;
    const int ra = r0 + I * 8 + fr, cb = r0 + J * 8 + fr;
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int k4 = 0; k4 < kMfPW; k4 += 4) {
      const int k = p0 + k4 + fk;
      const bool kin = k < pe;
      const double af = (kin && ra < m) ? Fk[ra + (long long)k * m] : 0.0;
      const double bf = (kin && cb < m) ? Fk[k + (long long)k * m] * Fk[cb + (long long)k * m] : 0.0;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1)
                   : "d"(af), "d"(bf));
    }
    const int r = r0 + I * 8 + fr, c = r0 + J * 8 + 2 * fk;
    if (r < m) {
      if (c < m && r >= c) Fk[r + (long long)c * m] -= c0;
      if (c + 1 < m && r >= c + 1) Fk[r + (long long)(c + 1) * m] -= c1;
    }
  }
}

__global__ void __launch_bounds__(256) k_mf_factor(MfSet S) {
  const int it = blockIdx.x;
  if (it >= S.nitem) return;
  const int p = S.it_prob[it], k = S.it_sn[it];
  const int t = S.prob_type[p];
  const int sk = S.type_snbase[t] + k;
  const int nc = S.ncol[sk], m = S.nrow[sk];
  double* Fk = S.F + S.prob_fbase[p] + S.foff[sk];
  const long long mm = (long long)m * m;
  for (long long q = threadIdx.x; q < mm; q += blockDim.x) Fk[q] = 0.0;
  __syncthreads();
  const double* Kv = S.Kv + S.prob_kval[p];
  const double* Gv = S.Gv ? S.Gv + S.prob_gval[p] : nullptr;
  for (int q = S.as_beg[sk] + threadIdx.x; q < S.as_beg[sk] + S.as_cnt[sk]; q += blockDim.x) {
    const int kid = S.as_kidx[q];
    Fk[S.as_fpos[q]] += kid >= 0 ? Kv[kid] : kid == -1 ? 1.0 : Gv[-2 - kid];
  }
  __syncthreads();
  for (int ci = 0; ci < S.ch_cnt[sk]; ++ci) {
    const int sc = S.type_snbase[t] + S.ch_idx[S.ch_beg[sk] + ci];
    const int ncc = S.ncol[sc], mc = S.nrow[sc], u = mc - ncc;
    const double* Fc = S.F + S.prob_fbase[p] + S.foff[sc];
    const int* rp = S.relpos + S.rp_beg[sc];
    // column-wise (coalesced in the child front), lower triangle only
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int b = warp; b < u; b += nw) {
      const int rb = rp[b];
      const double* src = Fc + (long long)(ncc + b) * mc + ncc;
      double* dst = Fk + (long long)rb * m;
      for (int a = b + lane; a < u; a += 32) dst[rp[a]] += src[a];
    }
    __syncthreads();
  }
  if (S.type_stop && k == S.type_stop[t]) return;  // root front: left assembled for the dense phase
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // partial LDL^T of the nc pivot columns in panels of kMfPW: the panel's own
  // columns by rank-1 updates, then everything right of the panel -- the
  // remaining pivot columns and the update matrix for the parent -- by one
  // trailing update F22 -= L_p D_p L_p^T on the FP64 tensor cores
  for (int p0 = 0; p0 < nc; p0 += kMfPW) {
    const int pe = min(nc, p0 + kMfPW);
    for (int j = p0; j < pe; ++j) {
      const double d = Fk[j + (long long)j * m];
      if (!(d != 0.0) || !isfinite(d)) {
        if (threadIdx.x == 0) atomicExch(S.err, 1);
        return;
      }
      const double inv = 1.0 / d;
      const double* cj = Fk + (long long)j * m;
      for (int c = j + 1 + warp; c < pe; c += nw) {
        const double lc = cj[c] * inv;
        double* col = Fk + (long long)c * m;
        for (int i = c + lane; i < m; i += 32) col[i] -= cj[i] * lc;
      }
      __syncthreads();
      for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) Fk[i + (long long)j * m] *= inv;
      __syncthreads();
    }
    mf_trailing_update(Fk, m, p0, pe, warp, lane, nw);
    __syncthreads();
  }
  if (!S.write_factor) return;
  double* L = S.L + S.prob_lval[p] + S.valoff[sk];
  for (int j = 0; j < nc; ++j)
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) L[blk_off(nc, m, i, j)] = Fk[i + (long long)j * m];
  double* D = S.D + S.prob_x[p] + S.col0[sk];
  for (int j = threadIdx.x; j < nc; j += blockDim.x) D[j] = Fk[j + (long long)j * m];
  __syncthreads();
  // the sweep's triangle units hold the inverse of each panel's unit-lower
  // diagonal block: lane j forms column j of Linv by forward substitution
  const int npan = (nc + kPW - 1) / kPW;
  for (int q = warp; q < npan; q += nw) {
    const int p0 = q * kPW, pw = min(kPW, nc - p0);
    double xc[kPW];
#pragma unroll
    for (int i = 0; i < kPW; ++i) {
      double v = i == lane ? 1.0 : 0.0;
      if (i > lane && i < pw) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < kPW; ++k)
          if (k >= lane && k < i) acc += Fk[(p0 + i) + (long long)(p0 + k) * m] * xc[k];
        v = -acc;
      }
      xc[i] = v;
    }
#pragma unroll
    for (int i = 0; i < kPW; ++i)
      if (i > lane && i < pw) L[blk_off(nc, m, p0 + i, p0 + lane)] = xc[i];
  }
}

/// Seeded residual check (feti.hpp:28-36) on the device: per problem p,
/// out = (||K y - b||^2, ||b||^2) with y, b in natural order; fixed dofs are
/// identity rows with no coupling (the regularised floating saddle).
struct ResidSet {
  int nprob;
  const int *prob_type, *type_dim, *kptr, *kcol;
  const long long *prob_kval, *prob_y, *type_kptr, *type_kcol, *type_b;
  const double *Kv, *b, *y;
  const char* fix;  // per type, natural order (offset type_b)
  double* out;
};

__global__ void k_residual_norms(ResidSet R) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  if (p >= R.nprob) return;
  const int t = R.prob_type[p];
  const int n = R.type_dim[t];
  const int* rp = R.kptr + R.type_kptr[t];
  const int* cc = R.kcol + R.type_kcol[t];
  const char* fx = R.fix + R.type_b[t];
  const double* b = R.b + R.type_b[t];
  const double* yy = R.y + R.prob_y[p];
  const double* kv = R.Kv + R.prob_kval[p];
  double rn = 0.0, bn = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double r;
    if (fx[i]) {
      r = yy[i] - b[i];
    } else {
      r = -b[i];
      for (int q = rp[i]; q < rp[i + 1]; ++q)
        if (!fx[cc[q]]) r += kv[q] * yy[cc[q]];
    }
    rn += r * r, bn += b[i] * b[i];
  }
  rn = block_sum(rn, red);
  __syncthreads();
  bn = block_sum(bn, red);
  if (threadIdx.x == 0) R.out[2 * p] = rn, R.out[2 * p + 1] = bn;
}

}  // namespace dev
}  // namespace pf
