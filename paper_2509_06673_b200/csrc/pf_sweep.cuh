// pf_sweep.cuh — the batched supernodal LDL^T sweep (the F-apply and
// Dirichlet-preconditioner hot loop), one warp per (subdomain, task).
//
// A task's factor values form one contiguous, 16-byte aligned byte stream
// (pf_layout.hpp: per panel a triangle unit, then row-block units).  Lane 0
// of the warp streams it into a shared-memory ring of kNs chunks of kCh
// bytes with TMA bulk copies (cp.async.bulk + mbarrier complete_tx), up to
// kNs chunks ahead of the consumer; chunks are large because the copy engine
// needs >= 2 KB per copy to reach full HBM bandwidth
// (bench_micro/bulk_bw.cu).  Whenever a chunk lands in ring slot 0 its first
// kMirror bytes are also copied behind the ring, so every unit — even one
// that wraps around the ring end — is contiguous in shared memory and is
// read with base + immediate addressing.  The slot list of the next
// supernode and the task's pivots are prefetched with cp.async.
//   forward : the triangle unit holds the inverse of the panel's unit-lower
//             diagonal block, so the panel solve is a dot product per lane;
//             row blocks are updated with one shared load + one DFMA/value;
//   backward: row blocks reduced into per-column partial sums (warp
//             transpose-reduction), then the transposed inverse triangle;
//             the same bytes are streamed in descending order.
// All shared memory is addressed as offsets from the dynamic shared array so
// every access compiles to LDS/STS with immediate offsets.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_layout.hpp"

namespace pf {
namespace dev {

extern __shared__ __align__(128) unsigned char g_sm[];

// Optional cycle accounting of the sweep (built with -DPF_SWEEP_PROF):
// per mode [total, ring waits, slot/pivot waits, task start, triangles, tasks]
__device__ unsigned long long g_sweep_prof[4][8];
#ifdef PF_SWEEP_PROF
#define PF_PROF(...) __VA_ARGS__
#else
#define PF_PROF(...)
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef PF_KCH
#define PF_KCH 4096
#endif
#ifndef PF_KNS
#define PF_KNS 2
#endif
constexpr int kCh = PF_KCH;               // bytes per bulk copy
constexpr int kNs = PF_KNS;               // chunks in the ring
constexpr int kRingB = kCh * kNs;         // ring bytes per warp
constexpr int kHalfCols = 8;              // row blocks are consumed in halves of 8 columns
constexpr int kMirror = kRB * kHalfCols * 8;  // largest piece consumed at once: mirrored behind the ring
constexpr int kSweepWarps = 1;            // warps per CTA
constexpr int kL2Ahead = 2;               // chunks prefetched into L2 beyond the ring (forward order)
constexpr int kSweepPad = 256;            // slack after the last warp region
static_assert(kMirror <= kCh, "a piece must fit in one chunk");
static_assert(kPW == 2 * kHalfCols, "row blocks are split into two column halves");

/// Per-warp shared memory: ring | mirror | barriers | meta | ws | pivots | 2 x slots.
struct SweepSmem {
  static constexpr int kBar = kRingB + kMirror;
  static constexpr int kMeta = (kBar + 8 * kNs + 15) & ~15;  // int2 per task supernode
  static constexpr int kWs = kMeta + 8 * kMaxTaskSn;   // ws doubles
  __host__ __device__ static int piv(int ws_max) { return kWs + 8 * ws_max; }
  __host__ __device__ static int slots(int ws_max) { return kWs + 16 * ws_max; }
  __host__ __device__ static int bytes(int ws_max, int smax) { return slots(ws_max) + 2 * ((2 * smax + 15) & ~15); }
};

__device__ __forceinline__ double lds(int byte) { return *reinterpret_cast<const double*>(g_sm + byte); }
/// supernode k of the task: (ncol, nrow, slot offset)
__device__ __forceinline__ int3 meta_at(int wb, int k) {
  const int2 v = *reinterpret_cast<const int2*>(g_sm + wb + SweepSmem::kMeta + 8 * k);
  return make_int3(v.x & 0xffff, (int)((unsigned)v.x >> 16), v.y);
}
__device__ __forceinline__ int slot_at(int slo, int r) { return *reinterpret_cast<const uint16_t*>(g_sm + slo + 2 * r); }
__device__ __forceinline__ double& ws_at(int wso, int s) { return *reinterpret_cast<double*>(g_sm + wso + 8 * s); }

/// Mutable ring state (registers) and its out-of-line refill paths: issuing
/// bulk copies and waiting is rare (once per chunk), so it is kept out of the
/// unrolled panel code to keep the kernel small (instruction-cache bound).
struct RingState {
  int keep, nx, wt;
  unsigned phase;
  PF_PROF(long long tw;)
};

struct RingConst {
  const unsigned char* g;  // task value stream (16-byte aligned)
  unsigned sbase;          // shared address of g_sm
  int wb, end16, lastc, lane;
  __device__ __forceinline__ unsigned bar(int s) const { return sbase + wb + SweepSmem::kBar + 8 * s; }
  template <int DIR>  // +1 forward stream, -1 backward stream
  __device__ __forceinline__ void issue(int c) const {
    if (lane == 0) {
      const int s = c % kNs, a = c * kCh, bytes = min(kCh, end16 - a);
      const int mb = s == 0 ? min(kMirror, bytes) : 0;
      const unsigned b = bar(s);
      fence_proxy_async();
      mbar_expect_tx(b, (unsigned)(bytes + mb));
      bulk_g2s(sbase + wb + s * kCh, g + a, (unsigned)bytes, b);
      if (mb) bulk_g2s(sbase + wb + kRingB, g + a, (unsigned)mb, b);
      // deepen the pipeline beyond the ring: the chunk kL2Ahead further on in
      // stream order is pulled into L2 now
      const int pa = a + DIR * kL2Ahead * kCh;
      if (kL2Ahead > 0 && pa >= 0 && pa < end16) prefetch_l2(g + pa, (unsigned)min(kCh, end16 - pa));
    }
  }
  __device__ __forceinline__ void wait(RingState& r, int c) const {
    const int s = c % kNs;
    PF_PROF(const long long t0 = clock64());
    mbar_wait(bar(s), (r.phase >> s) & 1u);
    PF_PROF(r.tw += clock64() - t0);
    r.phase ^= 1u << s;
  }
};

__device__ __noinline__ RingState ring_refill_fwd(RingState r, RingConst k, int first, int last) {
  if (first > r.keep) {  // chunks below `first` are consumed: refill their slots
    r.keep = first;
    __syncwarp();
    while (r.nx <= min(k.lastc, r.keep + kNs - 1)) k.template issue<1>(r.nx++);
  }
  while (r.wt <= last) k.wait(r, r.wt++);
  return r;
}
__device__ __noinline__ RingState ring_refill_bwd(RingState r, RingConst k, int first, int last) {
  if (last < r.keep) {
    r.keep = last;
    __syncwarp();
    while (r.nx >= max(0, r.keep - kNs + 1)) k.template issue<-1>(r.nx--);
  }
  while (r.wt >= first) k.wait(r, r.wt--);
  return r;
}

/// The task's value stream in a shared-memory chunk ring (warp-uniform state).
/// The fast path of need_*() is two compares against byte thresholds that
/// the out-of-line refill keeps current.
struct StreamRing {
  RingConst k;
  RingState r;
  int lim, rel;  // fwd: resident below lim, release when pos >= rel; bwd: resident from lim, release when end <= rel
  long long t_wait = 0;  // PF_SWEEP_PROF (not tracked in the out-of-line path)

  __device__ __forceinline__ void start_fwd() {
    r.nx = r.wt = r.keep = 0;
    while (r.nx <= min(k.lastc, kNs - 1)) k.template issue<1>(r.nx++);
    lim = 0, rel = kCh;
  }
  __device__ __forceinline__ void start_bwd() {
    r.nx = r.wt = r.keep = k.lastc;
    while (r.nx >= max(0, k.lastc - kNs + 1)) k.template issue<-1>(r.nx--);
    lim = (k.lastc + 1) * kCh, rel = k.lastc * kCh;
  }
  /// unit [pos, pos + sz) resident and contiguous; returns its g_sm offset
  __device__ __forceinline__ int need_fwd(int pos, int sz) {
    if (pos + sz > lim || pos >= rel) {
      r = ring_refill_fwd(r, k, pos / kCh, (pos + sz - 1) / kCh);
      lim = r.wt * kCh, rel = (r.keep + 1) * kCh;
    }
    return k.wb + (pos & (kRingB - 1));
  }
  __device__ __forceinline__ int need_bwd(int pos, int sz) {
    if (pos < lim || pos + sz <= rel) {
      r = ring_refill_bwd(r, k, pos / kCh, (pos + sz - 1) / kCh);
      lim = (r.wt + 1) * kCh, rel = r.keep * kCh;
    }
    return k.wb + (pos & (kRingB - 1));
  }
};
static_assert((kRingB & (kRingB - 1)) == 0, "ring size must be a power of two");

// Forward elimination of one panel; PWC >= pw compile-time bound, EXACT:
// pw == PWC.  The panel's own columns occupy consecutive workspace slots, so
// b and x are broadcast through shared memory.
template <int PWC, bool EXACT>
__device__ __forceinline__ void fwd_panel(StreamRing& R, int& pos, int slo, int p0, int pw, int m, int wso, int lane) {
  const bool mine = lane < pw;
  const int wp = wso + 8 * slot_at(slo, p0);
  if (pw > 1) {
    const int tb = 8 * tri_pad(pw);
    const int T = R.need_fwd(pos, tb) + 8 * (lane * (lane - 1) / 2);
    pos += tb;
    double lrow[PWC - 1];
#pragma unroll
    for (int j = 0; j < PWC - 1; ++j) lrow[j] = (lane > j && mine) ? lds(T + 8 * j) : 0.0;
    double a[4] = {mine ? lds(wp + 8 * lane) : 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < PWC - 1; ++j) a[j & 3] += lrow[j] * ((EXACT || j < pw) ? lds(wp + 8 * j) : 0.0);
    __syncwarp();
    if (mine) *reinterpret_cast<double*>(g_sm + wp + 8 * lane) = (a[0] + a[1]) + (a[2] + a[3]);
    __syncwarp();
  }
  double xr[PWC];
#pragma unroll
  for (int j = 0; j < PWC; ++j) xr[j] = (EXACT || j < pw) ? lds(wp + 8 * j) : 0.0;
  const int nb = m - p0 - pw;
  for (int b0 = 0; b0 < nb; b0 += kRB) {
    const int nr = min(kRB, nb - b0);
    const int ub = 8 * even_up(nr * pw);
    const int st = 8 * nr;                                // column stride (bytes)
    const int ha = pw > kHalfCols ? kHalfCols * st : ub;  // first half: columns 0..7
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    {
      const int V = R.need_fwd(pos, ha) + 8 * lane;
      if (lane < nr) {
#pragma unroll
        for (int j = 0; j < kHalfCols; j += 4) {
          if (EXACT || j < pw) a0 += lds(V + st * j) * xr[j];
          if (EXACT || j + 1 < pw) a1 += lds(V + st * (j + 1)) * xr[j + 1];
          if (EXACT || j + 2 < pw) a2 += lds(V + st * (j + 2)) * xr[j + 2];
          if (EXACT || j + 3 < pw) a3 += lds(V + st * (j + 3)) * xr[j + 3];
        }
      }
    }
    if (pw > kHalfCols) {  // second half: columns 8..pw-1
      const int V = R.need_fwd(pos + ha, ub - ha) + 8 * lane;
      if (lane < nr) {
#pragma unroll
        for (int j = kHalfCols; j < kPW; j += 4) {
          if (EXACT || j < pw) a0 += lds(V + st * (j - kHalfCols)) * xr[j];
          if (EXACT || j + 1 < pw) a1 += lds(V + st * (j + 1 - kHalfCols)) * xr[j + 1];
          if (EXACT || j + 2 < pw) a2 += lds(V + st * (j + 2 - kHalfCols)) * xr[j + 2];
          if (EXACT || j + 3 < pw) a3 += lds(V + st * (j + 3 - kHalfCols)) * xr[j + 3];
        }
      }
    }
    pos += ub;
    if (lane < nr) ws_at(wso, slot_at(slo, p0 + pw + b0 + lane)) -= (a0 + a1) + (a2 + a3);
  }
}

/// Backward substitution of one panel whose units end at stream byte `pos`
/// (pos moves down past them).
template <int PWC, bool EXACT>
__device__ __forceinline__ void bwd_panel(StreamRing& R, int& pos, int slo, int p0, int pw, int m, int wso, int lane) {
  double acc[PWC];
#pragma unroll
  for (int j = 0; j < PWC; ++j) acc[j] = 0.0;
  const int nb = m - p0 - pw;
  if (nb > 0) {
    for (int b0 = ((nb - 1) / kRB) * kRB; b0 >= 0; b0 -= kRB) {
      const int nr = min(kRB, nb - b0);
      const int ub = 8 * even_up(nr * pw);
      const int st = 8 * nr;
      const int ha = pw > kHalfCols ? kHalfCols * st : ub;
      pos -= ub;
      const double xr = lane < nr ? ws_at(wso, slot_at(slo, p0 + pw + b0 + lane)) : 0.0;
      if (pw > kHalfCols) {  // second half first (descending stream)
        const int V = R.need_bwd(pos + ha, ub - ha) + 8 * lane;
        if (lane < nr) {
#pragma unroll
          for (int j = kHalfCols; j < kPW; ++j)
            if (EXACT || j < pw) acc[j] += lds(V + st * (j - kHalfCols)) * xr;
        }
      }
      {
        const int V = R.need_bwd(pos, ha) + 8 * lane;
        if (lane < nr) {
#pragma unroll
          for (int j = 0; j < kHalfCols; ++j)
            if (EXACT || j < pw) acc[j] += lds(V + st * j) * xr;
        }
      }
    }
  }
  const double t = transpose_reduce<PWC>(acc, lane);
  const bool mine = lane < pw;
  const int wp = wso + 8 * slot_at(slo, p0);
  if (mine) *reinterpret_cast<double*>(g_sm + wp + 8 * lane) -= t;
  if (pw > 1) {
    // x = Linv^T c: lane i needs column i of Linv and every c_k, k > i
    const int tb = 8 * tri_pad(pw);
    pos -= tb;
    const int T = R.need_bwd(pos, tb) + 8 * lane;
    double lcol[PWC];
#pragma unroll
    for (int k = 1; k < PWC; ++k) lcol[k] = (k > lane && (EXACT || k < pw)) ? lds(T + 8 * (k * (k - 1) / 2)) : 0.0;
    __syncwarp();
    double a[4] = {mine ? lds(wp + 8 * lane) : 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 1; k < PWC; ++k) a[k & 3] += lcol[k] * ((EXACT || k < pw) ? lds(wp + 8 * k) : 0.0);
    __syncwarp();
    if (mine) *reinterpret_cast<double*>(g_sm + wp + 8 * lane) = (a[0] + a[1]) + (a[2] + a[3]);
  }
  __syncwarp();
}

__device__ __forceinline__ void fwd_sn(StreamRing& R, int& pos, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = 0; p0 < nc; p0 += kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) fwd_panel<kPW, true>(R, pos, slo, p0, pw, m, wso, lane);
    else fwd_panel<kPW, false>(R, pos, slo, p0, pw, m, wso, lane);
  }
}

__device__ __forceinline__ void bwd_sn(StreamRing& R, int& pos, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = ((nc - 1) / kPW) * kPW; p0 >= 0; p0 -= kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) bwd_panel<kPW, true>(R, pos, slo, p0, pw, m, wso, lane);
    else bwd_panel<kPW, false>(R, pos, slo, p0, pw, m, wso, lane);
  }
}

/// prefetch a supernode's slot list (cp.async, 16-byte pieces)
__device__ __forceinline__ void prefetch_slots(const uint16_t* table, int3 mt, unsigned dst, int lane) {
  const int n16 = (mt.y + 7) >> 3;
  for (int i = lane; i < n16; i += 32) cp_async16(dst + 16 * i, table + mt.z + 8 * i);
}

/// MODE 0: forward (fold children, eliminate, scale by D, emit contributions)
/// MODE 1: root (forward + scale + backward in one pass)
/// MODE 2: backward (ancestor values final in X)
/// MODE 3: streaming probe (forward stream consumed without arithmetic)
template <int MODE>
__global__ void __launch_bounds__(32 * kSweepWarps, 2) k_sweep(SolveSet S, int ws_max, int smax) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kSweepWarps + wib;
  if (w >= S.nwork) return;
  PF_PROF(const long long tk0 = clock64(); long long t_slot = 0, t_start = 0);
  const int wb = wib * SweepSmem::bytes(ws_max, smax);
  const int wso = wb + SweepSmem::kWs;
  const int pvo = wb + SweepSmem::piv(ws_max);
  const int slb = wb + SweepSmem::slots(ws_max);
  const int sls = (2 * smax + 15) & ~15;  // one slot buffer
  const WorkRec wr = S.work[w];
  const int c0 = wr.c0, nct = wr.nct, cbo = wr.cbo, cbl = wr.cbl, nsn = wr.nsn;
  StreamRing R;
  R.k.sbase = smem_u32(g_sm), R.k.wb = wb, R.k.lane = lane, R.r.phase = 0;
  PF_PROF(R.r.tw = 0);
  R.k.g = reinterpret_cast<const unsigned char*>(S.L + wr.lofs);
  const int end = wr.lbytes;
  R.k.end16 = (end + 15) & ~15, R.k.lastc = (R.k.end16 - 1) / kCh;
  if (lane == 0) {
    for (int i = 0; i < kNs; ++i) mbar_init(R.k.bar(i), 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (MODE != 2) R.start_fwd(); else R.start_bwd();  // first chunks in flight during the prologue
  for (int i = lane; i < nsn; i += 32)
    *reinterpret_cast<int2*>(g_sm + wb + SweepSmem::kMeta + 8 * i) = __ldg(S.sn_meta + wr.sn + i);
  __syncwarp();
  const uint16_t* table = S.slots + wr.slot_base;
  double* X = S.X + wr.xofs;
  double* CBp = S.CB + wr.cbofs;
  if (MODE == 3) {
    double acc = 0.0;
    for (int pos = 0; pos < end; pos += kMirror) {
      const int sz = min(kMirror, end - pos);
      acc += lds(R.need_fwd(pos, sz) + 8 * (lane % max(1, sz / 8)));
    }
    if (acc == 12345.678) X[c0] = acc;
    return;
  }
  if (MODE != 2) {
    // task inputs (children already folded into X by k_fold_level), pivots
    // and the first slot list: one cp.async group
    const double* Dp = S.D + wr.xofs + c0;
    for (int i = lane; i < nct; i += 32) {
      cp_async8(R.k.sbase + wso + 8 * i, X + c0 + i);
      cp_async8(R.k.sbase + pvo + 8 * i, Dp + i);
    }
    prefetch_slots(table, meta_at(wb, 0), R.k.sbase + slb, lane);
    cp_async_commit();
    for (int i = lane; i < cbl; i += 32) ws_at(wso, nct + i) = 0.0;
    int pos = 0;
    PF_PROF(t_start = clock64() - tk0);
    for (int k = 0; k < nsn; ++k) {
      if (k + 1 < nsn) prefetch_slots(table, meta_at(wb, k + 1), R.k.sbase + slb + sls * ((k + 1) & 1), lane);
      cp_async_commit();
      PF_PROF(const long long ts0 = clock64());
      cp_async_wait<1>();
      PF_PROF(t_slot += clock64() - ts0);
      __syncwarp();
      const int3 mt = meta_at(wb, k);
      fwd_sn(R, pos, slb + sls * (k & 1), mt.x, mt.y, wso, lane);
      __syncwarp();
    }
    for (int i = lane; i < nct; i += 32) ws_at(wso, i) /= lds(pvo + 8 * i);
    if (MODE == 0)
      for (int i = lane; i < cbl; i += 32) CBp[cbo + i] = ws_at(wso, nct + i);
    __syncwarp();
  }
  if (MODE == 1 || MODE == 2) {
    if (MODE == 1) R.start_bwd();
    if (MODE == 2) {
      // own values and the ancestor values (gathered into CB by k_gather_level)
      for (int i = lane; i < nct; i += 32) cp_async8(R.k.sbase + wso + 8 * i, X + c0 + i);
      for (int i = lane; i < cbl; i += 32) cp_async8(R.k.sbase + wso + 8 * (nct + i), CBp + cbo + i);
    }
    prefetch_slots(table, meta_at(wb, nsn - 1), R.k.sbase + slb, lane);
    cp_async_commit();
    int pos = end;
    PF_PROF(if (MODE == 2) t_start = clock64() - tk0);
    for (int k = nsn - 1, b = 0; k >= 0; --k, b ^= 1) {
      if (k > 0) prefetch_slots(table, meta_at(wb, k - 1), R.k.sbase + slb + sls * (b ^ 1), lane);
      cp_async_commit();
      PF_PROF(const long long ts0 = clock64());
      cp_async_wait<1>();
      PF_PROF(t_slot += clock64() - ts0);
      __syncwarp();
      const int3 mt = meta_at(wb, k);
      bwd_sn(R, pos, slb + sls * b, mt.x, mt.y, wso, lane);
      __syncwarp();
    }
  }
  cp_async_wait<0>();
  __syncwarp();
  for (int i = lane; i < nct; i += 32) X[c0 + i] = ws_at(wso, i);
  if (MODE == 1 || MODE == 2) {
    // backward: hand the final values to every descendant task that reads
    // them (the transpose of the forward fold: each CB entry has one writer),
    // so their prologues are contiguous loads
    const int* fp = S.fold_ptr + wr.fold_base;
    const int* fi = S.fold_idx + wr.foldidx_base;
    for (int i = lane; i < nct; i += 32) {
      const double v = ws_at(wso, i);
      for (int q = fp[c0 + i]; q < fp[c0 + i + 1]; ++q) CBp[fi[q]] = v;
    }
  }
#ifdef PF_SWEEP_PROF
  if (lane == 0) {
    atomicAdd(&g_sweep_prof[MODE][0], (unsigned long long)(clock64() - tk0));
    atomicAdd(&g_sweep_prof[MODE][1], (unsigned long long)R.r.tw);
    atomicAdd(&g_sweep_prof[MODE][2], (unsigned long long)t_slot);
    atomicAdd(&g_sweep_prof[MODE][3], (unsigned long long)t_start);
    atomicAdd(&g_sweep_prof[MODE][5], 1ull);
  }
#endif
}

/// Forward fold of a level: X[c] += child contributions (fixed order), one
/// warp per work item.  Runs between the sweeps of consecutive levels so a
/// task's prologue is a contiguous asynchronous load.
__global__ void k_fold_level(SolveSet S) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= S.nwork) return;
  const WorkRec wr = S.work[w];
  const int* fp = S.fold_ptr + wr.fold_base;
  const int* fi = S.fold_idx + wr.foldidx_base;
  const double* CBp = S.CB + wr.cbofs;
  double* X = S.X + wr.xofs;
  for (int i = lane; i < wr.nct; i += 32) {
    const int q0 = fp[wr.c0 + i], q1 = fp[wr.c0 + i + 1];
    if (q0 == q1) continue;
    double v = X[wr.c0 + i];
    for (int q = q0; q < q1; ++q) v += CBp[fi[q]];
    X[wr.c0 + i] = v;
  }
}

/// Backward hand-off of columns [c0, c0 + n) of a single-problem system (the
/// dense top block): CB[fold_idx[q]] = X[c] for every fold entry q of c.
__global__ void k_scatter_cols(int c0, int n, int cb_top, const int* __restrict__ fold_ptr,
                               const int* __restrict__ fold_idx, const double* __restrict__ X, double* CB) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = X[c0 + i];
  for (int q = fold_ptr[c0 + i]; q < fold_ptr[c0 + i + 1]; ++q) {
    const int f = fold_idx[q];
    if (f < cb_top) CB[f] = v;  // entries of the sparse levels only (top tasks never run)
  }
}


// ---------------------------------------------------------------------------
// Wide sweep: V same-type subdomains per warp task (SURVEY §8f rank 2 carried
// into the sweep).  When every member of a group of V subdomains reads the
// same (bitwise shared) factor copy, the task streams its factor values ONCE
// and applies each value to V right-hand sides: the L2 -> shared-memory
// traffic of the sweep, its bound, drops by V.  Vectors are interleaved,
// X[(xofs + pos) * V + v], CB[(cbofs + slot) * V + v]; the workspace holds V
// doubles per slot; pivots D stay one per column.  Every member's arithmetic
// is the scalar kernel's, operation for operation (same partial sums, same
// order), so a wide sweep returns bitwise what V scalar sweeps return.
// ---------------------------------------------------------------------------
template <int V>
struct SweepSmemW {
  static constexpr int kWs = SweepSmem::kWs;
  __host__ __device__ static int piv(int ws_max) { return kWs + 8 * V * ws_max; }
  __host__ __device__ static int slots(int ws_max) { return piv(ws_max) + 8 * ws_max; }
  __host__ __device__ static int bytes(int ws_max, int smax) { return slots(ws_max) + 2 * ((2 * smax + 15) & ~15); }
};

template <int V>
__device__ __forceinline__ void ldv(int byte, double (&d)[V]) {
  static_assert(V % 2 == 0, "wide sweep: even width");
#pragma unroll
  for (int k = 0; k < V; k += 2) {
    const double2 t = *reinterpret_cast<const double2*>(g_sm + byte + 8 * k);
    d[k] = t.x, d[k + 1] = t.y;
  }
}
template <int V>
__device__ __forceinline__ void stv(int byte, const double (&d)[V]) {
#pragma unroll
  for (int k = 0; k < V; k += 2) *reinterpret_cast<double2*>(g_sm + byte + 8 * k) = make_double2(d[k], d[k + 1]);
}

template <int PWC, bool EXACT, int V>
__device__ __forceinline__ void fwd_panel_w(StreamRing& R, int& pos, int slo, int p0, int pw, int m, int wso, int lane) {
  const bool mine = lane < pw;
  const int wp = wso + 8 * V * slot_at(slo, p0);
  if (pw > 1) {
    const int tb = 8 * tri_pad(pw);
    const int T = R.need_fwd(pos, tb) + 8 * (lane * (lane - 1) / 2);
    pos += tb;
    double lrow[PWC - 1];
#pragma unroll
    for (int j = 0; j < PWC - 1; ++j) lrow[j] = (lane > j && mine) ? lds(T + 8 * j) : 0.0;
    double a[4][V];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < V; ++v) a[q][v] = 0.0;
    if (mine) ldv<V>(wp + 8 * V * lane, a[0]);
#pragma unroll
    for (int j = 0; j < PWC - 1; ++j) {
      // operand selected first, then ONE fused multiply-add per member: the
      // scalar kernel's rounding (a product formed in both branches and added
      // afterwards would round twice)
      double xj[V];
#pragma unroll
      for (int v = 0; v < V; ++v) xj[v] = 0.0;
      if (EXACT || j < pw) ldv<V>(wp + 8 * V * j, xj);
#pragma unroll
      for (int v = 0; v < V; ++v) a[j & 3][v] = fma(lrow[j], xj[v], a[j & 3][v]);
    }
    __syncwarp();
    if (mine) {
      double t[V];
#pragma unroll
      for (int v = 0; v < V; ++v) t[v] = (a[0][v] + a[1][v]) + (a[2][v] + a[3][v]);
      stv<V>(wp + 8 * V * lane, t);
    }
    __syncwarp();
  }
  double xr[PWC][V];
#pragma unroll
  for (int j = 0; j < PWC; ++j) {
    if (EXACT || j < pw) {
      ldv<V>(wp + 8 * V * j, xr[j]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) xr[j][v] = 0.0;
    }
  }
  const int nb = m - p0 - pw;
  for (int b0 = 0; b0 < nb; b0 += kRB) {
    const int nr = min(kRB, nb - b0);
    const int ub = 8 * even_up(nr * pw);
    const int st = 8 * nr;
    const int ha = pw > kHalfCols ? kHalfCols * st : ub;
    double a[4][V];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < V; ++v) a[q][v] = 0.0;
    {
      const int U = R.need_fwd(pos, ha) + 8 * lane;
      if (lane < nr) {
#pragma unroll
        for (int j = 0; j < kHalfCols; ++j)
          if (EXACT || j < pw) {
            const double l = lds(U + st * j);
#pragma unroll
            for (int v = 0; v < V; ++v) a[j & 3][v] = fma(l, xr[j][v], a[j & 3][v]);
          }
      }
    }
    if (pw > kHalfCols) {
      const int U = R.need_fwd(pos + ha, ub - ha) + 8 * lane;
      if (lane < nr) {
#pragma unroll
        for (int j = kHalfCols; j < kPW; ++j)
          if (EXACT || j < pw) {
            const double l = lds(U + st * (j - kHalfCols));
#pragma unroll
            for (int v = 0; v < V; ++v) a[j & 3][v] = fma(l, xr[j][v], a[j & 3][v]);
          }
      }
    }
    pos += ub;
    if (lane < nr) {
      const int wsb = wso + 8 * V * slot_at(slo, p0 + pw + b0 + lane);
      double t[V];
      ldv<V>(wsb, t);
#pragma unroll
      for (int v = 0; v < V; ++v) t[v] -= (a[0][v] + a[1][v]) + (a[2][v] + a[3][v]);
      stv<V>(wsb, t);
    }
  }
}

template <int PWC, bool EXACT, int V>
__device__ __forceinline__ void bwd_panel_w(StreamRing& R, int& pos, int slo, int p0, int pw, int m, int wso, int lane) {
  double acc[V][PWC];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int j = 0; j < PWC; ++j) acc[v][j] = 0.0;
  const int nb = m - p0 - pw;
  if (nb > 0) {
    for (int b0 = ((nb - 1) / kRB) * kRB; b0 >= 0; b0 -= kRB) {
      const int nr = min(kRB, nb - b0);
      const int ub = 8 * even_up(nr * pw);
      const int st = 8 * nr;
      const int ha = pw > kHalfCols ? kHalfCols * st : ub;
      pos -= ub;
      double xr[V];
#pragma unroll
      for (int v = 0; v < V; ++v) xr[v] = 0.0;
      if (lane < nr) ldv<V>(wso + 8 * V * slot_at(slo, p0 + pw + b0 + lane), xr);
      if (pw > kHalfCols) {
        const int U = R.need_bwd(pos + ha, ub - ha) + 8 * lane;
        if (lane < nr) {
#pragma unroll
          for (int j = kHalfCols; j < kPW; ++j)
            if (EXACT || j < pw) {
              const double l = lds(U + st * (j - kHalfCols));
#pragma unroll
              for (int v = 0; v < V; ++v) acc[v][j] = fma(l, xr[v], acc[v][j]);
            }
        }
      }
      {
        const int U = R.need_bwd(pos, ha) + 8 * lane;
        if (lane < nr) {
#pragma unroll
          for (int j = 0; j < kHalfCols; ++j)
            if (EXACT || j < pw) {
              const double l = lds(U + st * j);
#pragma unroll
              for (int v = 0; v < V; ++v) acc[v][j] = fma(l, xr[v], acc[v][j]);
            }
        }
      }
    }
  }
  double t[V];
#pragma unroll
  for (int v = 0; v < V; ++v) t[v] = transpose_reduce<PWC>(acc[v], lane);
  const bool mine = lane < pw;
  const int wp = wso + 8 * V * slot_at(slo, p0);
  if (mine) {
    double c[V];
    ldv<V>(wp + 8 * V * lane, c);
#pragma unroll
    for (int v = 0; v < V; ++v) c[v] -= t[v];
    stv<V>(wp + 8 * V * lane, c);
  }
  if (pw > 1) {
    const int tb = 8 * tri_pad(pw);
    pos -= tb;
    const int T = R.need_bwd(pos, tb) + 8 * lane;
    double lcol[PWC];
#pragma unroll
    for (int k = 1; k < PWC; ++k) lcol[k] = (k > lane && (EXACT || k < pw)) ? lds(T + 8 * (k * (k - 1) / 2)) : 0.0;
    __syncwarp();
    double a[4][V];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < V; ++v) a[q][v] = 0.0;
    if (mine) ldv<V>(wp + 8 * V * lane, a[0]);
#pragma unroll
    for (int k = 1; k < PWC; ++k) {
      double xk[V];
#pragma unroll
      for (int v = 0; v < V; ++v) xk[v] = 0.0;
      if (EXACT || k < pw) ldv<V>(wp + 8 * V * k, xk);
#pragma unroll
      for (int v = 0; v < V; ++v) a[k & 3][v] = fma(lcol[k], xk[v], a[k & 3][v]);
    }
    __syncwarp();
    if (mine) {
      double c[V];
#pragma unroll
      for (int v = 0; v < V; ++v) c[v] = (a[0][v] + a[1][v]) + (a[2][v] + a[3][v]);
      stv<V>(wp + 8 * V * lane, c);
    }
  }
  __syncwarp();
}

template <int V>
__device__ __forceinline__ void fwd_sn_w(StreamRing& R, int& pos, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = 0; p0 < nc; p0 += kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) fwd_panel_w<kPW, true, V>(R, pos, slo, p0, pw, m, wso, lane);
    else fwd_panel_w<kPW, false, V>(R, pos, slo, p0, pw, m, wso, lane);
  }
}
template <int V>
__device__ __forceinline__ void bwd_sn_w(StreamRing& R, int& pos, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = ((nc - 1) / kPW) * kPW; p0 >= 0; p0 -= kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) bwd_panel_w<kPW, true, V>(R, pos, slo, p0, pw, m, wso, lane);
    else bwd_panel_w<kPW, false, V>(R, pos, slo, p0, pw, m, wso, lane);
  }
}

/// k_sweep for V interleaved right-hand sides per task (MODE 0 / 1 / 2 as above)
template <int MODE, int V>
__global__ void __launch_bounds__(32 * kSweepWarps, 1) k_sweep_w(SolveSet S, int ws_max, int smax) {
  using SM = SweepSmemW<V>;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kSweepWarps + wib;
  if (w >= S.nwork) return;
  const int wb = wib * SM::bytes(ws_max, smax);
  const int wso = wb + SM::kWs;
  const int pvo = wb + SM::piv(ws_max);
  const int slb = wb + SM::slots(ws_max);
  const int sls = (2 * smax + 15) & ~15;
  const WorkRec wr = S.work[w];
  const int c0 = wr.c0, nct = wr.nct, cbo = wr.cbo, cbl = wr.cbl, nsn = wr.nsn;
  StreamRing R;
  R.k.sbase = smem_u32(g_sm), R.k.wb = wb, R.k.lane = lane, R.r.phase = 0;
  PF_PROF(R.r.tw = 0);
  R.k.g = reinterpret_cast<const unsigned char*>(S.L + wr.lofs);
  const int end = wr.lbytes;
  R.k.end16 = (end + 15) & ~15, R.k.lastc = (R.k.end16 - 1) / kCh;
  if (lane == 0) {
    for (int i = 0; i < kNs; ++i) mbar_init(R.k.bar(i), 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (MODE != 2) R.start_fwd(); else R.start_bwd();
  for (int i = lane; i < nsn; i += 32)
    *reinterpret_cast<int2*>(g_sm + wb + SweepSmem::kMeta + 8 * i) = __ldg(S.sn_meta + wr.sn + i);
  __syncwarp();
  const uint16_t* table = S.slots + wr.slot_base;
  double* X = S.X + wr.xofs * V;
  double* CBp = S.CB + wr.cbofs * V;
  const int nv = nct * V, cv = cbl * V;
  if (MODE != 2) {
    const double* Dp = S.D + wr.xofs + c0;
    for (int i = lane; i < nv; i += 32) cp_async8(R.k.sbase + wso + 8 * i, X + (long long)c0 * V + i);
    for (int i = lane; i < nct; i += 32) cp_async8(R.k.sbase + pvo + 8 * i, Dp + i);
    prefetch_slots(table, meta_at(wb, 0), R.k.sbase + slb, lane);
    cp_async_commit();
    for (int i = lane; i < cv; i += 32) ws_at(wso, nv + i) = 0.0;
    int pos = 0;
    for (int k = 0; k < nsn; ++k) {
      if (k + 1 < nsn) prefetch_slots(table, meta_at(wb, k + 1), R.k.sbase + slb + sls * ((k + 1) & 1), lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const int3 mt = meta_at(wb, k);
      fwd_sn_w<V>(R, pos, slb + sls * (k & 1), mt.x, mt.y, wso, lane);
      __syncwarp();
    }
    for (int i = lane; i < nv; i += 32) ws_at(wso, i) /= lds(pvo + 8 * (i / V));
    if (MODE == 0)
      for (int i = lane; i < cv; i += 32) CBp[(long long)cbo * V + i] = ws_at(wso, nv + i);
    __syncwarp();
  }
  if (MODE == 1 || MODE == 2) {
    if (MODE == 1) R.start_bwd();
    if (MODE == 2) {
      for (int i = lane; i < nv; i += 32) cp_async8(R.k.sbase + wso + 8 * i, X + (long long)c0 * V + i);
      for (int i = lane; i < cv; i += 32) cp_async8(R.k.sbase + wso + 8 * (nv + i), CBp + (long long)cbo * V + i);
    }
    prefetch_slots(table, meta_at(wb, nsn - 1), R.k.sbase + slb, lane);
    cp_async_commit();
    int pos = end;
    for (int k = nsn - 1, b = 0; k >= 0; --k, b ^= 1) {
      if (k > 0) prefetch_slots(table, meta_at(wb, k - 1), R.k.sbase + slb + sls * (b ^ 1), lane);
      cp_async_commit();
      cp_async_wait<1>();
      __syncwarp();
      const int3 mt = meta_at(wb, k);
      bwd_sn_w<V>(R, pos, slb + sls * b, mt.x, mt.y, wso, lane);
      __syncwarp();
    }
  }
  cp_async_wait<0>();
  __syncwarp();
  for (int i = lane; i < nv; i += 32) X[(long long)c0 * V + i] = ws_at(wso, i);
  if (MODE == 1 || MODE == 2) {
    const int* fp = S.fold_ptr + wr.fold_base;
    const int* fi = S.fold_idx + wr.foldidx_base;
    for (int i = lane; i < nv; i += 32) {
      const double v = ws_at(wso, i);
      const int c = i / V, vv = i % V;
      for (int q = fp[c0 + c]; q < fp[c0 + c + 1]; ++q) CBp[(long long)fi[q] * V + vv] = v;
    }
  }
}

/// k_fold_level for V interleaved right-hand sides
template <int V>
__global__ void k_fold_level_w(SolveSet S) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= S.nwork) return;
  const WorkRec wr = S.work[w];
  const int* fp = S.fold_ptr + wr.fold_base;
  const int* fi = S.fold_idx + wr.foldidx_base;
  const double* CBp = S.CB + wr.cbofs * V;
  double* X = S.X + wr.xofs * V;
  for (int i = lane; i < wr.nct * V; i += 32) {
    const int c = i / V, vv = i % V;
    const int q0 = fp[wr.c0 + c], q1 = fp[wr.c0 + c + 1];
    if (q0 == q1) continue;
    double v = X[(long long)wr.c0 * V + i];
    for (int q = q0; q < q1; ++q) v += CBp[(long long)fi[q] * V + vv];
    X[(long long)wr.c0 * V + i] = v;
  }
}

/// scalar layout -> interleaved (dir 0) and back (dir 1): member p of the wide
/// system holds scalar problem p's vector at Xw[wx[p] + pos * V]
template <int V>
__global__ void k_wide_copy(int nprob, const long long* __restrict__ prob_x, const long long* __restrict__ wx,
                            const int* __restrict__ prob_n, double* Xs, double* Xw, int dir) {
  const int p = blockIdx.y;
  if (p >= nprob) return;
  const int n = prob_n[p];
  double* xs = Xs + prob_x[p];
  double* xw = Xw + wx[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (dir) xs[i] = xw[(long long)i * V];
    else xw[(long long)i * V] = xs[i];
  }
}

}  // namespace dev
}  // namespace pf
