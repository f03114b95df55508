// pf_sweep.cuh — the batched supernodal LDL^T sweep (the F-apply and
// Dirichlet-preconditioner hot loop), one warp per (subdomain, task).
//
// A task's factor values form one 16-byte aligned stream of units
// (pf_layout.hpp: per panel a triangle, then row blocks).  The warp runs a
// producer and a consumer over the same unit sequence:
//   producer: walks the sequence ahead of the consumer and issues one TMA
//             bulk copy (cp.async.bulk, mbarrier complete_tx) per unit into a
//             shared-memory ring (contiguous placement, wrapping to the ring
//             start), plus one per supernode for its slot list (per-type
//             table, L2 resident);
//   consumer: waits on the unit's mbarrier and computes straight from shared
//             memory with base+immediate addressing —
//             forward : triangle solved with register shuffles, row blocks
//                       updated with one shared load + one DFMA per value;
//             backward: row blocks reduced into per-column partial sums,
//                       warp transpose-reduction, then the transposed triangle.
// Up to kUnits units (ring bytes permitting) are in flight per warp, so the
// factor stream stays ahead of the dependency chain of the solve.  The
// backward sweep walks the same units in reverse order.  All shared memory is
// addressed as offsets from the kernel's dynamic shared array so every access
// compiles to LDS/STS with immediate offsets.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pf_layout.hpp"

namespace pf {
namespace dev {

extern __shared__ __align__(128) unsigned char g_sm[];

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

constexpr int kRingBytes = 8192;   // per warp; >= the largest unit (kRB*kPW*8)
constexpr int kUnits = 8;          // units in flight per warp (mbarriers)
constexpr int kSweepWarps = 4;     // warps per CTA
constexpr int kSweepPad = 256;     // slack after the last warp region

/// Per-warp shared memory: ring | barriers | task meta | ws | slots.
struct SweepSmem {
  static constexpr int kBar = kRingBytes;
  static constexpr int kMeta = kBar + 8 * kUnits;      // int4 per task supernode
  static constexpr int kWs = kMeta + 16 * kMaxTaskSn;  // ws doubles
  __host__ __device__ static int bytes(int ws_max, int smax) { return kWs + 8 * ws_max + ((2 * smax + 15) & ~15); }
};

/// unit descriptor (host-built, in consumption order): byte offset | size << 32 | source << 48
enum : int { kSrcValues = 0, kSrcSlots = 1, kSrcDiag = 2 };
__host__ __device__ inline unsigned long long unit_desc(long long off, int bytes, int src) {
  return (unsigned long long)(unsigned)off | ((unsigned long long)bytes << 32) | ((unsigned long long)src << 48);
}

__device__ __forceinline__ double lds(int byte) { return *reinterpret_cast<const double*>(g_sm + byte); }
__device__ __forceinline__ int4 meta_at(int wb, int k) {
  return *reinterpret_cast<const int4*>(g_sm + wb + SweepSmem::kMeta + 16 * k);
}

/// Producer + consumer state of one warp (warp-uniform registers).  The
/// producer walks a host-built descriptor list (two 32-entry register
/// windows, the next one prefetched); the consumer derives the same unit
/// sizes from its own loop structure and mirrors the ring placement.
struct SweepRing {
  int wb;                      // per-warp region (offset in g_sm)
  unsigned sbase;              // shared address of g_sm
  const unsigned char *sv, *ss, *sd;  // sources: values stream, slot table, pivots
  const unsigned long long* list;
  int nu, li, wbase;           // list length, next list entry to issue, window base
  unsigned long long wcur, wnxt;
  int issued, cons, head, tail, chead;
  int lane;

  __device__ __forceinline__ unsigned bar(int u) const { return sbase + wb + SweepSmem::kBar + 8 * (u & (kUnits - 1)); }

  __device__ __forceinline__ void start(const unsigned long long* l, int n) {
    list = l, nu = n, li = 0, wbase = 0;
    wcur = lane < n ? __ldg(l + lane) : 0ull;
    wnxt = 32 + lane < n ? __ldg(l + 32 + lane) : 0ull;
  }
  /// issue units ahead while barriers and ring space allow
  __device__ __forceinline__ void pump() {
    while (li < nu && issued - cons < kUnits) {
      if (li - wbase >= 32) {
        wcur = wnxt, wbase += 32;
        wnxt = wbase + 32 + lane < nu ? __ldg(list + wbase + 32 + lane) : 0ull;
      }
      const unsigned long long d = __shfl_sync(0xffffffffu, wcur, li - wbase);
      const int sz = (int)((d >> 32) & 0xffffu);
      int h = head;
      if ((h & (kRingBytes - 1)) + sz > kRingBytes) h += kRingBytes - (h & (kRingBytes - 1));
      if (h + sz - tail > kRingBytes) break;
      if (lane == 0) {
        const unsigned bb = bar(issued);
        fence_proxy_async();
        mbar_expect_tx(bb, (unsigned)sz);
        const int kind = (int)(d >> 48);
        const unsigned char* from = kind == kSrcValues ? sv : kind == kSrcSlots ? ss : sd;
        bulk_g2s(sbase + wb + (h & (kRingBytes - 1)), from + (unsigned)d, (unsigned)sz, bb);
      }
      head = h + sz;
      ++issued, ++li;
    }
  }
  /// offset (in g_sm) of the consumer's next unit (sz bytes), once resident
  __device__ __forceinline__ int acquire(int sz) {
    pump();
    int h = chead;
    if ((h & (kRingBytes - 1)) + sz > kRingBytes) h += kRingBytes - (h & (kRingBytes - 1));
    chead = h + sz;
    mbar_wait(bar(cons), (unsigned)(cons / kUnits) & 1u);
    return wb + (h & (kRingBytes - 1));
  }
  __device__ __forceinline__ void release() {
    __syncwarp();
    ++cons;
    tail = chead;
  }
};

/// copy the supernode's slot list out of the ring
template <class Ring>
__device__ __forceinline__ void take_slots(Ring& R, int slo, int m) {
  const int src = R.acquire(((m + 7) & ~7) * 2);
  for (int i = R.lane; i < (m + 7) >> 3; i += 32)
    *reinterpret_cast<int4*>(g_sm + slo + 16 * i) = *reinterpret_cast<const int4*>(g_sm + src + 16 * i);
  R.release();
}

__device__ __forceinline__ int slot_at(int slo, int r) { return *reinterpret_cast<const uint16_t*>(g_sm + slo + 2 * r); }
__device__ __forceinline__ double& ws_at(int wso, int s) { return *reinterpret_cast<double*>(g_sm + wso + 8 * s); }

/// Forward elimination of one panel; PWC >= pw compile-time bound, EXACT:
/// pw == PWC.  The triangle unit holds the INVERSE of the panel's unit-lower
/// diagonal block (pf_factor.cuh), so x = Linv b is a dot product per lane
/// with no sequential dependency; the panel's own columns occupy consecutive
/// workspace slots, so b and x are broadcast through shared memory.
template <int PWC, bool EXACT, class Ring>
__device__ __forceinline__ void fwd_panel(Ring& R, int slo, int p0, int pw, int m, int wso, int lane) {
  const bool mine = lane < pw;
  const int wp = wso + 8 * slot_at(slo, p0);
  if (pw > 1) {
    const int T = R.acquire(8 * tri_pad(pw)) + 8 * (lane * (lane - 1) / 2);
    double lrow[PWC - 1];
#pragma unroll
    for (int j = 0; j < PWC - 1; ++j) lrow[j] = (lane > j && mine) ? lds(T + 8 * j) : 0.0;
    R.release();
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
    const int V = R.acquire(8 * even_up(nr * pw)) + 8 * lane;
    if (lane < nr) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (nr == kRB) {
#pragma unroll
        for (int j = 0; j < PWC; j += 4) {
          if (EXACT || j < pw) a0 += lds(V + 8 * kRB * j) * xr[j];
          if (EXACT || j + 1 < pw) a1 += lds(V + 8 * kRB * (j + 1)) * xr[j + 1];
          if (EXACT || j + 2 < pw) a2 += lds(V + 8 * kRB * (j + 2)) * xr[j + 2];
          if (EXACT || j + 3 < pw) a3 += lds(V + 8 * kRB * (j + 3)) * xr[j + 3];
        }
      } else {
        const int st = 8 * nr;
#pragma unroll
        for (int j = 0; j < PWC; j += 4) {
          if (EXACT || j < pw) a0 += lds(V + st * j) * xr[j];
          if (EXACT || j + 1 < pw) a1 += lds(V + st * (j + 1)) * xr[j + 1];
          if (EXACT || j + 2 < pw) a2 += lds(V + st * (j + 2)) * xr[j + 2];
          if (EXACT || j + 3 < pw) a3 += lds(V + st * (j + 3)) * xr[j + 3];
        }
      }
      ws_at(wso, slot_at(slo, p0 + pw + b0 + lane)) -= (a0 + a1) + (a2 + a3);
    }
    R.release();
  }
}

/// backward substitution of one panel
template <int PWC, bool EXACT, class Ring>
__device__ __forceinline__ void bwd_panel(Ring& R, int slo, int p0, int pw, int m, int wso, int lane) {
  double acc[PWC];
#pragma unroll
  for (int j = 0; j < PWC; ++j) acc[j] = 0.0;
  const int nb = m - p0 - pw;
  if (nb > 0) {
    for (int b0 = ((nb - 1) / kRB) * kRB; b0 >= 0; b0 -= kRB) {
      const int nr = min(kRB, nb - b0);
      const int V = R.acquire(8 * even_up(nr * pw)) + 8 * lane;
      if (lane < nr) {
        const double xr = ws_at(wso, slot_at(slo, p0 + pw + b0 + lane));
        if (nr == kRB) {
#pragma unroll
          for (int j = 0; j < PWC; ++j)
            if (EXACT || j < pw) acc[j] += lds(V + 8 * kRB * j) * xr;
        } else {
          const int st = 8 * nr;
#pragma unroll
          for (int j = 0; j < PWC; ++j)
            if (EXACT || j < pw) acc[j] += lds(V + st * j) * xr;
        }
      }
      R.release();
    }
  }
  const double t = transpose_reduce<PWC>(acc, lane);
  const bool mine = lane < pw;
  const int wp = wso + 8 * slot_at(slo, p0);
  if (mine) *reinterpret_cast<double*>(g_sm + wp + 8 * lane) -= t;
  if (pw > 1) {
    // x = Linv^T c: lane i needs column i of Linv and every c_k, k > i
    const int T = R.acquire(8 * tri_pad(pw)) + 8 * lane;
    double lcol[PWC];
#pragma unroll
    for (int k = 1; k < PWC; ++k) lcol[k] = (k > lane && (EXACT || k < pw)) ? lds(T + 8 * (k * (k - 1) / 2)) : 0.0;
    R.release();
    __syncwarp();
    double a[4] = {mine ? lds(wp + 8 * lane) : 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 1; k < PWC; ++k) a[k & 3] += lcol[k] * ((EXACT || k < pw) ? lds(wp + 8 * k) : 0.0);
    __syncwarp();
    if (mine) *reinterpret_cast<double*>(g_sm + wp + 8 * lane) = (a[0] + a[1]) + (a[2] + a[3]);
  }
  __syncwarp();
}

template <class Ring>
__device__ __forceinline__ void fwd_sn(Ring& R, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = 0; p0 < nc; p0 += kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) fwd_panel<kPW, true>(R, slo, p0, pw, m, wso, lane);
    else if (kPW > 16 && pw > 16) fwd_panel<kPW, false>(R, slo, p0, pw, m, wso, lane);
    else if (pw > 8) fwd_panel<(kPW < 16 ? kPW : 16), false>(R, slo, p0, pw, m, wso, lane);
    else fwd_panel<8, false>(R, slo, p0, pw, m, wso, lane);
  }
}

template <class Ring>
__device__ __forceinline__ void bwd_sn(Ring& R, int slo, int nc, int m, int wso, int lane) {
  for (int p0 = ((nc - 1) / kPW) * kPW; p0 >= 0; p0 -= kPW) {
    const int pw = min(kPW, nc - p0);
    if (pw == kPW) bwd_panel<kPW, true>(R, slo, p0, pw, m, wso, lane);
    else if (kPW > 16 && pw > 16) bwd_panel<kPW, false>(R, slo, p0, pw, m, wso, lane);
    else if (pw > 8) bwd_panel<(kPW < 16 ? kPW : 16), false>(R, slo, p0, pw, m, wso, lane);
    else bwd_panel<8, false>(R, slo, p0, pw, m, wso, lane);
  }
}

/// Consumer side of one task (one warp): gather inputs, stream the units,
/// write outputs.  MODE 0: forward (fold children, eliminate, scale by D, emit
/// contributions); 1: root (forward + scale + backward); 2: backward (ancestor
/// values final in X).  Ring::pump() starts the self-producing variant.
template <int MODE, class Ring>
__device__ __forceinline__ void sweep_task(const SolveSet& S, Ring& R, int w, int wb, int ws_max, int lane,
                                           bool self_produce) {
  const int wso = wb + SweepSmem::kWs;
  const int slo = wso + 8 * ws_max;
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int c0 = S.task_c0[t], c1 = S.task_c1[t], nct = c1 - c0;
  const int cbo = S.task_cboff[t], cbl = S.task_cblen[t];
  const int nsn = S.task_sn1[t] - S.task_sn0[t];
  const unsigned long long* ul = S.udesc + T.udesc_base;
  double* X = S.X + S.prob_x[p];
  double* CBp = S.CB + S.prob_cb[p];
  if (MODE == 3) {  // streaming probe: consume the forward units without computing
    if (self_produce) R.start(ul + S.task_uf[t], S.task_nuf[t]), R.pump();
    const unsigned long long* l = ul + S.task_uf[t];
    double acc = 0.0;
    for (int u = 0; u < S.task_nuf[t]; ++u) {
      const int sz = (int)((__ldg(l + u) >> 32) & 0xffffu);
      const int o = R.acquire(sz);
      acc += lds(o + 8 * (lane % (sz / 8)));
      R.release();
    }
    if (acc == 12345.678) X[c0] = acc;
    return;
  }
  if (MODE != 2) {
    if (self_produce) R.start(ul + S.task_uf[t], S.task_nuf[t]), R.pump();  // first units in flight
    const int* fp = S.fold_ptr + T.fold_base;
    const int* fi = S.fold_idx + T.foldidx_base;
    for (int i = lane; i < nct; i += 32) {
      double v = X[c0 + i];
      for (int q = fp[c0 + i]; q < fp[c0 + i + 1]; ++q) v += CBp[fi[q]];  // children, fixed order
      ws_at(wso, i) = v;
    }
    for (int i = lane; i < cbl; i += 32) ws_at(wso, nct + i) = 0.0;
    for (int k = 0; k < nsn; ++k) {
      const int4 mt = meta_at(wb, k);
      take_slots(R, slo, mt.y);
      fwd_sn(R, slo, mt.x, mt.y, wso, lane);
    }
    {
      // pivots of the task's columns: the last unit of the forward list
      const int sh = c0 & 1;
      const int dof = R.acquire(8 * even_up(sh + nct)) + 8 * sh;
      for (int i = lane; i < nct; i += 32) ws_at(wso, i) /= lds(dof + 8 * i);
      R.release();
    }
    if (MODE == 0)
      for (int i = lane; i < cbl; i += 32) CBp[cbo + i] = ws_at(wso, nct + i);
    __syncwarp();
  }
  if (MODE != 0) {
    if (self_produce) R.start(ul + S.task_ub[t], S.task_nub[t]), R.pump();
    if (MODE == 2) {
      const int* cbr = S.cb_rows + T.cb_base + cbo;
      for (int i = lane; i < nct; i += 32) ws_at(wso, i) = X[c0 + i];
      for (int i = lane; i < cbl; i += 32) ws_at(wso, nct + i) = X[cbr[i]];
    }
    __syncwarp();
    for (int k = nsn - 1; k >= 0; --k) {
      const int4 mt = meta_at(wb, k);
      take_slots(R, slo, mt.y);
      bwd_sn(R, slo, mt.x, mt.y, wso, lane);
    }
  }
  __syncwarp();
  for (int i = lane; i < nct; i += 32) X[c0 + i] = ws_at(wso, i);
}

/// task metadata of work item w into the warp's region
__device__ __forceinline__ void load_meta(const SolveSet& S, int w, int wb, int lane) {
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  const int sn0 = S.task_sn0[t], nsn = S.task_sn1[t] - sn0;
  for (int i = lane; i < nsn; i += 32)
    *reinterpret_cast<int4*>(g_sm + wb + SweepSmem::kMeta + 16 * i) = __ldg(S.sn_meta + T.sn_base + sn0 + i);
}

/// Self-producing sweep: every warp streams and consumes its own task.
template <int MODE>
__global__ void __launch_bounds__(32 * kSweepWarps) k_sweep(SolveSet S, int ws_max, int smax) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int w = blockIdx.x * kSweepWarps + wib;
  if (w >= S.nwork) return;
  const int wb = wib * SweepSmem::bytes(ws_max, smax);
  SweepRing R;
  R.sbase = smem_u32(g_sm), R.wb = wb, R.lane = lane;
  if (lane == 0) {
    for (int i = 0; i < kUnits; ++i) mbar_init(R.bar(i), 1);
    fence_mbar_init();
  }
  load_meta(S, w, wb, lane);
  __syncwarp();
  const int p = S.work_prob[w];
  const TypeDesc T = S.types[S.prob_type[p]];
  const int t = T.task_base + S.work_task[w];
  R.sv = reinterpret_cast<const unsigned char*>(S.L + S.prob_lval[p] + S.task_lbeg[t]);
  R.ss = reinterpret_cast<const unsigned char*>(S.slots + T.slot_base);
  R.sd = reinterpret_cast<const unsigned char*>(S.D + S.prob_x[p]);
  R.issued = R.cons = R.head = R.tail = R.chead = 0;
  sweep_task<MODE>(S, R, w, wb, ws_max, lane, true);
}

// ---------------------------------------------------------------------------
// Warp-specialised sweep: warp 0 of the CTA is the producer, warps 1..kWsCons
// consume one task each.  Producer lane c walks consumer c's descriptor list
// (staged into shared memory 64 entries at a time by bulk copies) and issues
// a unit as soon as the consumer has released ring space; the consumer only
// waits on its full barriers and publishes (consumed units, ring tail).
// ---------------------------------------------------------------------------
constexpr int kWsCons = 7;        // consumer warps per CTA
constexpr int kListChunk = 64;    // descriptors per staged list chunk

/// extra per-consumer shared memory of the warp-specialised sweep (after the
/// SweepSmem region): ctrl int2 | 2 list barriers | 2 x kListChunk descriptors
struct WsSmem {
  static constexpr int kCtrl = 0;
  static constexpr int kLBar = 16;
  static constexpr int kList = 32;
  static constexpr int kBytes = kList + 2 * 8 * kListChunk;
  __host__ __device__ static int bytes(int ws_max, int smax) { return ((SweepSmem::bytes(ws_max, smax) + 15) & ~15) + kBytes; }
};

struct ConsumerRing {
  int wb, ctrl;          // region offset; ctrl offset (cons, tail)
  unsigned sbase;
  int cons, chead, lane;
  __device__ __forceinline__ unsigned bar(int u) const { return sbase + wb + SweepSmem::kBar + 8 * (u & (kUnits - 1)); }
  __device__ __forceinline__ void start(const unsigned long long*, int) {}
  __device__ __forceinline__ void pump() {}
  __device__ __forceinline__ int acquire(int sz) {
    int h = chead;
    if ((h & (kRingBytes - 1)) + sz > kRingBytes) h += kRingBytes - (h & (kRingBytes - 1));
    chead = h + sz;
    mbar_wait(bar(cons), (unsigned)(cons / kUnits) & 1u);
    return wb + (h & (kRingBytes - 1));
  }
  __device__ __forceinline__ void release() {
    __syncwarp();
    ++cons;
    if (lane == 0) {
      __threadfence_block();
      *reinterpret_cast<volatile unsigned long long*>(g_sm + ctrl) =
          (unsigned long long)(unsigned)cons | ((unsigned long long)(unsigned)chead << 32);
    }
  }
};

template <int MODE>
__global__ void __launch_bounds__(32 * (kWsCons + 1)) k_sweep_ws(SolveSet S, int ws_max, int smax) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rb = WsSmem::bytes(ws_max, smax);
  const unsigned sbase = smem_u32(g_sm);
  if (wid == 0) {
    // ---------------- producer: lane c serves consumer warp c + 1 ----------------
    const int c = lane;
    const int w = blockIdx.x * kWsCons + c;
    const bool valid = c < kWsCons && w < S.nwork;
    const int wb = c * rb;
    const int xb = wb + ((SweepSmem::bytes(ws_max, smax) + 15) & ~15);
    if (valid) {
      for (int i = 0; i < kUnits; ++i) mbar_init(sbase + wb + SweepSmem::kBar + 8 * i, 1);
      mbar_init(sbase + xb + WsSmem::kLBar, 1), mbar_init(sbase + xb + WsSmem::kLBar + 8, 1);
      *reinterpret_cast<int2*>(g_sm + xb + WsSmem::kCtrl) = make_int2(0, 0);
      fence_mbar_init();
    }
    __syncthreads();
    if (!valid) return;
    const int p = S.work_prob[w];
    const TypeDesc T = S.types[S.prob_type[p]];
    const int t = T.task_base + S.work_task[w];
    const unsigned char* sv = reinterpret_cast<const unsigned char*>(S.L + S.prob_lval[p] + S.task_lbeg[t]);
    const unsigned char* ss = reinterpret_cast<const unsigned char*>(S.slots + T.slot_base);
    const unsigned char* sd = reinterpret_cast<const unsigned char*>(S.D + S.prob_x[p]);
    const unsigned long long* ul = S.udesc + T.udesc_base;
    int phase = MODE == 2 ? 1 : 0;
    const unsigned long long* list = ul + (phase ? S.task_ub[t] : S.task_uf[t]);
    int nu = phase ? S.task_nub[t] : S.task_nuf[t];
    int li = 0, issued = 0, head = 0, lphase = 0, lwait = 0;  // lphase: parity bits of the 2 list barriers
    auto list_issue = [&](int chunk) {  // stage descriptors [chunk*64, ...) of the current list
      const int base = chunk * kListChunk;
      if (base >= nu) return;
      const int cnt = min(kListChunk, nu - base);
      const unsigned bytes = (unsigned)(8 * ((cnt + 1) & ~1));
      const unsigned lb = sbase + xb + WsSmem::kLBar + 8 * (chunk & 1);
      fence_proxy_async();
      mbar_expect_tx(lb, bytes);
      bulk_g2s(sbase + xb + WsSmem::kList + 8 * kListChunk * (chunk & 1), list + base, bytes, lb);
    };
    list_issue(0), list_issue(1);
    const volatile unsigned long long* ctrl =
        reinterpret_cast<const volatile unsigned long long*>(g_sm + xb + WsSmem::kCtrl);
    while (true) {
      if (li == nu) {
        if (MODE == 1 && phase == 0) {
          // both staged chunks of the forward list have been waited (li == nu);
          // the backward list restarts the chunk sequence on the same buffers
          phase = 1, list = ul + S.task_ub[t], nu = S.task_nub[t], li = 0, lwait = 0;
          list_issue(0), list_issue(1);
          continue;
        }
        break;
      }
      const unsigned long long cv = *ctrl;
      const int2 ct = make_int2((int)(unsigned)cv, (int)(unsigned)(cv >> 32));
      bool progress = false;
      while (li < nu && issued - ct.x < kUnits) {
        const int slot = (li / kListChunk) & 1;
        if (li / kListChunk >= lwait) {  // entering a staged chunk (waited once)
          mbar_wait(sbase + xb + WsSmem::kLBar + 8 * slot, (lphase >> slot) & 1u);
          lphase ^= 1u << slot;
          lwait = li / kListChunk + 1;
        }
        const unsigned long long d = *reinterpret_cast<const unsigned long long*>(
            g_sm + xb + WsSmem::kList + 8 * kListChunk * slot + 8 * (li % kListChunk));
        const int sz = (int)((d >> 32) & 0xffffu);
        int h = head;
        if ((h & (kRingBytes - 1)) + sz > kRingBytes) h += kRingBytes - (h & (kRingBytes - 1));
        if (h + sz - ct.y > kRingBytes) break;
        const unsigned bb = sbase + wb + SweepSmem::kBar + 8 * (issued & (kUnits - 1));
        fence_proxy_async();
        mbar_expect_tx(bb, (unsigned)sz);
        const int kind = (int)(d >> 48);
        const unsigned char* from = kind == kSrcValues ? sv : kind == kSrcSlots ? ss : sd;
        bulk_g2s(sbase + wb + (h & (kRingBytes - 1)), from + (unsigned)d, (unsigned)sz, bb);
        head = h + sz;
        ++issued, ++li;
        progress = true;
        if (li % kListChunk == 0) list_issue(li / kListChunk + 1);  // refill the chunk just finished
      }
      if (!progress) __nanosleep(32);
    }
    return;
  }
  // ---------------- consumers ----------------
  const int c = wid - 1;
  const int w = blockIdx.x * kWsCons + c;
  const int wb = c * rb;
  const int xb = wb + ((SweepSmem::bytes(ws_max, smax) + 15) & ~15);
  if (w < S.nwork) load_meta(S, w, wb, lane);
  __syncthreads();
  if (w >= S.nwork) return;
  ConsumerRing R;
  R.wb = wb, R.ctrl = xb + WsSmem::kCtrl, R.sbase = sbase, R.cons = 0, R.chead = 0, R.lane = lane;
  sweep_task<MODE>(S, R, w, wb, ws_max, lane, false);
}

}  // namespace dev
}  // namespace pf
