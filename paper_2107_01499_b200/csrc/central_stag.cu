// central_stag.cu -- C_LP_S (uint8, +/- error feedback) at g >= 2 on a
// STAGGERED schedule (scatter_reduce_lp, collectives.cpp:91-163).
//
// The first design (collectives.cu central_kernel) computes every chunk's
// (min, max) in one pass before any code exists: that pass (400 MB at 100M)
// leaves NVLink idle, and the owner then pulls the g - 1 contributions to its
// chunk while everybody encodes, so the phase-2 NVLink transfer starts late
// and ends NVLink-bound well after the encode.  Here every rank walks its
// chunks in the order me+1, me+2, ..., me (own chunk last), one chunk per
// step, and the transfer follows the encode chunk by chunk:
//
//   pipe A (x, HBM-bound)    step 0: minmax(k0)
//                            step s: encode(k_{s-1}) || minmax(k_s)   (tiles interleaved)
//                            step g: encode(me)
//                            after every minmax: a barrier of pipe A's
//                            warps across the grid, the chunk's header to
//                            its owner
//   pipe B (NVLink, local)   landing: pull source j's codes of MY chunk as
//                            soon as j's encode of each region is signalled
//                            (per-source region counters) into a local slot
//                            -- at step s the contribution of rank me-1-s
//                            arrives, so the NVLink transfer runs under the
//                            HBM-bound steps; then the fold of my chunk from
//                            local memory (g slots, fp64 ascending rank order,
//                            one rounding) as soon as each region is complete,
//                            reducing the second (min, max) -- y2 is not
//                            stored
//   grid barrier             header 2
//   pipe A                   Q2: the fold again from the local slots (y2 is
//                            recomputed: g bytes per element instead of 8),
//                            quantize into out2 (+ epsilon), decode my own
//                            chunk of x directly, publish out2 per region
//   pipe B                   gather: pull every other owner's out2 region by
//                            region as it is published, decode into x
//
// Taken at g = 2 when every chunk is 16-element aligned (n % 32 == 0: the
// BASELINE sizes; comm.cu).  Measured at 100M: g = 2
// 0.360 ms against 0.381-0.386 for central_kernel; at g = 4 the landing and
// the fold (7 warps, fp64) finish ~55 us after the last encode and the split
// gather pulls at ~440 GB/s, 0.488 against 0.428 ms -- so g >= 3 keeps
// central_kernel (B2_STAG=<g> forces this kernel for A/B runs).  Results are
// identical to central_kernel's (the same arithmetic per element, bit-exact
// vs the reference).
#include <cuda_runtime.h>

#include "b2_host.h"
#include "collectives.cuh"
#include "fold.cuh"
#include "ring.cuh"

namespace b2 {

namespace {

constexpr float kInfS = __builtin_huge_valf();

__device__ __forceinline__ WinHdr* hdr_at(uint8_t* w) { return reinterpret_cast<WinHdr*>(w); }

// named barriers of the two split groups (0: __syncthreads, 1: all consumers)
__device__ __forceinline__ void group_sync(bool a) {
  if (a)
    asm volatile("bar.sync 2, %0;" ::"n"(32 * kSplitWarpsA) : "memory");
  else
    asm volatile("bar.sync 3, %0;" ::"n"(32 * (kConsumerWarps - kSplitWarpsA)) : "memory");
}
// (lo, hi) over the consumers of one split group; valid in all of them
__device__ __forceinline__ float2 group_minmax(bool a, int gct, float lo, float hi, float2* red) {
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  const int w = gct >> 5, l = threadIdx.x & 31;
  const int nw = a ? kSplitWarpsA : kConsumerWarps - kSplitWarpsA;
  group_sync(a);
  if (l == 0) red[w] = make_float2(lo, hi);
  group_sync(a);
  const float2 v = l < nw ? red[l] : red[0];
  return make_float2(warp_min_nan(v.x), warp_max_nan(v.y));
}
// grid barrier among the group-A consumers of every CTA
__device__ __forceinline__ void group_a_grid_sync(int gct, unsigned* ws) {
  __threadfence();
  group_sync(true);
  if (gct == 0) {
    volatile unsigned* gen = ws + 1;
    const unsigned g0 = *gen;
    if (atomicAdd(ws, 1u) == gridDim.x - 1) {
      atomicExch(ws, 0u);
      __threadfence();
      atomicAdd(ws + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  group_sync(true);
}

__device__ __forceinline__ void mm4(float& lo, float& hi, float4 v) {
  lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
  hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
}

#define B2S_TRACE(pt)                                                                          \
  do {                                                                                         \
    if (a.trace && r.ct == 0) a.trace[size_t(blockIdx.x) * kTraceSlots + (pt)] = globaltimer(); \
  } while (0)
#define B2S_TRACE_B(pt)                                                                                     \
  do {                                                                                                      \
    if (a.trace && r.ct == 32 * kSplitWarpsA) a.trace[size_t(blockIdx.x) * kTraceSlots + (pt)] = globaltimer(); \
  } while (0)

template <bool EC>
__device__ __forceinline__ void stag_body(const CentralArgs& a, Ring& r) {
  __shared__ float2 redA[32], redB[32], redAll[32];
  __shared__ U8Params s_p1[kMaxRanks];  // header params of chunk k_s (step order)
  __shared__ SrcDec s_dec[kMaxRanks];   // fold: contribution headers, ascending rank
  __shared__ int s_fast;
  __shared__ SrcDec s_dec3[kMaxRanks];  // gather: owner headers (pass order)
  __shared__ int s_fast3[kMaxRanks];
  __shared__ PassDesc s_mm[kMaxRanks];    // minmax of chunk k_s, forward
  __shared__ PassDesc s_enc[kMaxRanks];   // encode of chunk k_s, reversed (its tail is in L2)
  __shared__ PassDesc s_b[kMaxRanks + 1]; // landing of source (me-1-i), then [g-1]: the fold
  __shared__ PassDesc s_q;                // Q2: the fold again
  __shared__ PassDesc s_pp[kMaxRanks];    // gather of owner (me+1+i)'s out2
  __shared__ volatile int s_qgo;          // consumers -> producer: every CTA's phase S is complete
  const int G = gridDim.x, g = a.g, me = a.me;
  const size_t c = a.n / size_t(g);  // every chunk has c elements, 16-aligned
  const size_t mlo = size_t(me) * c;
  WinHdr* mine = hdr_at(a.win[me]);
  const unsigned long long ep = a.epoch, gmul = (unsigned long long)g * ep;
  float4* x4 = reinterpret_cast<float4*>(a.x);
  float4* dl4 = reinterpret_cast<float4*>(a.delta);
  // y2 of my chunk: recomputed in Q2 from the g local code slots at g = 2
  // (the two-term fold is two FADDs, fold.cuh sum2_exact), cached in x's own
  // chunk at g >= 3 (4 bytes written + read beat re-running the fp64 fold)
  const bool cache_y2 = a.g >= 3;
  const Rounder r1 = make_rounder(a.sr_on, a.sr_seed, me, 1), r2 = make_rounder(a.sr_on, a.sr_seed, me, 2);
  auto kstep = [&](int s) { return (me + 1 + s) % g; };  // chunk of step s; s = g-1: my own
  auto src_of = [&](int i) { return (me + g - 1 - i) % g; };  // landing pass i: source rank
  uint8_t* land = a.win[me] + a.off_land;
  uint8_t* own = a.win[me] + a.off_recv1 + size_t(me) * a.slot_stride;
  auto slot_of = [&](int j) -> const uint8_t* {  // element e of source j's codes of my chunk: base + (e - mlo)
    return (j == me ? own : land + size_t(j) * a.slot_stride) - mlo;
  };
  if (threadIdx.x == 0) {
    s_qgo = 0;
    for (int s = 0; s < g; ++s) {
      const int k = kstep(s);
      PassDesc p = PassDesc::make();
      p.s = size_t(k) * c;
      p.n = c;
      p.eb = 4;
      p.nsrc = EC ? 2 : 1;
      p.base[0] = reinterpret_cast<const uint8_t*>(a.x);
      if (EC) p.base[1] = reinterpret_cast<const uint8_t*>(a.delta);
      s_mm[s] = p;
      p.reverse = true;
      s_enc[s] = p;
    }
    for (int i = 0; i + 1 < g; ++i) {  // landing of source j = me-1-i: arrives at j's step i
      const int j = src_of(i);
      PassDesc& p = s_b[i];
      p = PassDesc::make();
      p.s = mlo;
      p.n = c;
      p.eb = 1;
      p.nsrc = 1;
      p.base[0] = a.win[j] + a.off_recv1 + size_t(me) * a.slot_stride - mlo;
      p.gate = reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_sgate);
      p.gate_mult = 1;
      p.gate_nsrc = 1;
      p.gate_src[0] = j;
      p.gate_tgt[0] = ep;
      p.gate_stride = a.sgate_stride;
      p.reverse = true;  // j encodes my chunk in reverse
    }
    PassDesc& f = s_b[g - 1];  // the fold: g local slots, each region once all g landed
    f = PassDesc::make();
    f.s = mlo;
    f.n = c;
    f.eb = 1;
    f.nsrc = g;
    for (int j = 0; j < g; ++j) f.base[j] = slot_of(j);
    f.gate = reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate);
    f.gate_mult = gmul;
    f.wait_flag = &mine->arrive1;  // every contribution's header
    f.wait_target = gmul;
    f.reverse = true;
    s_q = f;
    s_q.gate = nullptr;  // after the grid barrier every slot is complete
    s_q.wait_flag = nullptr;
    if (g >= 3) {  // the cached y2 in x's own chunk
      s_q.eb = 4;
      s_q.nsrc = 1;
      s_q.base[0] = reinterpret_cast<const uint8_t*>(a.x);
    }
    for (int i = 0; i + 1 < g; ++i) {
      const int k = (me + 1 + i) % g;
      PassDesc& p = s_pp[i];
      p = PassDesc::make();
      p.s = size_t(k) * c;
      p.n = c;
      p.eb = 1;
      p.nsrc = 1;
      p.base[0] = a.win[k] + a.off_out2 - size_t(k) * c;
      p.wait_flag = &hdr_at(a.win[k])->ready2;  // owner k's second header
      p.wait_target = ep;
      p.gate = reinterpret_cast<const unsigned long long*>(a.win[k] + a.off_qgate);
      p.gate_mult = ep;
      p.reverse = true;  // owners publish out2 in reverse region order
    }
  }
  __syncthreads();
  B2S_TRACE(kTrStart);
  const bool cons = r.ct >= 0;
  r.timed = a.trace != nullptr;

  // =============================================== phase S: steps + landing + fold
  float lo2 = kInfS, hi2 = -kInfS;  // group B: the second (min, max)
  r.split_begin();
  const int gct = r.gct, gn = r.gn;
  const bool ga = r.group_a(), gb = r.group_b();
  if (r.storer && (threadIdx.x & 31) == 0) r.signal_loop();  // pipe A's encode credits
  if (r.producer || ga) {
    for (int s = 0; s <= g; ++s) {
      PassDesc* ps = s == 0 ? &s_mm[0] : &s_enc[s - 1];
      const int np = (s == 0 || s == g) ? 1 : 2;  // step s: enc(k_{s-1}) [+ mm(k_s)]
      // the two passes of one step are consecutive in shared memory only if
      // enc(k_{s-1}) and mm(k_s) are; build the step's pair in place
      __shared__ PassDesc s_step[2];
      if (r.producer && (threadIdx.x & 31) == 0) {
        if (s == 0) {
          s_step[0] = s_mm[0];
        } else {
          s_step[0] = s_enc[s - 1];
          if (s < g) s_step[1] = s_mm[s];
        }
      }
      (void)ps;
      float clo = kInfS, chi = -kInfS;
      r.stream_at(
          s_step, np, 2 * s,
          [&](int i, const uint8_t* st, size_t e0, size_t units, int T) {
            const float4* xs = reinterpret_cast<const float4*>(st);
            const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
            if (s > 0 && i == 0) {  // encode chunk k_{s-1} into my slot, credit its owner
              const int k = kstep(s - 1);
              const U8Params p = s_p1[s - 1];
              uint32_t* dst = reinterpret_cast<uint32_t*>(a.win[me] + a.off_recv1 + size_t(k) * a.slot_stride +
                                                          (e0 - size_t(k) * c));
              r.slot_acquire();
              for (int gi = gct; gi < int(units * 4); gi += gn) {
                float4 y = xs[gi];
                if (EC) y = sub4(y, ds[gi]);
                const uint32_t q = q4r(y, p.lo, p.inv, r1, e0 + 4 * size_t(gi));
                dst[gi] = q;
                if (EC) dl4[(e0 >> 2) + gi] = sub4(y, dequant4(q, p));
              }
              const size_t region = ((e0 >> 4) - (size_t(k) * c >> 4)) / kGateUnits;
              unsigned long long* sig =
                  k == me ? reinterpret_cast<unsigned long long*>(a.win[me] + a.off_gate) + region
                          : reinterpret_cast<unsigned long long*>(a.win[k] + a.off_sgate) +
                                size_t(me) * a.sgate_stride + region;
              r.slot_commit(sig, unsigned(units));
            } else {  // minmax of chunk k_s
              for (int gi = gct; gi < int(units * 4); gi += gn) {
                float4 v = xs[gi];
                if (EC) v = sub4(v, ds[gi]);
                mm4(clo, chi, v);
              }
            }
          },
          [](int) {});
      if (ga && s < g) {  // chunk k_s's header: reduce, barrier, params, send to its owner
        const int k = kstep(s);
        const float2 m = group_minmax(true, gct, clo, chi, redA);
        if (gct == 0) a.partials[size_t(s) * G + blockIdx.x] = m;
        group_a_grid_sync(gct, a.gridbar);
        float l2 = kInfS, h2 = -kInfS;
        for (int i = gct; i < G; i += gn) {
          const float2 v = __ldcg(a.partials + size_t(s) * G + i);
          l2 = fmin_nan(l2, v.x);
          h2 = fmax_nan(h2, v.y);
        }
        const float2 mm = group_minmax(true, gct, l2, h2, redA);
        if (gct == 0) {
          s_p1[s] = u8_params(mm.x, mm.y);
          if (blockIdx.x == 0) {
            hdr_at(a.win[k])->hdr1[me] = mm;
            if (!(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
            __threadfence_system();
            red_relaxed_sys_add(&hdr_at(a.win[k])->arrive1, 1ull);
          }
        }
        group_sync(true);
        if (s == 0) B2S_TRACE(kTrP1FirstA);
      }
    }
    if (ga) {  // marker: the signaller confirms everything and stops
      r.slot_acquire();
      r.slot_commit(nullptr, 0u, true);
    }
    B2S_TRACE(kTrP1Done);
  } else if (r.producer2 || gb) {
    auto load_dec = [&]() {  // contribution headers -> smem (producer2 lane)
      int fast = 1;
      for (int j = 0; j < g; ++j) {
        const float2 h = __ldcg(&mine->hdr1[j]);
        const U8Params q = u8_params(h.x, h.y);
        s_dec[j] = SrcDec{q.lo, q.step, q.c23};
        if (!(q.fastdec && fold_fast_ok(q.lo, q.step))) fast = 0;
      }
      s_fast = fast;
    };
    unsigned long long* fgate = reinterpret_cast<unsigned long long*>(a.win[me] + a.off_gate);
    r.stream_at(
        s_b, g, 2 * (g + 1),
        [&](int i, const uint8_t* st, size_t e0, size_t units, int T) {
          if (i + 1 < g) {  // landing: copy source src_of(i)'s codes of this region to its local slot
            const int j = src_of(i);
            uint4* dst = reinterpret_cast<uint4*>(land + size_t(j) * a.slot_stride + (e0 - mlo));
            const uint4* src = reinterpret_cast<const uint4*>(st);
            for (int k = gct; k < int(units); k += gn) dst[k] = src[k];
            fence_proxy_async();  // the fold reads the slot with TMA
            group_sync(false);
            if (gct == 0) {
              __threadfence();
              atomicAdd(fgate + ((e0 >> 4) - (mlo >> 4)) / kGateUnits, (unsigned long long)units);
            }
          } else {  // the fold: second (min, max) only, y2 is recomputed in Q2
            const bool fast = s_fast != 0;
            const int ng = int(units * 4);
            for (int gi = gct; gi < ng; gi += 2 * gn) {
              const int g1 = gi + gn;
              const bool has1 = g1 < ng;
              float4 y0, y1;
              fold2<kU8>(g, fast, st, gi, has1 ? g1 : gi, T, s_dec, 1.0, y0, y1);
              if (EC) y0 = sub4(y0, reinterpret_cast<const float4*>(a.eps)[((e0 - mlo) >> 2) + gi]);
              mm4(lo2, hi2, y0);
              if (cache_y2) x4[(e0 >> 2) + gi] = y0;  // x's own chunk was consumed by my encode
              if (has1) {
                if (EC) y1 = sub4(y1, reinterpret_cast<const float4*>(a.eps)[((e0 - mlo) >> 2) + g1]);
                mm4(lo2, hi2, y1);
                if (cache_y2) x4[(e0 >> 2) + g1] = y1;
              }
            }
          }
        },
        [&](int i) {
          if (i == g - 1) load_dec();
        });
    fence_proxy_async();  // the cached y2 is read by Q2's TMA
    B2S_TRACE_B(kTrP2Ready);
  }
  r.split_end();
  r.npass = 2 * (g + 1) + g;  // pass ids used so far (the tile counters finish() resets)
  if (a.trace) {
    unsigned long long* tw = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrWait;
    if (r.producer && threadIdx.x == 0) tw[2] = r.wt[1];
    if (r.producer2 && threadIdx.x == kProducer2) tw[1] = r.wt[0];
    if (r.ct == 32 * kSplitWarpsA) tw[5] = r.wt[2];
    if (r.ct == 0) tw[4] = r.wt[2];
  }
  r.timed = false;

  // =============================================== second header
  U8Params p2{};
  if (cons) {
    const float2 m = consumer_minmax(lo2, hi2, redAll);
    if (r.ct == 0) a.partials[size_t(kMaxRanks) * G + blockIdx.x] = m;
    consumer_grid_sync(a.gridbar);
    float l2 = kInfS, h2 = -kInfS;
    for (int i = r.ct; i < G; i += kConsumers) {
      const float2 v = __ldcg(a.partials + size_t(kMaxRanks) * G + i);
      l2 = fmin_nan(l2, v.x);
      h2 = fmax_nan(h2, v.y);
    }
    const float2 mm = consumer_minmax(l2, h2, redAll);
    p2 = u8_params(mm.x, mm.y);
    if (blockIdx.x == 0 && r.ct == 0) {
      mine->hdr2 = mm;
      if (!(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
      __threadfence_system();
      st_relaxed_sys(&mine->ready2, ep);
    }
    if (r.ct == 0) s_qgo = 1;
  }
  B2S_TRACE(kTrP2A);

  // =============================================== Q2 || gather
  r.timed = a.trace != nullptr;
  r.split_begin();
  const int qct = r.gct, qn = r.gn;
  if (r.storer && (threadIdx.x & 31) == 0) r.signal_loop();  // Q2's publication credits
  const int pq = 2 * (g + 1) + g;
  uint8_t* out2 = a.win[me] + a.off_out2;
  if (r.producer || r.group_a()) {
    if (r.producer && (threadIdx.x & 31) == 0) {  // Q2 streams data other CTAs wrote in phase S
      while (s_qgo == 0) __nanosleep(32);
      fence_proxy_async();
    }
    r.stream_at(
        &s_q, 1, pq,
        [&](int, const uint8_t* st, size_t e0, size_t units, int T) {
          const bool fast = s_fast != 0;
          const int ng = int(units * 4);
          r.slot_acquire();
          if (cache_y2) {
            const float4* ys = reinterpret_cast<const float4*>(st);
            for (int gi = qct; gi < ng; gi += qn) {
              const size_t e = e0 + 4 * size_t(gi);
              const float4 v = ys[gi];  // y2 (- eps already applied in the fold)
              const uint32_t q = q4r(v, p2.lo, p2.inv, r2, e);
              *reinterpret_cast<uint32_t*>(out2 + (e - mlo)) = q;
              const float4 d = dequant4(q, p2);
              if (EC) reinterpret_cast<float4*>(a.eps)[(e - mlo) >> 2] = sub4(v, d);
              __stcs(x4 + (e >> 2), d);
            }
            r.slot_commit(reinterpret_cast<unsigned long long*>(a.win[me] + a.off_qgate) +
                              ((e0 >> 4) - (mlo >> 4)) / kGateUnits,
                          unsigned(units));
            return;
          }
          for (int gi = qct; gi < ng; gi += 2 * qn) {
            const int g1 = gi + qn;
            const bool has1 = g1 < ng;
            float4 y[2];
            fold2<kU8>(g, fast, st, gi, has1 ? g1 : gi, T, s_dec, 1.0, y[0], y[1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 1 && !has1) break;
              const int gg = h ? g1 : gi;
              const size_t e = e0 + 4 * size_t(gg);
              float4 v = y[h];
              if (EC) v = sub4(v, reinterpret_cast<const float4*>(a.eps)[(e - mlo) >> 2]);
              const uint32_t q = q4r(v, p2.lo, p2.inv, r2, e);
              *reinterpret_cast<uint32_t*>(out2 + (e - mlo)) = q;
              const float4 d = dequant4(q, p2);
              if (EC) reinterpret_cast<float4*>(a.eps)[(e - mlo) >> 2] = sub4(v, d);
              __stcs(x4 + (e >> 2), d);  // my own chunk of x: D2(Q2(y2))
            }
          }
          r.slot_commit(reinterpret_cast<unsigned long long*>(a.win[me] + a.off_qgate) +
                            ((e0 >> 4) - (mlo >> 4)) / kGateUnits,
                        unsigned(units));
        },
        [](int) {});
    if (r.group_a()) {
      r.slot_acquire();
      r.slot_commit(nullptr, 0u, true);
    }
    B2S_TRACE(kTrP2Done);
  } else if (r.producer2 || r.group_b()) {
    auto load_hdr = [&](int i) {
      const int k = (me + 1 + i) % g;
      const float2 h = ld_peer_f2(&hdr_at(a.win[k])->hdr2);
      const U8Params q = u8_params(h.x, h.y);
      s_dec3[i] = SrcDec{q.lo, q.step, q.c23};
      s_fast3[i] = q.fastdec;
    };
    r.stream_at(
        s_pp, g - 1, pq + 1,
        [&](int i, const uint8_t* st, size_t e0, size_t units, int) {
          const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
          const SrcDec kd = s_dec3[i];
          if (s_fast3[i]) {
            for (int gi = qct; gi < int(units * 4); gi += qn)
              __stcs(x4 + ((e0 >> 2) + gi), dequant4_fast(cs[gi], kd.lo, kd.step, kd.c23));
          } else {
            for (int gi = qct; gi < int(units * 4); gi += qn)
              __stcs(x4 + ((e0 >> 2) + gi), dequant4(cs[gi], kd.lo, kd.step));
          }
        },
        load_hdr);
    B2S_TRACE_B(kTrP3First);
  }
  r.split_end();
  r.npass = pq + g;
  if (a.trace) {
    unsigned long long* tw = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrWait;
    if (r.producer2 && threadIdx.x == kProducer2) tw[0] = r.wt[0];  // gather producer: gates
  }
  r.timed = false;
  B2S_TRACE(kTrEnd);
}

template <bool EC>
__global__ void __launch_bounds__(kRingThreads, 1) central_stag_kernel(CentralArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring r;
  r.init(smem, a.status, a.timeout_ns, a.sched);
  stag_body<EC>(a, r);
  r.finish(a.sched_end);
}

}  // namespace

// the staggered C_LP_S (uint8) launch; the caller checks the shape
// (g >= 2, n % (16 g) == 0)
int launch_central_stag(const CentralArgs& a, bool ec, cudaStream_t s, int sms) {
  const void* fn = ec ? reinterpret_cast<const void*>(central_stag_kernel<true>)
                      : reinterpret_cast<const void*>(central_stag_kernel<false>);
  B2_CUDA_TRY(ensure_ring_smem(fn));
  const int grid = sms > 0 && sms < sm_count() ? sms : sm_count();
  CentralArgs copy = a;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kRingThreads), params, kRingSmem, s));
  return B2_OK;
}

}  // namespace b2
