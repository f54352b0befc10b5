// collectives.cu -- fused single-launch kernels for the four synchronous
// primitives over NVLink/NVSwitch peer memory.
//
//   central_kernel<CODEC,EC>  C_LP_S (uint8 / identity, +/- error feedback) and
//                             C_FP_S (identity, no finiteness check)
//                             = scatter_reduce_lp / scatter_reduce_fp,
//                             collectives.cpp:42-163
//   decent_kernel<CODEC>      D_LP_S / D_FP_S, collectives.cpp:229-288
//
// One persistent launch per call: grid = one CTA per SM, a producer warp
// streaming tiles with cp.async.bulk (TMA) into a 5 x 32 KB shared-memory
// ring, 17 consumer warps computing from shared memory, a signaller warp and
// a second producer for split mode (ring.cuh).
//
// C_LP_S uint8 dataflow on rank `me` (g >= 2; chunk k = partition_range(N, g, k)):
//  1A   one pass over x, chunks interleaved: every chunk's (min, max) (NaN /
//       Inf propagate: the non-finite check of codec.cpp:24-27); a grid
//       barrier; CTA 0 sends owner k its header.
//  1B   split mode.  Pipe A re-streams the chunks in reverse (tails in L2)
//       and quantizes chunk k into MY window slot k, crediting owner k's
//       region counters.  Pipe B is my fold: its tiles TMA-pull the g
//       encodings of a region of my chunk from the g windows once the region
//       has landed, decode, fold in ascending rank order in fp64 (kernels.cpp
//       add_f64), round once, cache y2 in x's own chunk (already encoded) and
//       reduce the second (min, max).
//  Q2   after a grid barrier: quantize y2 into out2, publish ready2.
//  3    pull every owner's out2 with TMA (all owners at once, round-robin),
//       decode into x (own chunk from the local out2).
//  g == 1 stateless: the output is a function of the first code alone (see
//       the g == 1 branch), two passes, 12 N bytes = the algorithmic minimum.
//       With error feedback the single-term fold is exact in fp32
//       ((float)(0.0 + d) == d + 0.0f) and three passes remain.
// Identity at g >= 2: the same without 1A (pipe A copies y, pipe B folds
// straight into out2).
//
// D_* dataflow: (uint8) one (min, max) of the bucket and its header, then
// split mode: pipe A encodes (or stages) the bucket into my window's parity
// buffer, crediting every neighbour's per-source region counter; pipe B
// pulls each region of the |N| buffers once all have landed, folds in
// ascending neighbour order in fp64, multiplies by 1/|N| in fp64, rounds once.
// A parity buffer is only overwritten after every neighbour that read it two
// rounds ago acknowledged (dreads), so no rank ever clobbers data a slow
// neighbour is still reading.
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <utility>

#include "b2_host.h"
#include "collectives.cuh"
#include "fold.cuh"
#include "ring.cuh"

namespace b2 {

namespace {

constexpr float kInf = __builtin_huge_valf();

__device__ __forceinline__ void part_range(size_t n, int g, int k, size_t& lo, size_t& sz) {
  const size_t base = n / size_t(g), extra = n % size_t(g), uk = size_t(k);
  lo = uk * base + (uk < extra ? uk : extra);
  sz = base + (uk < extra ? 1 : 0);
}

__device__ __forceinline__ float2 reduce_partials(const float2* p, int G, float2* red, int ct) {
  float lo = kInf, hi = -kInf;
  for (int i = ct; i < G; i += kConsumers) {
    const float2 v = __ldcg(p + i);
    lo = fmin_nan(lo, v.x);
    hi = fmax_nan(hi, v.y);
  }
  return consumer_minmax(lo, hi, red);
}

__device__ __forceinline__ void mm_acc(float& lo, float& hi, float4 v) {
  lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
  hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
}
__device__ __forceinline__ void mm_acc1(float& lo, float& hi, float v) {
  lo = fmin_nan(lo, v);
  hi = fmax_nan(hi, v);
}
__device__ __forceinline__ bool finite4(float4 v) {
  return finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w);
}
__device__ __forceinline__ float4 add0(float4 v) {  // (float)(0.0 + (double)v), exactly
  return make_float4(__fadd_rn(v.x, 0.0f), __fadd_rn(v.y, 0.0f), __fadd_rn(v.z, 0.0f), __fadd_rn(v.w, 0.0f));
}

__device__ __forceinline__ WinHdr* hdr_of(uint8_t* w) { return reinterpret_cast<WinHdr*>(w); }

#define B2_TRACE(pt)                                                                   \
  do {                                                                                 \
    if (a.trace && ct == 0) a.trace[size_t(blockIdx.x) * kTraceSlots + (pt)] = globaltimer(); \
  } while (0)

// Per-CTA smem gate: the producer waits for it before streaming data that
// other CTAs of this grid wrote in an earlier pass (after a grid barrier).
__device__ __forceinline__ void gate_wait(volatile int* gate, int target) {
  while (*gate < target) __nanosleep(32);
  fence_proxy_async();
}

// Load a 4-element group / element of y2 = s - eps (eps is owned-length,
// indexed from the chunk start, not 16-byte aligned).
__device__ __forceinline__ float4 eps4(const float* eps, size_t e, size_t lo) {
  const float* p = eps + (e - lo);
  return make_float4(p[0], p[1], p[2], p[3]);
}
__device__ __forceinline__ void set_eps4(float* eps, size_t e, size_t lo, float4 v) {
  float* p = eps + (e - lo);
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
  p[3] = v.w;
}

// ---------------------------------------------------------------- C_* kernel
template <int CODEC, bool EC>
__device__ __forceinline__ void central_body(const CentralArgs& a, Ring& r) {
  __shared__ float2 red[32];
  __shared__ float s_lo[kMaxRanks], s_step[kMaxRanks];
  __shared__ SrcDec s_dec[kMaxRanks];
  __shared__ SrcDec s_dec3[kMaxRanks];  // phase-3 owner headers (written by the producer)
  __shared__ U8Params s_p1[kMaxRanks];   // phase-1 params of chunk pass i
  __shared__ float2 s_mm1[kMaxRanks];
  __shared__ int s_fast3[kMaxRanks];
  __shared__ int s_fast;
  __shared__ int s_flag;
  __shared__ volatile int s_gate;
  // Pass tables live in shared memory, written once by thread 0: a
  // PassDesc is 128 bytes and per-thread copies would cost local-memory
  // traffic for all 640 threads of every CTA.
  __shared__ PassDesc s_pc[kMaxRanks];      // chunk (me+1+i)%g, forward (phase 1A / identity push)
  __shared__ PassDesc s_pq[kMaxRanks + 1];  // uint8 phase 1B: the chunks reversed; [g]: my fold
  __shared__ PassDesc s_pp[kMaxRanks];      // phase 3: owner (me+1+i)%g's payload
  __shared__ PassDesc s_m[3];               // g=1: all of x, reversed, codes; g>1: [1] = y2 cache
  const int G = gridDim.x, g = a.g, me = a.me, ct = r.ct;
  const bool cons = r.ct >= 0;
  float4* x4 = reinterpret_cast<float4*>(a.x);
  float4* dl4 = reinterpret_cast<float4*>(a.delta);
  int bad = 0;
  size_t mlo, msz;
  part_range(a.n, g, me, mlo, msz);
  WinHdr* mine = hdr_of(a.win[me]);
  const size_t mbase = mlo & ~size_t(15);
  const unsigned long long gmul = (unsigned long long)g * a.epoch;
  const bool any_edges = a.n % (16 * size_t(g)) != 0;  // some chunk boundary is not 16-element aligned
  const Rounder r1 = make_rounder(CODEC == kU8 && a.sr_on, a.sr_seed, me, 1);  // the first encode
  const Rounder r2 = make_rounder(CODEC == kU8 && a.sr_on, a.sr_seed, me, 2);  // the owner's second

  auto xpass = [&](size_t lo, size_t sz) {
    PassDesc p = PassDesc::make();
    p.s = lo;
    p.n = sz;
    p.eb = 4;
    p.nsrc = EC ? 2 : 1;
    p.base[0] = reinterpret_cast<const uint8_t*>(a.x);
    if (EC) p.base[1] = reinterpret_cast<const uint8_t*>(a.delta);
    return p;
  };
  B2_TRACE(kTrP1Fenced + 7);  // kernel entry (before the pass tables are built)
  if (threadIdx.x == 0) {
    s_gate = 0;
    s_m[0] = xpass(0, a.n);
    s_m[1] = g == 1 ? s_m[0] : xpass(mlo, msz);
    s_m[1].reverse = true;
    if (g > 1) s_m[1].nsrc = 1;
    s_m[2] = s_m[0];
    s_m[2].eb = 1;
    s_m[2].nsrc = 1;
    s_m[2].base[0] = a.win[0] + a.off_recv1;  // g=1 EC: element e -> codes[e]
    const size_t cbase = a.n / size_t(g), cextra = a.n - cbase * size_t(g);
    for (int i = 0; i < g; ++i) {
      const int k = (me + 1 + i) % g;  // i == g-1: my own chunk
      const size_t lo = size_t(k) * cbase + (size_t(k) < cextra ? size_t(k) : cextra);
      const size_t sz = cbase + (size_t(k) < cextra ? 1 : 0);
      s_pc[i] = xpass(lo, sz);
      s_pq[i] = s_pc[i];
      s_pq[i].reverse = CODEC == kU8;  // re-read backwards: the tails are in L2
      PassDesc& pp = s_pp[i];
      pp = PassDesc::make();
      pp.s = lo;
      pp.n = sz;
      pp.eb = CODEC == kU8 ? 1 : 4;
      pp.nsrc = 1;
      pp.base[0] = a.win[k] + a.off_out2 - size_t(pp.eb) * (lo & ~size_t(15));
      pp.wait_flag = &hdr_of(a.win[k])->ready2;
      pp.wait_target = a.epoch;
    }
    PassDesc& pf = s_pq[g];  // my fold: the g contributions to my chunk
    pf = PassDesc::make();
    pf.s = mlo;
    pf.n = msz;
    pf.eb = CODEC == kU8 ? 1 : 4;
    pf.nsrc = g;
    // g >= 2: every rank writes its y of chunk k into ITS window (slot k) and
    // the owner pulls them; g == 1 (identity): the old push into slot j
    for (int j = 0; j < g; ++j)
      pf.base[j] = (g >= 2 ? a.win[j] + a.off_recv1 + size_t(me) * a.slot_stride
                           : a.win[me] + a.off_recv1 + size_t(j) * a.slot_stride) -
                   size_t(pf.eb) * mbase;
    if (g >= 2) {  // each tile waits for its region's g contributions
      pf.gate = reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate);
      pf.gate_mult = gmul;
    }
    if (CODEC == kU8) {
      pf.wait_flag = &mine->arrive1;  // every rank's header
      pf.wait_target = gmul;
      pf.reverse = true;
    } else if (g == 1) {
      pf.wait_flag = &mine->arrive1;  // my own push
      pf.wait_target = gmul;
    }
  }
  __syncthreads();
  B2_TRACE(kTrStart);
  // minmax pass over y = x (- delta) of [lo, lo+sz) -> partial slot
  auto minmax_pass = [&](const PassDesc& p, int slot) {
    float lo = kInf, hi = -kInf;
    r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int T) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        float4 v = xs[gi];
        if (EC) v = sub4(v, ds[gi]);
        mm_acc(lo, hi, v);
      }
    });
    r.edges(p, [&](size_t e) {
      float v = a.x[e];
      if (EC) v = __fsub_rn(v, a.delta[e]);
      mm_acc1(lo, hi, v);
    });
    if (cons) {
      const float2 mm = consumer_minmax(lo, hi, red);
      if (ct == 0) a.partials[size_t(slot) * G + blockIdx.x] = mm;
    }
  };
  auto finish_minmax = [&](int slot) -> float2 {  // consumers only
    consumer_grid_sync(a.gridbar);
    return reduce_partials(a.partials + size_t(slot) * G, G, red, ct);
  };

  if (CODEC == kU8 && g == 1 && !EC && !a.sr_on) {  // (stochastic Q1 need not emit code 255: no shortcut)
    // ------------------------------------------- single rank, stateless
    // D1(q) = lo1 + q*step1 is monotone in q and codes 0 and 255 always occur
    // (0 at the minimum element, 255 at the maximum; all 0 when degenerate),
    // so the second header is (D1(0), D1(qmax)) without a pass and the output
    // D2(Q2(D1(q1))) is a function of q1 alone: two passes, 12 N bytes.
    const PassDesc& px = s_m[0];
    minmax_pass(px, 0);
    U8Params p1{}, p2{};
    if (cons) {
      const float2 mm1 = finish_minmax(0);
      B2_TRACE(kTrP1FirstA);
      p1 = u8_params(mm1.x, mm1.y);
      const float lo2 = __fadd_rn(dequant1(uint8_t(0), p1), 0.0f);
      const float hi2 = __fadd_rn(dequant1(uint8_t(p1.degenerate ? 0 : 255), p1), 0.0f);
      p2 = u8_params(lo2, hi2);
      if (blockIdx.x == 0 && ct == 0) {
        hdr_of(a.win[0])->hdr1[0] = mm1;
        hdr_of(a.win[0])->hdr2 = make_float2(lo2, hi2);
        if (a.n && !(finite_f(mm1.x) && finite_f(mm1.y) && finite_f(lo2) && finite_f(hi2)))
          latch(a.status, kStatusNonFinite);
      }
    }
    const PassDesc& pb = s_m[1];  // reversed: the tail of x that pass A just read is still in L2
    r.run(pb, [&](const uint8_t* st, size_t e0, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        const float4 d1 = add0(dequant4(q4r(xs[gi], p1.lo, p1.inv, r1, e0 + 4 * size_t(gi)), p1));
        __stcs(x4 + ((e0 >> 2) + gi), dequant4(q4r(d1, p2.lo, p2.inv, r2, e0 + 4 * size_t(gi)), p2));
      }
    });
    r.edges(px, [&](size_t e) {
      const float d1 = __fadd_rn(dequant1(q1r(a.x[e], p1.lo, p1.inv, r1, e), p1), 0.0f);
      a.x[e] = dequant1(q1r(d1, p2.lo, p2.inv, r2, e), p2);
    });
    B2_TRACE(kTrEnd);
    return;
  }
  if (CODEC == kU8 && g == 1) {
    // ------------------------------------------------ single rank, error feedback
    const PassDesc& px = s_m[0];
    minmax_pass(px, 0);
    float2 mm1 = make_float2(0.f, 0.f);
    U8Params p1{};
    if (cons) {
      mm1 = finish_minmax(0);
      B2_TRACE(kTrP1FirstA);
      p1 = u8_params(mm1.x, mm1.y);
      if (blockIdx.x == 0 && ct == 0 && a.n && !(finite_f(mm1.x) && finite_f(mm1.y)))
        latch(a.status, kStatusNonFinite);
    }
    uint8_t* codes = a.win[0] + a.off_recv1;  // element e -> codes[e] (chunk 0 starts at 0)
    float lo2 = kInf, hi2 = -kInf;
    r.run(px, [&](const uint8_t* st, size_t e0, size_t units, int T) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        float4 y = xs[gi];
        if (EC) y = sub4(y, ds[gi]);
        const size_t e = e0 + 4 * size_t(gi);
        const uint32_t q = q4r(y, p1.lo, p1.inv, r1, e);
        *reinterpret_cast<uint32_t*>(codes + e) = q;
        const float4 d = dequant4(q, p1);
        if (EC) dl4[e >> 2] = sub4(y, d);
        float4 y2 = add0(d);
        if (EC) y2 = sub4(y2, eps4(a.eps, e, 0));
        mm_acc(lo2, hi2, y2);
      }
    });
    r.edges(px, [&](size_t e) {
      float y = a.x[e];
      if (EC) y = __fsub_rn(y, a.delta[e]);
      const uint8_t q = q1r(y, p1.lo, p1.inv, r1, e);
      codes[e] = q;
      const float d = dequant1(q, p1.lo, p1.step);
      if (EC) a.delta[e] = __fsub_rn(y, d);
      float y2 = __fadd_rn(d, 0.0f);
      if (EC) y2 = __fsub_rn(y2, a.eps[e]);
      mm_acc1(lo2, hi2, y2);
    });
    U8Params p2{};
    if (cons) {
      const float2 mm = consumer_minmax(lo2, hi2, red);
      if (ct == 0) a.partials[size_t(1) * G + blockIdx.x] = mm;
      fence_proxy_async();
      const float2 mm2 = finish_minmax(1);  // includes the grid barrier
      B2_TRACE(kTrP1Done);
      p2 = u8_params(mm2.x, mm2.y);
      if (blockIdx.x == 0 && ct == 0) {
        hdr_of(a.win[0])->hdr2 = mm2;
        if (a.n && !(finite_f(mm2.x) && finite_f(mm2.y))) latch(a.status, kStatusNonFinite);
      }
      if (ct == 0) s_gate = 1;  // codes of every CTA are written: release the producer
    }
    const PassDesc& pc = s_m[2];  // the codes
    if (r.producer && (threadIdx.x & 31) == 0) gate_wait(&s_gate, 1);
    r.run(pc, [&](const uint8_t* st, size_t e0, size_t units, int) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        const size_t e = e0 + 4 * size_t(gi);
        float4 y2 = add0(dequant4(cs[gi], p1));
        if (EC) y2 = sub4(y2, eps4(a.eps, e, 0));
        const float4 d2 = dequant4(q4r(y2, p2.lo, p2.inv, r2, e), p2);
        __stcs(x4 + (e >> 2), d2);
        if (EC) set_eps4(a.eps, e, 0, sub4(y2, d2));
      }
    });
    r.edges(pc, [&](size_t e) {
      float y2 = __fadd_rn(dequant1(codes[e], p1.lo, p1.step), 0.0f);
      if (EC) y2 = __fsub_rn(y2, a.eps[e]);
      const float d2 = dequant1(q1r(y2, p2.lo, p2.inv, r2, e), p2.lo, p2.step);
      a.x[e] = d2;
      if (EC) a.eps[e] = __fsub_rn(y2, d2);
    });
    B2_TRACE(kTrEnd);
    return;
  }

  // ------------------------------------------------------ phase 1 / 2 common
  const PassDesc& pf = s_pq[g];  // my fold
  // pairs of aligned groups through the fold (8 fp64 chains per thread)
  auto fold_pairs = [&](const uint8_t* st, size_t units, int T, bool fast, int gct, int gn, auto&& body) {
    const int ng = int(units * 4);
    for (int gi = gct; gi < ng; gi += 2 * gn) {
      const int g1 = gi + gn;
      const bool has1 = g1 < ng;
      float4 y0, y1;
      fold2<CODEC>(g, fast, st, gi, has1 ? g1 : gi, T, s_dec, 1.0, y0, y1);
      body(gi, y0);
      if (has1) body(g1, y1);
    }
  };
  auto fold1 = [&](size_t e) -> float {
    double acc = 0.0;
    for (int j = 0; j < g; ++j) {
      const uint8_t* slot = g >= 2 ? a.win[j] + a.off_recv1 + size_t(me) * a.slot_stride
                                   : a.win[me] + a.off_recv1 + size_t(j) * a.slot_stride;
      const float d = CODEC == kU8 ? dequant1(__ldcg(slot + (e - mbase)), s_dec[j].lo, s_dec[j].step)
                                   : __ldcg(reinterpret_cast<const float*>(slot) + (e - mbase));
      acc = __dadd_rn(acc, double(d));
    }
    return __double2float_rn(acc);
  };
  uint8_t* out2 = a.win[me] + a.off_out2;
  // chunk k = (me+1+i) % g for pass i; i == g-1 is my own chunk
  const PassDesc* pc = s_pc;
  auto ck = [&](int i) { return i + me + 1 < g ? i + me + 1 : i + me + 1 - g; };

  if (CODEC == kU8) {
    // ---------------------------------------- phase 1A: (min, max) of every chunk
    // One pass over x with the chunks' tiles interleaved; per-chunk partials,
    // one grid barrier, then CTA 0 sends each owner its header.
    float cl[kMaxRanks], ch[kMaxRanks];
#pragma unroll
    for (int j = 0; j < kMaxRanks; ++j) {
      cl[j] = kInf;
      ch[j] = -kInf;
    }
    r.run_multi(pc, g, [&](int i, const uint8_t* st, size_t, size_t units, int T) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
      float lo = kInf, hi = -kInf;
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        float4 v = xs[gi];
        if (EC) v = sub4(v, ds[gi]);
        mm_acc(lo, hi, v);
      }
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j)
        if (j == i) {
          cl[j] = fmin_nan(cl[j], lo);
          ch[j] = fmax_nan(ch[j], hi);
        }
    });
#pragma unroll
    for (int j = 0; j < kMaxRanks; ++j)
      if (j < g)
        r.edges(pc[j], [&](size_t e) {
          float v = a.x[e];
          if (EC) v = __fsub_rn(v, a.delta[e]);
          mm_acc1(cl[j], ch[j], v);
        });
    B2_TRACE(kTrP1Step + 2);  // this CTA's share of the min/max pass streamed
    if (cons) {
#pragma unroll
      for (int j = 0; j < kMaxRanks; ++j)
        if (j < g) {
          const float2 mm = consumer_minmax(cl[j], ch[j], red);
          if (ct == 0) a.partials[size_t(j) * G + blockIdx.x] = mm;
        }
      consumer_grid_sync(a.gridbar);
      B2_TRACE(kTrP1Step + 3);
      for (int j = 0; j < g; ++j) {
        const float2 mm = reduce_partials(a.partials + size_t(j) * G, G, red, ct);
        if (ct == 0) {
          s_mm1[j] = mm;
          s_p1[j] = u8_params(mm.x, mm.y);
        }
      }
      B2_TRACE(kTrP1FirstA);
      if (blockIdx.x == 0 && ct == 0) {
        for (int j = 0; j < g; ++j) {
          hdr_of(a.win[ck(j)])->hdr1[me] = s_mm1[j];  // remote 8-byte store into owner's header
          if (pc[j].n && !(finite_f(s_mm1[j].x) && finite_f(s_mm1[j].y))) latch(a.status, kStatusNonFinite);
        }
        B2_TRACE(kTrP1Fenced + 4);  // headers stored
        __threadfence_system();
        B2_TRACE(kTrP1Fenced + 5);  // headers fenced
        // one fence above orders the headers before every signal (relaxed reds:
        // a .release per red would repeat the fence g times)
        for (int j = 0; j < g; ++j) red_relaxed_sys_add(&hdr_of(a.win[ck(j)])->arrive1, 1ull);
        B2_TRACE(kTrP1Fenced + 6);  // headers signalled
      }
      consumer_sync();
    }

    // ------------------------- phase 1B + 2A: encode every chunk, fold as it lands
    // Pass i < g quantizes chunk ck(i) into MY window (slot ck(i)); the
    // signaller warp confirms the stores (one system fence per batch of
    // tiles) and adds each tile's units to owner ck(i)'s region counter.  Pass
    // g is my fold: its tiles PULL the g encodings of a region of my chunk
    // straight from the g windows with TMA once the region's counter says all
    // g have landed -- so the NVLink transfer is asynchronous TMA reads (warps
    // never stall on remote stores, which measured 168 us for this pass mix)
    // and the fold runs under the encode instead of after it.  Chunks are
    // walked backwards (their tails are still in L2 from phase 1A).
    auto load_dec = [&]() {  // contribution headers -> smem (one thread)
      int fast = 1;
      for (int j = 0; j < g; ++j) {
        const float2 h = __ldcg(&mine->hdr1[j]);
        const U8Params q = u8_params(h.x, h.y);
        s_dec[j] = SrcDec{q.lo, q.step, q.c23};
        if (!(q.fastdec && fold_fast_ok(q.lo, q.step))) fast = 0;
      }
      s_fast = fast;
    };
    r.timed = a.trace != nullptr;
    if (r.storer && (threadIdx.x & 31) == 0) {
      r.signal_loop();
      if (a.trace) {
        a.trace[size_t(blockIdx.x) * kTraceSlots + kTrP1Step + 1] = globaltimer();  // pushes landed
        a.trace[size_t(blockIdx.x) * kTraceSlots + kTrWait + 3] = r.wt[1];           // storer: retiring
      }
    }
    float lo2 = kInf, hi2 = -kInf;
    // split mode: pipe A (3 stages, 10 consumer warps) encodes from local x,
    // pipe B (2 stages, 8 warps) folds from the TMA pulls
    r.split_begin();
    const int gct = r.gct, gn = r.gn;
    r.stream_split(
        s_pq, g,
        [&](int i, const uint8_t* st, size_t e0, size_t units, int T) {
          const int k = ck(i);
          const U8Params p = s_p1[i];
          const float4* xs = reinterpret_cast<const float4*>(st);
          const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
          uint32_t* dst = reinterpret_cast<uint32_t*>(a.win[me] + a.off_recv1 + size_t(k) * a.slot_stride +
                                                      (e0 - (pc[i].s & ~size_t(15))));
          r.slot_acquire();
          for (int gi = gct; gi < int(units * 4); gi += gn) {
            float4 y = xs[gi];
            if (EC) y = sub4(y, ds[gi]);
            const uint32_t q = q4r(y, p.lo, p.inv, r1, e0 + 4 * size_t(gi));
            dst[gi] = q;  // my codes of chunk k, in my window: owner k pulls them
            if (EC) dl4[(e0 >> 2) + gi] = sub4(y, dequant4(q, p));
          }
          unsigned long long* sig = reinterpret_cast<unsigned long long*>(a.win[k] + a.off_gate) +
                                    ((e0 >> 4) - pc[i].u0()) / kGateUnits;
          r.slot_commit(sig, unsigned(units));
        },
        [](int) {}, s_pq + g, 1,
        [&](int, const uint8_t* st, size_t e0, size_t units, int T) {
          fold_pairs(st, units, T, s_fast != 0, gct, gn, [&](int gi, float4 y) {
            const size_t e = e0 + 4 * size_t(gi);
            if (EC) y = sub4(y, eps4(a.eps, e, mlo));
            x4[e >> 2] = y;  // x's own chunk was consumed by its encode: cache y2 there
            mm_acc(lo2, hi2, y);
          });
        },
        [&](int) {
          load_dec();
          if (a.trace) a.trace[size_t(blockIdx.x) * kTraceSlots + kTrP1Step + 7] = globaltimer();  // headers in
        });
    if (r.group_a()) {  // marker: the signaller confirms everything and stops
      r.slot_acquire();
      r.slot_commit(nullptr, 0u, true);
    }
    r.split_end();
    if (a.trace) {
      unsigned long long* tw = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrWait;
      unsigned long long* ts = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrP1Step;
      if (ct == 0) {
        tw[0] = r.wt[0];  // encode consumers: free credit
        tw[4] = r.wt[2];  // encode consumers: full stage
      } else if (ct == 32 * kSplitWarpsA) {
        tw[5] = r.wt[2];  // fold consumers: full stage
      } else if (r.producer && threadIdx.x == 0) {
        tw[2] = r.wt[1];  // encode producer: free stage
        unsigned long long enc = 0;
        for (int i = 0; i < g; ++i) enc = r.pst[i].last > enc ? r.pst[i].last : enc;
        ts[4] = enc;  // p1_step4: last encode tile issued
      } else if (r.producer2 && threadIdx.x == kProducer2) {
        tw[1] = r.wt[0];        // fold producer: arrival gates
        ts[5] = r.pst2[0].first;  // p1_step5: first fold tile issued
        ts[6] = r.pst2[0].last;   // p1_step6: last fold tile issued
      }
    }
    r.timed = false;
    B2_TRACE(kTrP1Done);
    // unaligned heads/tails (warp 0 of the last CTA): pushed with plain stores,
    // announced on arrive_e; then the fold of my chunk's own heads/tails.
    // Every rank knows from (n, g) alone whether any chunk has one: when none
    // has (n % 16g == 0, the BASELINE sizes) the rendezvous is skipped.
    if (cons && blockIdx.x == G - 1 && ct < 32 && any_edges) {
      for (int i = 0; i < g; ++i) {
        const U8Params p = s_p1[i];
        uint8_t* dst = a.win[me] + a.off_recv1 + size_t(ck(i)) * a.slot_stride;
        const size_t ebase = pc[i].s & ~size_t(15);
        r.edges(pc[i], [&](size_t e) {
          float y = a.x[e];
          if (EC) y = __fsub_rn(y, a.delta[e]);
          const uint8_t q = q1r(y, p.lo, p.inv, r1, e);
          dst[e - ebase] = q;
          if (EC) a.delta[e] = __fsub_rn(y, dequant1(q, p.lo, p.step));
        });
      }
      __threadfence_system();
      __syncwarp();
      if (ct == 0) {
        for (int i = 0; i < g; ++i) red_relaxed_sys_add(&hdr_of(a.win[ck(i)])->arrive_e, 1ull);
        wait_geq(&mine->arrive_e, gmul, a.timeout_ns, a.status);
        wait_geq(&mine->arrive1, gmul, a.timeout_ns, a.status);
        load_dec();
      }
      __syncwarp();
      r.edges(pf, [&](size_t e) {
        float y = fold1(e);
        if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
        a.x[e] = y;
        mm_acc1(lo2, hi2, y);
      });
    }
    U8Params p{};
    if (cons) {
      const float2 mm0 = consumer_minmax(lo2, hi2, red);
      if (ct == 0) a.partials[size_t(kMaxRanks) * G + blockIdx.x] = mm0;
      fence_proxy_async();
      const float2 mm = finish_minmax(kMaxRanks);
      B2_TRACE(kTrP2A);
      p = u8_params(mm.x, mm.y);
      if (blockIdx.x == 0 && ct == 0) {
        mine->hdr2 = mm;
        if (msz && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
      }
      if (ct == 0) s_gate = 1;
    }
    // second Q: only the payload is written here, so ready2 can be published
    // as early as possible; the owner's own chunk of x is decoded from it in
    // phase 3, in the shadow of the NVLink pulls.
    auto emit = [&](size_t e, float4 y) {
      const uint32_t q = q4r(y, p.lo, p.inv, r2, e);
      *reinterpret_cast<uint32_t*>(out2 + (e - mbase)) = q;
      if (EC) set_eps4(a.eps, e, mlo, sub4(y, dequant4(q, p)));
    };
    auto emit1 = [&](size_t e, float y) {
      const uint8_t q = q1r(y, p.lo, p.inv, r2, e);
      out2[e - mbase] = q;
      if (EC) a.eps[e - mlo] = __fsub_rn(y, dequant1(q, p.lo, p.step));
    };
    const PassDesc& ps = s_m[1];  // the y2 cached in x's own chunk (reversed)
    if (r.producer && (threadIdx.x & 31) == 0) gate_wait(&s_gate, 1);
    r.run(ps, [&](const uint8_t* st, size_t e0, size_t units, int) {
      const float4* ys = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) emit(e0 + 4 * size_t(gi), ys[gi]);
    });
    r.edges(ps, [&](size_t e) { emit1(e, a.x[e]); });
  } else if (g >= 2) {
    // -------------------------------- identity: copy to my window + pulled fold
    // The uint8 phase-1B scheme without codes: pipe A copies y of chunk ck(i)
    // into my window slot ck(i) and credits owner ck(i)'s region counters;
    // pipe B folds my chunk from the g windows (TMA pulls) region by region
    // as they land, straight into out2.
    float* outf = reinterpret_cast<float*>(out2);
    r.timed = a.trace != nullptr;
    r.split_begin();
    const int gct = r.gct, gn = r.gn;
    if (r.storer && (threadIdx.x & 31) == 0) r.signal_loop();
    r.stream_split(
        s_pq, g,
        [&](int i, const uint8_t* st, size_t e0, size_t units, int T) {
          const int k = ck(i);
          const float4* xs = reinterpret_cast<const float4*>(st);
          const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
          float4* dst = reinterpret_cast<float4*>(a.win[me] + a.off_recv1 + size_t(k) * a.slot_stride) +
                        ((e0 - (pc[i].s & ~size_t(15))) >> 2);
          r.slot_acquire();
          for (int gi = gct; gi < int(units * 4); gi += gn) {
            float4 y = xs[gi];
            if (EC) y = sub4(y, ds[gi]);
            dst[gi] = y;
            if (a.check_finite) bad |= !finite4(y);
            if (EC) dl4[(e0 >> 2) + gi] = sub4(y, y);
          }
          unsigned long long* sig = reinterpret_cast<unsigned long long*>(a.win[k] + a.off_gate) +
                                    ((e0 >> 4) - pc[i].u0()) / kGateUnits;
          r.slot_commit(sig, unsigned(units));
        },
        [](int) {}, s_pq + g, 1,
        [&](int, const uint8_t* st, size_t e0, size_t units, int T) {
          fold_pairs(st, units, T, true, gct, gn, [&](int gi, float4 y) {
            const size_t e = e0 + 4 * size_t(gi);
            if (EC) y = sub4(y, eps4(a.eps, e, mlo));
            if (a.check_finite) bad |= !finite4(y);
            if (EC) set_eps4(a.eps, e, mlo, sub4(y, y));
            *reinterpret_cast<float4*>(outf + (e - mbase)) = y;
          });
        },
        [](int) {});
    if (r.group_a()) {  // marker: the signaller confirms everything and stops
      r.slot_acquire();
      r.slot_commit(nullptr, 0u, true);
    }
    r.split_end();
    r.timed = false;
    B2_TRACE(kTrP1Done);
    // unaligned heads/tails (warp 0 of the last CTA): copies, announced on
    // arrive_e; then the fold of my chunk's own heads/tails (skipped when no
    // chunk has one, as above)
    if (cons && blockIdx.x == G - 1 && ct < 32 && any_edges) {
      for (int i = 0; i < g; ++i) {
        float* dstf = reinterpret_cast<float*>(a.win[me] + a.off_recv1 + size_t(ck(i)) * a.slot_stride);
        const size_t ebase = pc[i].s & ~size_t(15);
        r.edges(pc[i], [&](size_t e) {
          float y = a.x[e];
          if (EC) y = __fsub_rn(y, a.delta[e]);
          dstf[e - ebase] = y;
          if (a.check_finite) bad |= !finite_f(y);
          if (EC) a.delta[e] = __fsub_rn(y, y);
        });
      }
      __threadfence_system();
      __syncwarp();
      if (ct == 0) {
        for (int i = 0; i < g; ++i) red_relaxed_sys_add(&hdr_of(a.win[ck(i)])->arrive_e, 1ull);
        wait_geq(&mine->arrive_e, gmul, a.timeout_ns, a.status);
      }
      __syncwarp();
      r.edges(pf, [&](size_t e) {
        float y = fold1(e);
        if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
        if (a.check_finite) bad |= !finite_f(y);
        if (EC) a.eps[e - mlo] = __fsub_rn(y, y);
        outf[e - mbase] = y;
      });
    }
  } else {
    // ------------------------------------- identity, one rank: phase 1 push
    // Step i stores chunk me+1+i into its owner's window (a permutation of
    // destinations across ranks); the last CTA to finish a step signals.
    for (int i = 0; i < g; ++i) {
      const int k = ck(i);
      const PassDesc& px = pc[i];
      float* dstf = reinterpret_cast<float*>(a.win[k] + a.off_recv1 + size_t(me) * a.slot_stride);
      const size_t ebase = px.s & ~size_t(15);  // slot element index = e - ebase
      r.run(px, [&](const uint8_t* st, size_t e0, size_t units, int T) {
        const float4* xs = reinterpret_cast<const float4*>(st);
        const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
        for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
          float4 y = xs[gi];
          if (EC) y = sub4(y, ds[gi]);
          const size_t e = e0 + 4 * size_t(gi);
          *reinterpret_cast<float4*>(dstf + (e - ebase)) = y;
          if (a.check_finite) bad |= !finite4(y);
          if (EC) dl4[e >> 2] = sub4(y, y);
        }
      });
      r.edges(px, [&](size_t e) {
        float y = a.x[e];
        if (EC) y = __fsub_rn(y, a.delta[e]);
        dstf[e - ebase] = y;
        if (a.check_finite) bad |= !finite_f(y);
        if (EC) a.delta[e] = __fsub_rn(y, y);
      });
      if (i == 0) B2_TRACE(kTrP1FirstB);
      B2_TRACE(kTrP1Step + i);
      if (cons && consumer_arrive<true>(a.cta_done + k, &s_flag) && ct == 0)
        red_relaxed_sys_add(&hdr_of(a.win[k])->arrive1, 1ull);  // consumer_arrive fenced (sys)
      B2_TRACE(kTrP1Fenced + i);
    }
    B2_TRACE(kTrP1Done);

    // ------------------------------------------ identity: phase 2 owner reduce
    if (cons && ct == 0) wait_geq(&mine->arrive1, pf.wait_target, a.timeout_ns, a.status);
    B2_TRACE(kTrP2Ready);
    float* outf = reinterpret_cast<float*>(out2);
    r.run(pf, [&](const uint8_t* st, size_t e0, size_t units, int T) {
      fold_pairs(st, units, T, true, ct, kConsumers, [&](int gi, float4 y) {
        const size_t e = e0 + 4 * size_t(gi);
        if (EC) y = sub4(y, eps4(a.eps, e, mlo));
        if (a.check_finite) bad |= !finite4(y);
        if (EC) set_eps4(a.eps, e, mlo, sub4(y, y));
        if (g > 1)
          *reinterpret_cast<float4*>(outf + (e - mbase)) = y;
        else
          __stcs(x4 + (e >> 2), y);
      });
    });
    r.edges(pf, [&](size_t e) {
      float y = fold1(e);
      if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
      if (a.check_finite) bad |= !finite_f(y);
      if (EC) a.eps[e - mlo] = __fsub_rn(y, y);
      if (g > 1)
        outf[e - mbase] = y;
      else
        a.x[e] = y;
    });
  }
  if (bad) latch(a.status, kStatusNonFinite);
  if (g == 1) {
    B2_TRACE(kTrEnd);
    return;
  }
  B2_TRACE(kTrP2Pass);
  if (cons && consumer_arrive<false>(a.cta_done + kMaxRanks, &s_flag) && ct == 0)
    st_relaxed_sys(&mine->ready2, a.epoch);  // the last CTA's fence.sys in consumer_arrive orders it
  B2_TRACE(kTrP2Done);

  // ------------------------------------------------------ phase 3: pull + decode
  // Every other owner's payload is pulled with TMA over NVLink, all owners at
  // once with tiles interleaved round-robin (balanced fan-in whatever the rank
  // skew), plus the owner's own payload decoded into its own chunk.
  {
    const PassDesc* pp = s_pp;
    auto powner = [&](int i) { return i + me + 1 < g ? i + me + 1 : i + me + 1 - g; };  // g-1: self
    // header of owner i: read by the producer after owner i's flag (ready
    // callback) or, for the edge elements, by consumer warp 0 of the last CTA
    auto load_hdr = [&](int i) {
      const int k = powner(i);
      WinHdr* hk = hdr_of(a.win[k]);
      if (CODEC == kU8) {
        const float2 h = k == me ? mine->hdr2 : ld_peer_f2(&hk->hdr2);
        const U8Params q = u8_params(h.x, h.y);
        s_dec3[i] = SrcDec{q.lo, q.step, q.c23};
        s_fast3[i] = q.fastdec;
      }
    };
    if (cons) B2_TRACE(kTrP3First);
    if (CODEC == kU8) {
      r.run_multi(
          pp, g,
          [&](int i, const uint8_t* st, size_t e0, size_t units, int) {
            const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
            const SrcDec kd = s_dec3[i];
            if (s_fast3[i]) {
              for (int gi = ct; gi < int(units * 4); gi += kConsumers)
                __stcs(x4 + ((e0 >> 2) + gi), dequant4_fast(cs[gi], kd.lo, kd.step, kd.c23));
            } else {
              for (int gi = ct; gi < int(units * 4); gi += kConsumers)
                __stcs(x4 + ((e0 >> 2) + gi), dequant4(cs[gi], kd.lo, kd.step));
            }
          },
          load_hdr);
    } else {
      r.run_multi(pp, g, [&](int, const uint8_t* st, size_t e0, size_t units, int) {
        const float4* fs = reinterpret_cast<const float4*>(st);
        for (int gi = ct; gi < int(units * 4); gi += kConsumers) __stcs(x4 + ((e0 >> 2) + gi), fs[gi]);
      });
    }
    // unaligned heads/tails (last CTA, consumer warp 0): wait + header per owner
    if (cons && blockIdx.x == gridDim.x - 1 && ct < 32) {
      for (int i = 0; i < g; ++i) {
        if (pp[i].body_begin() == pp[i].s && pp[i].body_end() == pp[i].s + pp[i].n) continue;
        if (ct == 0) {
          wait_geq(&hdr_of(a.win[powner(i)])->ready2, a.epoch, a.timeout_ns, a.status);
          load_hdr(i);
        }
        __syncwarp();
        const uint8_t* src = a.win[powner(i)] + a.off_out2;
        const SrcDec kd = s_dec3[i];
        r.edges(pp[i], [&](size_t e) {
          a.x[e] = CODEC == kU8 ? dequant1(__ldcg(src + (e - (pp[i].s & ~size_t(15)))), kd.lo, kd.step)
                               : __ldcg(reinterpret_cast<const float*>(src) + (e - (pp[i].s & ~size_t(15))));
        });
        __syncwarp();
      }
    }
  }
  B2_TRACE(kTrEnd);
}

// The kernels: ring setup, the body, then the dynamic tile counters are reset
// for the next launch on this window.
template <int CODEC, bool EC>
__global__ void __launch_bounds__(kRingThreads, 1) central_kernel(CentralArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring r;
  r.init(smem, a.status, a.timeout_ns, a.sched);
  central_body<CODEC, EC>(a, r);
  r.finish(a.sched_end);
}

// ---------------------------------------------------------------- D_* kernel
template <int CODEC>
__device__ __forceinline__ void decent_body(const DecentArgs& a, Ring& r) {
  __shared__ float2 red[32];
  __shared__ SrcDec s_dec[kMaxRanks];
  __shared__ int s_fast;
  __shared__ int s_flag;
  const int G = gridDim.x, me = a.me, p = a.parity, ct = r.ct;
  const bool cons = r.ct >= 0;
  WinHdr* mine = hdr_of(a.win[me]);
  uint8_t* mybuf = a.win[me] + a.off_dbuf;
  const Rounder rd = make_rounder(CODEC == kU8 && a.sr_on, a.sr_seed, me, 3);
  float4* x4 = reinterpret_cast<float4*>(a.x);
  int bad = 0;
  B2_TRACE(kTrStart);

  __shared__ PassDesc s_d[3];  // all of x, all of x reversed, the gather (shared: see central_body)
  if (threadIdx.x == 0) {
    PassDesc& px = s_d[0];
    px = PassDesc::make();
    px.n = a.n;
    px.base[0] = reinterpret_cast<const uint8_t*>(a.x);
    s_d[1] = px;
    s_d[1].reverse = true;
    PassDesc& pg = s_d[2];  // every neighbour's buffer (self included), ascending order
    pg = PassDesc::make();
    pg.n = a.n;
    pg.eb = CODEC == kU8 ? 1 : 4;
    pg.nsrc = a.nnb;
    for (int i = 0; i < a.nnb; ++i) pg.base[i] = a.win[a.nbrs[i]] + a.off_dbuf;
    pg.gate = reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate);
    pg.gate_mult = 1;  // units(r) = gate_target(r)
    pg.gate_nsrc = a.nnb;
    for (int i = 0; i < a.nnb; ++i) {
      pg.gate_src[i] = a.nbrs[i];
      pg.gate_tgt[i] = a.sends[i];
    }
    pg.gate_stride = a.gate_stride;
    pg.reverse = true;  // regions land in the order of the (reversed) encode
  }
  __syncthreads();
  const PassDesc& px = s_d[0];

  if (a.nnb == 1) {
    // ----- the neighbourhood is {self}: nothing is published or read;
    // x' = (float)((0.0 + (double)D(Q(x))) * inv) = D(Q(x)) + 0.0f (identity:
    // x + 0.0f) because inv == 1.0 for a single term.
    if (CODEC == kU8) {
      float lo = kInf, hi = -kInf;
      r.run(px, [&](const uint8_t* st, size_t, size_t units, int) {
        const float4* xs = reinterpret_cast<const float4*>(st);
        for (int gi = ct; gi < int(units * 4); gi += kConsumers) mm_acc(lo, hi, xs[gi]);
      });
      r.edges(px, [&](size_t e) { mm_acc1(lo, hi, a.x[e]); });
      U8Params q8{};
      if (cons) {
        const float2 m0 = consumer_minmax(lo, hi, red);
        if (ct == 0) a.partials[blockIdx.x] = m0;
        consumer_grid_sync(a.gridbar);
        const float2 mm = reduce_partials(a.partials, G, red, ct);
        q8 = u8_params(mm.x, mm.y);
        if (blockIdx.x == 0 && ct == 0 && a.n && !(finite_f(mm.x) && finite_f(mm.y)))
          latch(a.status, kStatusNonFinite);
      }
      const PassDesc& pb = s_d[1];
      r.run(pb, [&](const uint8_t* st, size_t e0, size_t units, int) {
        const float4* xs = reinterpret_cast<const float4*>(st);
        for (int gi = ct; gi < int(units * 4); gi += kConsumers)
          __stcs(x4 + ((e0 >> 2) + gi), add0(dequant4(q4r(xs[gi], q8.lo, q8.inv, rd, e0 + 4 * size_t(gi)), q8)));
      });
      r.edges(px, [&](size_t e) {
        a.x[e] = __fadd_rn(dequant1(q1r(a.x[e], q8.lo, q8.inv, rd, e), q8), 0.0f);
      });
    } else {
      r.run(px, [&](const uint8_t* st, size_t e0, size_t units, int) {
        const float4* xs = reinterpret_cast<const float4*>(st);
        for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
          if (a.check_finite) bad |= !finite4(xs[gi]);
          __stcs(x4 + ((e0 >> 2) + gi), add0(xs[gi]));
        }
      });
      r.edges(px, [&](size_t e) {
        if (a.check_finite) bad |= !finite_f(a.x[e]);
        a.x[e] = __fadd_rn(a.x[e], 0.0f);
      });
      if (bad) latch(a.status, kStatusNonFinite);
    }
    B2_TRACE(kTrEnd);
    return;
  }

  // ----- publish: one (min,max) of the whole bucket (collectives.cpp:266),
  // the header, then -- in split mode -- pipe A encodes (or stages) the bucket
  // into my parity buffer while pipe B gathers: each tile TMA-pulls the |N|
  // encodings of one region (neighbours over NVLink, self locally) as soon as
  // the region's counter says all |N| have landed, folds them in fp64 in
  // ascending neighbour order, scales by 1/|N| and overwrites x (my own encode
  // of that region has consumed it).  Counters are per call parity: a
  // neighbour runs at most one call ahead.
  U8Params q8{};
  if (CODEC == kU8) {
    float lo = kInf, hi = -kInf;
    r.run(px, [&](const uint8_t* st, size_t, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) mm_acc(lo, hi, xs[gi]);
    });
    r.edges(px, [&](size_t e) { mm_acc1(lo, hi, a.x[e]); });
    if (cons) {
      const float2 m0 = consumer_minmax(lo, hi, red);
      if (ct == 0) a.partials[blockIdx.x] = m0;
      consumer_grid_sync(a.gridbar);
      const float2 mm = reduce_partials(a.partials, G, red, ct);
      B2_TRACE(kTrP1FirstA);
      q8 = u8_params(mm.x, mm.y);
      if (ct == 0) {
        // the neighbours of two rounds ago must be done reading this buffer
        if (a.expected_reads) wait_geq(&mine->dreads[p], a.expected_reads, a.timeout_ns, a.status);
        if (blockIdx.x == 0) {
          mine->dhdr[p] = mm;
          if (a.n && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
          __threadfence_system();
          st_relaxed_sys(&mine->dready[p], a.epoch);  // header published
        }
      }
      consumer_sync();
    }
  } else if (cons) {
    if (ct == 0 && a.expected_reads) wait_geq(&mine->dreads[p], a.expected_reads, a.timeout_ns, a.status);
    consumer_sync();
  }
  const double inv = a.inv;
  r.timed = a.trace != nullptr;
  r.split_begin();
  const int gct = r.gct, gn = r.gn;
  if (r.storer && (threadIdx.x & 31) == 0) {
    // a credit's "sig" carries the region index: every neighbour's counter of
    // that region for me (self included) gets the tile's units
    r.signal_loop([&](unsigned long long* sig, unsigned v) {
      const size_t region = reinterpret_cast<size_t>(sig) - 1;
      for (int i = 0; i < a.nnb; ++i)
        red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[a.nbrs[i]] + a.off_gate) +
                                size_t(me) * a.gate_stride + region,
                            v);
    });
  }
  auto load_dec = [&]() {  // neighbours' headers -> smem (one thread)
    if (CODEC != kU8) {
      s_fast = 1;
      return;
    }
    int fast = 1;
    for (int i = 0; i < a.nnb; ++i) {
      WinHdr* hk = hdr_of(a.win[a.nbrs[i]]);
      wait_geq(&hk->dready[p], a.epoch, a.timeout_ns, a.status);
      const float2 h = ld_peer_f2(&hk->dhdr[p]);
      const U8Params q = u8_params(h.x, h.y);
      s_dec[i] = SrcDec{q.lo, q.step, q.c23};
      if (!(q.fastdec && fold_fast_ok(q.lo, q.step))) fast = 0;
    }
    s_fast = fast;
  };
  r.stream_split(
      &s_d[1], 1,
      [&](int, const uint8_t* st, size_t e0, size_t units, int) {
        const float4* xs = reinterpret_cast<const float4*>(st);
        r.slot_acquire();
        if (CODEC == kU8) {
          uint32_t* b32 = reinterpret_cast<uint32_t*>(mybuf + e0);
          for (int gi = gct; gi < int(units * 4); gi += gn)
            b32[gi] = q4r(xs[gi], q8.lo, q8.inv, rd, e0 + 4 * size_t(gi));
        } else {
          float4* b4 = reinterpret_cast<float4*>(mybuf + 4 * e0);
          for (int gi = gct; gi < int(units * 4); gi += gn) {
            b4[gi] = xs[gi];
            if (a.check_finite) bad |= !finite4(xs[gi]);
          }
        }
        r.slot_commit(reinterpret_cast<unsigned long long*>((e0 >> 4) / kGateUnits + 1), unsigned(units));
      },
      [](int) {}, &s_d[2], 1,
      [&](int, const uint8_t* st, size_t e0, size_t units, int T) {
        const int ng = int(units * 4);
        const bool fast = s_fast != 0;
        for (int gi = gct; gi < ng; gi += 2 * gn) {
          const int g1 = gi + gn;
          const bool has1 = g1 < ng;
          float4 y0, y1;
          fold2<CODEC>(a.nnb, fast, st, gi, has1 ? g1 : gi, T, s_dec, inv, y0, y1);
          __stcs(x4 + ((e0 >> 2) + gi), y0);
          if (has1) __stcs(x4 + ((e0 >> 2) + g1), y1);
        }
      },
      [&](int) { load_dec(); });
  if (r.group_a()) {  // marker: the signaller confirms everything and stops
    r.slot_acquire();
    r.slot_commit(nullptr, 0u, true);
  }
  r.split_end();
  if (a.trace) {
    unsigned long long* tw = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrWait;
    if (ct == 0) {
      tw[0] = r.wt[0];  // encode consumers: free credit
      tw[4] = r.wt[2];  // encode consumers: full stage
    } else if (ct == 32 * kSplitWarpsA) {
      tw[5] = r.wt[2];  // gather consumers: full stage
    } else if (r.producer && threadIdx.x == 0) {
      tw[2] = r.wt[1];  // encode producer: free stage
    } else if (r.producer2 && threadIdx.x == kProducer2) {
      tw[1] = r.wt[0];  // gather producer: arrival slots
      unsigned long long* ts = a.trace + size_t(blockIdx.x) * kTraceSlots + kTrP1Step;
      ts[5] = r.pst2[0].first;  // p1_step5: first gather tile issued
      ts[6] = r.pst2[0].last;   // p1_step6: last gather tile issued
    } else if (r.storer && threadIdx.x == 32) {
      tw[3] = r.wt[1];  // signaller: fences
    }
  }
  r.timed = false;
  B2_TRACE(kTrP1Done);
  // unaligned tail (warp 0 of the last CTA): encode it, announce it on every
  // neighbour's arrive_e, then fold it once every neighbour's tail is in
  // (every rank skips it alike when n % 16 == 0: there is no tail)
  if (cons && blockIdx.x == G - 1 && ct < 32 && (a.n & 15)) {
    r.edges(px, [&](size_t e) {
      if (CODEC == kU8) {
        mybuf[e] = q1r(a.x[e], q8.lo, q8.inv, rd, e);
      } else {
        reinterpret_cast<float*>(mybuf)[e] = a.x[e];
        if (a.check_finite) bad |= !finite_f(a.x[e]);
      }
    });
    __threadfence_system();
    __syncwarp();
    if (ct == 0) {
      // the tail's counter (index gate_stride - 1) per source, counted like the regions
      const size_t tail = a.gate_stride - 1;
      for (int i = 0; i < a.nnb; ++i)
        red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[a.nbrs[i]] + a.off_gate) +
                                size_t(me) * a.gate_stride + tail,
                            1ull);
      for (int i = 0; i < a.nnb; ++i)
        wait_geq(reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate) +
                     size_t(a.nbrs[i]) * a.gate_stride + tail,
                 a.sends[i], a.timeout_ns, a.status);
      load_dec();
    }
    __syncwarp();
    const PassDesc& pg = s_d[2];
    r.edges(pg, [&](size_t e) {
      double acc = 0.0;
      for (int j = 0; j < a.nnb; ++j) {
        const uint8_t* buf = a.win[a.nbrs[j]] + a.off_dbuf;
        const float d = CODEC == kU8 ? dequant1(__ldcg(buf + e), s_dec[j].lo, s_dec[j].step)
                                     : __ldcg(reinterpret_cast<const float*>(buf) + e);
        acc = __dadd_rn(acc, double(d));
      }
      a.x[e] = __double2float_rn(__dmul_rn(acc, inv));
    });
  }
  if (bad) latch(a.status, kStatusNonFinite);
  // ----- acknowledge the reads so each neighbour may reuse its buffer
  if (cons && consumer_arrive<false>(a.cta_done + 1, &s_flag) && ct == 0)
    for (int i = 0; i < a.nnb; ++i)
      if (a.nbrs[i] != me) red_relaxed_sys_add(&hdr_of(a.win[a.nbrs[i]])->dreads[p], 1ull);
  B2_TRACE(kTrEnd);
}

template <int CODEC>
__global__ void __launch_bounds__(kRingThreads, 1) decent_kernel(DecentArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring r;
  r.init(smem, a.status, a.timeout_ns, a.sched);
  decent_body<CODEC>(a, r);
  r.finish(a.sched_end);
}

template <typename K, typename A>
int launch_ring(K kernel, const A& args, cudaStream_t s, int sms) {
  static_assert(sizeof(A) < 4000, "kernel argument block too large");
  B2_CUDA_TRY(ensure_ring_smem(reinterpret_cast<const void*>(kernel)));
  // one persistent CTA per SM (all co-resident), or the communicator's SM
  // budget: fewer CTAs leave SMs to concurrent compute (the engine overlap)
  const int grid = sms > 0 && sms < sm_count() ? sms : sm_count();
  A copy = args;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(kRingThreads),
                                          params, kRingSmem, s));
  return B2_OK;
}

}  // namespace

// The 192 KB ring exceeds the default 48 KB dynamic-smem limit: opt in once
// per (kernel, device).
cudaError_t ensure_ring_smem(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}

int launch_central(const CentralArgs& a, int codec, bool ec, cudaStream_t s, int sms) {
  if (codec == kU8)
    return ec ? launch_ring(central_kernel<kU8, true>, a, s, sms) : launch_ring(central_kernel<kU8, false>, a, s, sms);
  return ec ? launch_ring(central_kernel<kIdentity, true>, a, s, sms)
            : launch_ring(central_kernel<kIdentity, false>, a, s, sms);
}

int launch_decent(const DecentArgs& a, int codec, cudaStream_t s, int sms) {
  return codec == kU8 ? launch_ring(decent_kernel<kU8>, a, s, sms) : launch_ring(decent_kernel<kIdentity>, a, s, sms);
}

int max_persistent_grid() { return sm_count() * 4; }

}  // namespace b2
