// small_coll.cu -- latency path of D_LP_S / D_FP_S (collectives.cpp:229-288)
// for buckets that fit in the registers of one co-resident grid (the low end
// of BASELINE.json's D_LP_S sweep, 1M elements; the engine's 8 MiB buckets).
//
// The TMA-ring kernels (collectives.cu) pay a ring set-up, ~10 grid-wide
// barriers and several cross-GPU round trips per call, which is what a 1M
// bucket costs (47-51 us at g = 2/4).  Here every thread keeps its R float4
// groups of x in registers for the whole call and the ranks synchronise PER
// CTA: every rank launches the same grid over the same n, so CTA b owns the
// same elements on every rank.
//
//   1  load x (R float4 per thread), (min, max) per CTA -> partial
//   2  one grid barrier; every CTA reduces the partials (same order on every
//      CTA: the same header everywhere) -- uint8 only
//   3  wait until the neighbours that read this parity buffer two calls ago
//      acknowledged (dreads), quantize from registers into my window's
//      dbuf[p] (identity: the fp32 values), write the header dhdr[p] (every
//      CTA writes the same value, so whichever CTA a reader synchronises
//      with, the header is visible), fence, one relaxed red per neighbour on
//      its counter [me][b]
//   4  wait for every neighbour's counter [j][b] (cumulative: the number of
//      calls in which j sent to me), load the neighbours' codes of CTA b's
//      elements over NVLink, fold in ascending neighbour order in fp64 (the
//      self term from registers), times 1/|N| in fp64, round once, store x
//   5  acknowledge the reads: one red per neighbour on its dreads[p]
//
// One grid barrier, one cross-GPU hand-off per CTA; bit-exact like the ring
// kernels (same quantize / dequantize / fold arithmetic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "b2_host.h"
#include "collectives.cuh"

namespace b2 {
namespace {

namespace cg = cooperative_groups;

constexpr int kSmallThr = 256;
constexpr int kSmallMaxGrid = int(kSmallMaxGridD);  // per-source CTA counters (comm.cu gate_stride)

__device__ __forceinline__ WinHdr* whdr(uint8_t* w) { return reinterpret_cast<WinHdr*>(w); }

// NB > 0: the neighbourhood size is a compile-time constant (every remote load
// of a thread is issued before the fold: one NVLink round trip); NB = 0:
// runtime size, loads interleaved with the fold.
template <int CODEC, int R, int NB>
__global__ void __launch_bounds__(kSmallThr) decent_small_kernel(DecentArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ float2 wred[kSmallThr / 32];
  __shared__ int s_bad;
  const int me = a.me, p = a.parity, b = blockIdx.x;
  const size_t T = size_t(gridDim.x) * kSmallThr, gt = size_t(b) * kSmallThr + threadIdx.x;
  const size_t n = a.n, ng = n >> 2;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float4* x4 = reinterpret_cast<float4*>(a.x);
  WinHdr* mine = whdr(a.win[me]);
  if (threadIdx.x == 0) s_bad = 0;
  const Rounder rd = make_rounder(CODEC == kU8 && a.sr_on, a.sr_seed, me, 3);
  // phase stamps (b2_comm_enable_trace): start, header final, published, neighbours in, end
  unsigned long long* tr = a.trace ? a.trace + size_t(b) * kTraceSlots : nullptr;
  if (tr && threadIdx.x == 0) tr[kTrStart] = globaltimer();
  // ---- 1: x into registers
  float4 y[R];
  float yt[3] = {0.f, 0.f, 0.f};
  const bool tail = gt == T - 1 && (n & 3);
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  int bad = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const size_t g = gt + size_t(k) * T;
    if (g < ng) {
      y[k] = x4[g];
      lo = fmin_nan(lo, fmin_nan(fmin_nan(y[k].x, y[k].y), fmin_nan(y[k].z, y[k].w)));
      hi = fmax_nan(hi, fmax_nan(fmax_nan(y[k].x, y[k].y), fmax_nan(y[k].z, y[k].w)));
      if (CODEC != kU8 && a.check_finite)
        bad |= !(finite_f(y[k].x) && finite_f(y[k].y) && finite_f(y[k].z) && finite_f(y[k].w));
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      yt[e - 4 * ng] = a.x[e];
      lo = fmin_nan(lo, yt[e - 4 * ng]);
      hi = fmax_nan(hi, yt[e - 4 * ng]);
      if (CODEC != kU8 && a.check_finite) bad |= !finite_f(yt[e - 4 * ng]);
    }
  // ---- 2: the bucket's (min, max) (uint8: one encode of the whole bucket, collectives.cpp:266)
  U8Params q{};
  if (CODEC == kU8) {
    lo = warp_min_nan(lo);
    hi = warp_max_nan(hi);
    if (l == 0) wred[w] = make_float2(lo, hi);
    __syncthreads();
    if (threadIdx.x < 32) {
      const float2 v = l < kSmallThr / 32 ? wred[l] : wred[0];
      const float mn = warp_min_nan(v.x), mx = warp_max_nan(v.y);
      if (l == 0) a.partials[b] = make_float2(mn, mx);
    }
    grid.sync();
    lo = __int_as_float(0x7f800000);
    hi = -__int_as_float(0x7f800000);
    for (unsigned c = threadIdx.x; c < gridDim.x; c += kSmallThr) {
      const float2 v = __ldcg(a.partials + c);
      lo = fmin_nan(lo, v.x);
      hi = fmax_nan(hi, v.y);
    }
    lo = warp_min_nan(lo);
    hi = warp_max_nan(hi);
    __syncthreads();
    if (l == 0) wred[w] = make_float2(lo, hi);
    __syncthreads();
    const float2 v = l < kSmallThr / 32 ? wred[l] : wred[0];
    lo = warp_min_nan(v.x);
    hi = warp_max_nan(v.y);
    q = u8_params(lo, hi);
    if (gt == 0 && n && !(finite_f(lo) && finite_f(hi))) latch(a.status, kStatusNonFinite);
    if (tr && threadIdx.x == 0) tr[kTrP1FirstA] = globaltimer();
  }
  uint32_t c[R];
  uint8_t ct[3] = {0, 0, 0};
  if (CODEC == kU8) {
#pragma unroll
    for (int k = 0; k < R; ++k) c[k] = q4r(y[k], q.lo, q.inv, rd, 4 * (gt + size_t(k) * T));
    if (tail)
      for (size_t e = 4 * ng; e < n; ++e) ct[e - 4 * ng] = q1r(yt[e - 4 * ng], q.lo, q.inv, rd, e);
  }
  if (a.nnb == 1) {
    // ---- the neighbourhood is {self}: x' = (float)((0.0 + (double)D(Q(x))) * 1.0) = D(Q(x)) + 0.0f
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const size_t g = gt + size_t(k) * T;
      if (g < ng) {
        const float4 d = CODEC == kU8 ? dequant4(c[k], q) : y[k];
        x4[g] = make_float4(__fadd_rn(d.x, 0.0f), __fadd_rn(d.y, 0.0f), __fadd_rn(d.z, 0.0f), __fadd_rn(d.w, 0.0f));
      }
    }
    if (tail)
      for (size_t e = 4 * ng; e < n; ++e)
        a.x[e] = __fadd_rn(CODEC == kU8 ? dequant1(ct[e - 4 * ng], q) : yt[e - 4 * ng], 0.0f);
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_bad) latch(a.status, kStatusNonFinite);
      fail_epilogue(a.status);
    }
    return;
  }
  // ---- 3: publish my contribution of CTA b's elements
  if (threadIdx.x == 0 && a.expected_reads)
    wait_geq(&mine->dreads[p], a.expected_reads * gridDim.x, a.timeout_ns, a.status);
  __syncthreads();
  uint8_t* mybuf = a.win[me] + a.off_dbuf;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const size_t g = gt + size_t(k) * T;
    if (g < ng) {
      if (CODEC == kU8)
        reinterpret_cast<uint32_t*>(mybuf)[g] = c[k];
      else
        reinterpret_cast<float4*>(mybuf)[g] = y[k];
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      if (CODEC == kU8)
        mybuf[e] = ct[e - 4 * ng];
      else
        reinterpret_cast<float*>(mybuf)[e] = yt[e - 4 * ng];
    }
  if (CODEC == kU8 && threadIdx.x == 0) mine->dhdr[p] = make_float2(lo, hi);
  __syncthreads();
  if (threadIdx.x < a.nnb && a.nbrs[threadIdx.x] != me) {
    // the CTA's stores (ordered by bar.sync) before the signal; peers read
    // this buffer through this GPU's L2, so gpu scope suffices for the data
    __threadfence();
    red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[a.nbrs[threadIdx.x]] + a.off_gate) +
                            size_t(me) * a.gate_stride + b,
                        1ull);
  }
  if (tr && threadIdx.x == 0) tr[kTrP1Done] = globaltimer();
  // ---- 4: wait for every neighbour's CTA b, fold in ascending neighbour order
  __shared__ SrcDecS s_dec[kMaxRanks];
  if (threadIdx.x < a.nnb) {
    const int j = a.nbrs[threadIdx.x];
    if (j != me)
      wait_geq(reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate) + size_t(j) * a.gate_stride + b,
               a.sends[threadIdx.x], a.timeout_ns, a.status);
    if (CODEC == kU8) {
      const float2 h = j == me ? make_float2(lo, hi) : __ldcg(&whdr(a.win[j])->dhdr[p]);
      const U8Params qj = u8_params(h.x, h.y);
      s_dec[threadIdx.x] = SrcDecS{qj.lo, qj.step, qj.c23, qj.fastdec ? 1 : 0};
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[kTrP2Ready] = globaltimer();
  const double inv = a.inv;
  constexpr int NBX = NB > 0 ? NB : 1;
  const int nnb = NB > 0 ? NB : a.nnb;
  // NB > 0: every remote load of this thread first (one NVLink round trip)
  uint32_t rc[R][NBX];
  float4 rf[CODEC == kU8 ? 1 : R][CODEC == kU8 ? 1 : NBX];
  if (NB > 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const size_t g = gt + size_t(k) * T;
#pragma unroll
      for (int i = 0; i < NBX; ++i) {
        const int j = a.nbrs[i];
        if (g < ng && j != me) {
          if (CODEC == kU8)
            rc[k][i] = __ldcg(reinterpret_cast<const uint32_t*>(a.win[j] + a.off_dbuf) + g);
          else
            rf[CODEC == kU8 ? 0 : k][CODEC == kU8 ? 0 : i] =
                __ldcg(reinterpret_cast<const float4*>(a.win[j] + a.off_dbuf) + g);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const size_t g = gt + size_t(k) * T;
    if (g < ng) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int i = 0; i < (NB > 0 ? NBX : kMaxRanks); ++i) {
        if (NB == 0 && i >= nnb) break;
        const int j = a.nbrs[i];
        float4 d;
        if (CODEC == kU8) {
          const uint32_t cj = j == me ? c[k]
                              : NB > 0 ? rc[k][NB > 0 ? i : 0]
                                       : __ldcg(reinterpret_cast<const uint32_t*>(a.win[j] + a.off_dbuf) + g);
          const SrcDecS sd = s_dec[i];
          d = sd.fast ? dequant4_fast(cj, sd.lo, sd.step, sd.c23) : dequant4(cj, sd.lo, sd.step);
        } else {
          d = j == me ? y[k]
              : NB > 0 ? rf[CODEC == kU8 ? 0 : k][CODEC == kU8 ? 0 : (NB > 0 ? i : 0)]
                       : __ldcg(reinterpret_cast<const float4*>(a.win[j] + a.off_dbuf) + g);
        }
        a0 = __dadd_rn(a0, double(d.x));
        a1 = __dadd_rn(a1, double(d.y));
        a2 = __dadd_rn(a2, double(d.z));
        a3 = __dadd_rn(a3, double(d.w));
      }
      x4[g] = make_float4(__double2float_rn(__dmul_rn(a0, inv)), __double2float_rn(__dmul_rn(a1, inv)),
                          __double2float_rn(__dmul_rn(a2, inv)), __double2float_rn(__dmul_rn(a3, inv)));
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      double acc = 0.0;
      for (int i = 0; i < a.nnb; ++i) {
        const int j = a.nbrs[i];
        float d;
        if (CODEC == kU8) {
          const uint8_t cj = j == me ? ct[e - 4 * ng] : __ldcg(a.win[j] + a.off_dbuf + e);
          d = dequant1(cj, s_dec[i].lo, s_dec[i].step);
        } else {
          d = j == me ? yt[e - 4 * ng] : __ldcg(reinterpret_cast<const float*>(a.win[j] + a.off_dbuf) + e);
        }
        acc = __dadd_rn(acc, double(d));
      }
      a.x[e] = __double2float_rn(__dmul_rn(acc, inv));
    }
  // ---- 5: my reads of CTA b's elements are done: acknowledge to every neighbour
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x < a.nnb && a.nbrs[threadIdx.x] != me)  // every remote load of the CTA was consumed above
    red_relaxed_sys_add(&whdr(a.win[a.nbrs[threadIdx.x]])->dreads[p], 1ull);
  if (threadIdx.x == 0) {
    if (s_bad) latch(a.status, kStatusNonFinite);
    fail_epilogue(a.status);
    if (tr) tr[kTrEnd] = globaltimer();
  }
}

// Buckets beyond the register capacity (4M-25M elements): the same per-CTA
// protocol, streaming -- x is read for the (min, max), again (from L2) to
// quantize into my window, and my own codes are re-read for the self term.
template <int CODEC>
__global__ void __launch_bounds__(kSmallThr) decent_stream_kernel(DecentArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ float2 wred[kSmallThr / 32];
  __shared__ int s_bad;
  __shared__ SrcDecS s_dec[kMaxRanks];
  const int me = a.me, p = a.parity, b = blockIdx.x;
  const size_t T = size_t(gridDim.x) * kSmallThr, gt = size_t(b) * kSmallThr + threadIdx.x;
  const size_t n = a.n, ng = n >> 2;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  float4* x4 = reinterpret_cast<float4*>(a.x);
  WinHdr* mine = whdr(a.win[me]);
  uint8_t* mybuf = a.win[me] + a.off_dbuf;
  if (threadIdx.x == 0) s_bad = 0;
  const Rounder rd = make_rounder(CODEC == kU8 && a.sr_on, a.sr_seed, me, 3);
  unsigned long long* tr = a.trace ? a.trace + size_t(b) * kTraceSlots : nullptr;
  if (tr && threadIdx.x == 0) tr[kTrStart] = globaltimer();
  const bool tail = gt == T - 1 && (n & 3);
  int bad = 0;
  U8Params q{};
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  if (CODEC == kU8) {  // ---- 1-2: the bucket's (min, max), collectives.cpp:266
    for (size_t g = gt; g < ng; g += T) {
      const float4 v = __ldcg(x4 + g);
      lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
      hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
    }
    if (tail)
      for (size_t e = 4 * ng; e < n; ++e) {
        lo = fmin_nan(lo, a.x[e]);
        hi = fmax_nan(hi, a.x[e]);
      }
    lo = warp_min_nan(lo);
    hi = warp_max_nan(hi);
    if (l == 0) wred[w] = make_float2(lo, hi);
    __syncthreads();
    if (threadIdx.x < 32) {
      const float2 v = l < kSmallThr / 32 ? wred[l] : wred[0];
      const float mn = warp_min_nan(v.x), mx = warp_max_nan(v.y);
      if (l == 0) a.partials[b] = make_float2(mn, mx);
    }
    grid.sync();
    lo = __int_as_float(0x7f800000);
    hi = -__int_as_float(0x7f800000);
    for (unsigned c = threadIdx.x; c < gridDim.x; c += kSmallThr) {
      const float2 v = __ldcg(a.partials + c);
      lo = fmin_nan(lo, v.x);
      hi = fmax_nan(hi, v.y);
    }
    lo = warp_min_nan(lo);
    hi = warp_max_nan(hi);
    __syncthreads();
    if (l == 0) wred[w] = make_float2(lo, hi);
    __syncthreads();
    const float2 v = l < kSmallThr / 32 ? wred[l] : wred[0];
    lo = warp_min_nan(v.x);
    hi = warp_max_nan(v.y);
    q = u8_params(lo, hi);
    if (gt == 0 && n && !(finite_f(lo) && finite_f(hi))) latch(a.status, kStatusNonFinite);
    if (tr && threadIdx.x == 0) tr[kTrP1FirstA] = globaltimer();
  }
  if (a.nnb == 1) {  // {self}: x' = D(Q(x)) + 0.0f (identity: x + 0.0f)
    for (size_t g = gt; g < ng; g += T) {
      const float4 v = x4[g];
      if (CODEC != kU8 && a.check_finite) bad |= !(finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w));
      const float4 d = CODEC == kU8 ? dequant4(q4r(v, q.lo, q.inv, rd, 4 * g), q) : v;
      x4[g] = make_float4(__fadd_rn(d.x, 0.0f), __fadd_rn(d.y, 0.0f), __fadd_rn(d.z, 0.0f), __fadd_rn(d.w, 0.0f));
    }
    if (tail)
      for (size_t e = 4 * ng; e < n; ++e) {
        if (CODEC != kU8 && a.check_finite) bad |= !finite_f(a.x[e]);
        a.x[e] = __fadd_rn(CODEC == kU8 ? dequant1(q1r(a.x[e], q.lo, q.inv, rd, e), q) : a.x[e], 0.0f);
      }
    if (bad) atomicOr(&s_bad, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_bad) latch(a.status, kStatusNonFinite);
      fail_epilogue(a.status);
    }
    return;
  }
  // ---- 3: publish CTA b's elements
  if (threadIdx.x == 0 && a.expected_reads)
    wait_geq(&mine->dreads[p], a.expected_reads * gridDim.x, a.timeout_ns, a.status);
  __syncthreads();
  for (size_t g = gt; g < ng; g += T) {
    const float4 v = x4[g];
    if (CODEC == kU8) {
      reinterpret_cast<uint32_t*>(mybuf)[g] = q4r(v, q.lo, q.inv, rd, 4 * g);
    } else {
      reinterpret_cast<float4*>(mybuf)[g] = v;
      if (a.check_finite) bad |= !(finite_f(v.x) && finite_f(v.y) && finite_f(v.z) && finite_f(v.w));
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      if (CODEC == kU8) {
        mybuf[e] = q1r(a.x[e], q.lo, q.inv, rd, e);
      } else {
        reinterpret_cast<float*>(mybuf)[e] = a.x[e];
        if (a.check_finite) bad |= !finite_f(a.x[e]);
      }
    }
  if (CODEC == kU8 && threadIdx.x == 0) mine->dhdr[p] = make_float2(lo, hi);
  __syncthreads();
  if (threadIdx.x < a.nnb && a.nbrs[threadIdx.x] != me) {
    __threadfence();  // peers read this buffer through this GPU's L2
    red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[a.nbrs[threadIdx.x]] + a.off_gate) +
                            size_t(me) * a.gate_stride + b,
                        1ull);
  }
  if (tr && threadIdx.x == 0) tr[kTrP1Done] = globaltimer();
  // ---- 4: every neighbour's CTA b in, fold in ascending neighbour order
  if (threadIdx.x < a.nnb) {
    const int j = a.nbrs[threadIdx.x];
    if (j != me)
      wait_geq(reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_gate) + size_t(j) * a.gate_stride + b,
               a.sends[threadIdx.x], a.timeout_ns, a.status);
    if (CODEC == kU8) {
      const float2 h = j == me ? make_float2(lo, hi) : __ldcg(&whdr(a.win[j])->dhdr[p]);
      const U8Params qj = u8_params(h.x, h.y);
      s_dec[threadIdx.x] = SrcDecS{qj.lo, qj.step, qj.c23, qj.fastdec ? 1 : 0};
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[kTrP2Ready] = globaltimer();
  const double inv = a.inv;
  const int nnb = a.nnb;
  // U groups per iteration: every load of the U groups first (one NVLink
  // round trip per U groups, not per group), then the folds
  constexpr int U = CODEC == kU8 ? 4 : 2;
  for (size_t g0 = gt; g0 < ng; g0 += U * T) {
    uint32_t cw[U][kMaxRanks];
    float4 fw[CODEC == kU8 ? 1 : U][CODEC == kU8 ? 1 : kMaxRanks];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t g = g0 + size_t(u) * T;
#pragma unroll
      for (int i = 0; i < kMaxRanks; ++i)
        if (i < nnb && g < ng) {
          const uint8_t* src = a.win[a.nbrs[i]] + a.off_dbuf;
          if (CODEC == kU8)
            cw[u][i] = __ldcg(reinterpret_cast<const uint32_t*>(src) + g);
          else
            fw[CODEC == kU8 ? 0 : u][CODEC == kU8 ? 0 : i] = __ldcg(reinterpret_cast<const float4*>(src) + g);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t g = g0 + size_t(u) * T;
      if (g >= ng) break;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
      for (int i = 0; i < kMaxRanks; ++i)
        if (i < nnb) {
          float4 d;
          if (CODEC == kU8) {
            const SrcDecS sd = s_dec[i];
            d = sd.fast ? dequant4_fast(cw[u][i], sd.lo, sd.step, sd.c23) : dequant4(cw[u][i], sd.lo, sd.step);
          } else {
            d = fw[CODEC == kU8 ? 0 : u][CODEC == kU8 ? 0 : i];
          }
          a0 = __dadd_rn(a0, double(d.x));
          a1 = __dadd_rn(a1, double(d.y));
          a2 = __dadd_rn(a2, double(d.z));
          a3 = __dadd_rn(a3, double(d.w));
        }
      __stcs(x4 + g, make_float4(__double2float_rn(__dmul_rn(a0, inv)), __double2float_rn(__dmul_rn(a1, inv)),
                                 __double2float_rn(__dmul_rn(a2, inv)), __double2float_rn(__dmul_rn(a3, inv))));
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      double acc = 0.0;
      for (int i = 0; i < nnb; ++i) {
        const uint8_t* src = a.win[a.nbrs[i]] + a.off_dbuf;
        const float d = CODEC == kU8 ? dequant1(__ldcg(src + e), s_dec[i].lo, s_dec[i].step)
                                     : __ldcg(reinterpret_cast<const float*>(src) + e);
        acc = __dadd_rn(acc, double(d));
      }
      a.x[e] = __double2float_rn(__dmul_rn(acc, inv));
    }
  // ---- 5: acknowledge the reads
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x < a.nnb && a.nbrs[threadIdx.x] != me)
    red_relaxed_sys_add(&whdr(a.win[a.nbrs[threadIdx.x]])->dreads[p], 1ull);
  if (threadIdx.x == 0) {
    if (s_bad) latch(a.status, kStatusNonFinite);
    fail_epilogue(a.status);
    if (tr) tr[kTrEnd] = globaltimer();
  }
}

template <int CODEC>
int try_stream(const DecentArgs& a, cudaStream_t s, int sms) {
  const void* fn = reinterpret_cast<const void*>(decent_stream_kernel<CODEC>);
  const int per_sm = occupancy(fn, kSmallThr);
  if (per_sm < 1) return B2_ERR_UNSUPPORTED;
  const int nsm = sms > 0 && sms < sm_count() ? sms : sm_count();
  const int grid = std::min(nsm * per_sm, kSmallMaxGrid);
  DecentArgs copy = a;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSmallThr), params, 0, s));
  return B2_OK;
}

template <int CODEC, int R>
int try_small(const DecentArgs& a, cudaStream_t s, int sms) {
  const void* fn = a.nnb == 2   ? reinterpret_cast<const void*>(decent_small_kernel<CODEC, R, 2>)
                   : a.nnb == 3 ? reinterpret_cast<const void*>(decent_small_kernel<CODEC, R, 3>)
                                : reinterpret_cast<const void*>(decent_small_kernel<CODEC, R, 0>);
  const int per_sm = occupancy(fn, kSmallThr);
  const int nsm = sms > 0 && sms < sm_count() ? sms : sm_count();
  const size_t cap = size_t(nsm) * size_t(per_sm > 0 ? per_sm : 0);
  const size_t per_block = size_t(kSmallThr) * R, ng = a.n >> 2;
  const size_t need = (ng + per_block - 1) / per_block;
  if (per_sm < 1 || need > cap || cap == 0) return B2_ERR_UNSUPPORTED;
  // one CTA per SM at least (spread the loads); the grid is a function of
  // (n, SM count, budget, occupancy) only, so every rank launches the same
  const int grid = int(std::min<size_t>(std::min<size_t>(cap, std::max<size_t>(need, size_t(nsm))),
                                        size_t(kSmallMaxGrid)));
  if (size_t(grid) * per_block < ng) return B2_ERR_UNSUPPORTED;
  DecentArgs copy = a;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kSmallThr), params, 0, s));
  return B2_OK;
}

template <int CODEC>
int small_decent(const DecentArgs& a, cudaStream_t s, int sms) {
  int rc = try_small<CODEC, 2>(a, s, sms);
  if (rc == B2_ERR_UNSUPPORTED) rc = try_small<CODEC, 4>(a, s, sms);
  if (rc == B2_ERR_UNSUPPORTED) rc = try_small<CODEC, 8>(a, s, sms);
  if (rc == B2_ERR_UNSUPPORTED) rc = try_stream<CODEC>(a, s, sms);
  return rc;
}

}  // namespace

// D_* latency path; B2_ERR_UNSUPPORTED when the bucket exceeds its capacity
// (the caller then takes the TMA-ring kernel).  The choice depends only on
// (n, SM count, budget), so all ranks of a window take the same path.
int launch_decent_small(const DecentArgs& a, int codec, cudaStream_t s, int sms) {
  static const size_t limit = [] {  // B2_SMALL_MAX=<elements> moves the cut-over (A/B runs)
    const char* e = getenv("B2_SMALL_MAX");
    return e ? size_t(std::strtoull(e, nullptr, 10)) : kSmallDecentMax;
  }();
  if (a.n > limit) return B2_ERR_UNSUPPORTED;
  return codec == kU8 ? small_decent<kU8>(a, s, sms) : small_decent<kIdentity>(a, s, sms);
}

}  // namespace b2
