// collectives.cu -- fused single-launch kernels for the four synchronous
// primitives over NVLink/NVSwitch peer memory.
//
//   central_kernel<CODEC,EC>   C_LP_S (uint8 / identity, +/- error feedback)
//                              and C_FP_S (identity, no finiteness check)
//                              = scatter_reduce_lp / scatter_reduce_fp,
//                              collectives.cpp:42-163
//   decent_kernel<CODEC>       D_LP_S / D_FP_S, collectives.cpp:229-288
//
// One cooperative persistent launch per call (grid = SMs x resident CTAs).
//
// C_* dataflow per rank `me` (g ranks, partition k = partition_range(N,g,k)):
//   phase 1  encode chunk k for k = me+1, me+2, ..., me (own chunk last: the
//            staggered order makes the NVLink traffic a permutation at every
//            instant) and PUSH the codes straight into owner k's window
//            (remote 32-bit stores, one coalesced 128-B line per warp store),
//            so the NVLink scatter overlaps the HBM-bound encode.  uint8 needs
//            the chunk-global (min,max) first: pass A (min/max) of chunk k+1
//            runs in the same grid segment as pass B (quantize+push) of chunk
//            k, one grid barrier per chunk, and pass B re-reads the chunk from
//            L2 (a 100M/8 chunk is 50 MB).  After each chunk every CTA fences
//            at system scope and the last CTA bumps owner k's arrive1 counter.
//   phase 2  owner: wait arrive1 == g*epoch, fold the g decoded contributions
//            from its LOCAL window in ascending rank order in fp64 (kernels.cpp
//            add_f64), round once, second (min,max) + quantize; decode its
//            own payload straight into x; publish ready2 = epoch.
//   phase 3  PULL every other owner's phase-2 payload over NVLink (peer
//            loads), decode into x.  Owners are visited in staggered order.
//
// D_* dataflow: encode (or stage) the whole bucket into my window's parity
// buffer, publish dready, then pull the neighbours' buffers, fold in
// ascending neighbour order in fp64, multiply by 1/|N| in fp64, round once.
// Overwriting a parity buffer waits until every neighbour has acknowledged
// reading it (dreads), so no rank can clobber data a slow neighbour still
// reads.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "b2_host.h"
#include "collectives.cuh"

namespace b2 {
namespace cg = cooperative_groups;

namespace {

constexpr int UX = 4;  // x passes: 4 x float4 in flight per thread
constexpr int UR = 2;  // reduce passes: 2 groups x g sources in flight

__device__ __forceinline__ void part_range(size_t n, int g, int k, size_t& lo, size_t& sz) {
  const size_t base = n / size_t(g), extra = n % size_t(g), uk = size_t(k);
  lo = uk * base + (uk < extra ? uk : extra);
  sz = base + (uk < extra ? 1 : 0);
}

__device__ __forceinline__ float2 reduce_partials(const float2* p, int G, float2* smem) {
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  for (int i = threadIdx.x; i < G; i += blockDim.x) {
    const float2 v = __ldcg(p + i);
    lo = fmin_nan(lo, v.x);
    hi = fmax_nan(hi, v.y);
  }
  return block_minmax(lo, hi, smem);
}

// Head/tail scalar slot: thread t < 8 of the last CTA handles element
// head[t] (t < 4) or tail[t-4]; returns false when there is no such element.
__device__ __forceinline__ bool edge_elem(const Span& sp, size_t& e) {
  if (blockIdx.x != gridDim.x - 1 || threadIdx.x >= 8) return false;
  if (threadIdx.x < 4) {
    e = sp.s + threadIdx.x;
    return e < sp.head_end;
  }
  e = sp.tail_begin + (threadIdx.x - 4);
  return e < sp.s + sp.n;
}

// (min, max) of y = x (- delta) over sp, reduced over the CTA.
template <bool EC>
__device__ float2 minmax_span(const float* x, const float* delta, const Span& sp, float2* red) {
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* d4 = reinterpret_cast<const float4*>(delta);
  for (size_t base = sp.g0 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; base < sp.g1;
       base += stride * UX) {
    float4 v[UX];
#pragma unroll
    for (int u = 0; u < UX; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) {
        v[u] = __ldcg(x4 + gi);
        if (EC) v[u] = sub4(v[u], __ldcg(d4 + gi));
      }
    }
#pragma unroll
    for (int u = 0; u < UX; ++u) {
      if (base + u * stride < sp.g1) {
        lo = fmin_nan(lo, fmin_nan(fmin_nan(v[u].x, v[u].y), fmin_nan(v[u].z, v[u].w)));
        hi = fmax_nan(hi, fmax_nan(fmax_nan(v[u].x, v[u].y), fmax_nan(v[u].z, v[u].w)));
      }
    }
  }
  size_t e;
  if (edge_elem(sp, e)) {
    float v = x[e];
    if (EC) v = __fsub_rn(v, delta[e]);
    lo = fmin_nan(lo, v);
    hi = fmax_nan(hi, v);
  }
  return block_minmax(lo, hi, red);
}

// Fence this CTA's writes at system scope; the last CTA to arrive (of G)
// resets the counter and returns true.
__device__ __forceinline__ bool cta_arrive(unsigned* ctr) {
  __threadfence_system();
  __syncthreads();
  __shared__ int last;
  if (threadIdx.x == 0) {
    const unsigned old = atomicAdd(ctr, 1u);
    last = (old == gridDim.x - 1);
    if (last) {
      atomicExch(ctr, 0u);
      __threadfence_system();
    }
  }
  __syncthreads();
  return last != 0;
}

__device__ __forceinline__ WinHdr* hdr_of(uint8_t* w) { return reinterpret_cast<WinHdr*>(w); }

// ------------------------------------------------------------ C_* kernel
template <int CODEC, bool EC>
__global__ void __launch_bounds__(kThreads) central_kernel(CentralArgs a) {
  __shared__ float2 red[32];
  __shared__ float s_lo[kMaxRanks], s_step[kMaxRanks];
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, g = a.g, me = a.me;
  const size_t stride = size_t(G) * blockDim.x;
  const size_t t0 = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr size_t W = CODEC == kU8 ? 1 : 4;  // wire bytes per element
  int bad = 0;                                // identity: non-finite seen

  // ------------------------------------------------ phase 1: encode + push
  if (CODEC == kU8) {
    size_t lo, sz;
    part_range(a.n, g, (me + 1) % g, lo, sz);
    const float2 r = minmax_span<EC>(a.x, a.delta, make_span(lo, sz), red);
    if (threadIdx.x == 0) a.partials[size_t((me + 1) % g) * G + blockIdx.x] = r;
    grid.sync();
  }
  for (int i = 0; i < g; ++i) {
    const int k = (me + 1 + i) % g;
    size_t lo, sz;
    part_range(a.n, g, k, lo, sz);
    const Span sp = make_span(lo, sz);
    uint8_t* dst = a.win[k] + a.off_recv1 + size_t(me) * a.slot_stride;
    const size_t gbase = lo >> 2;          // slot index of group gi = gi - gbase
    const size_t ebase = lo & ~size_t(3);  // slot index of element e = e - ebase
    if (CODEC == kU8) {
      const float2 mm = reduce_partials(a.partials + size_t(k) * G, G, red);
      const U8Params p = u8_params(mm.x, mm.y);
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr_of(a.win[k])->hdr1[me] = mm;  // remote 8-byte store into owner k's header
        if (sz && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
      }
      uint32_t* d32 = reinterpret_cast<uint32_t*>(dst);
      const float4* x4 = reinterpret_cast<const float4*>(a.x);
      float4* dl4 = reinterpret_cast<float4*>(a.delta);
      for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
        float4 v[UX];
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) {
            v[u] = __ldcs(x4 + gi);
            if (EC) v[u] = sub4(v[u], dl4[gi]);
          }
        }
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) {
            const uint32_t q = quantize4(v[u], p.lo, p.inv);
            d32[gi - gbase] = q;
            if (EC) dl4[gi] = sub4(v[u], dequant4(q, p.lo, p.step));
          }
        }
      }
      size_t e;
      if (edge_elem(sp, e)) {
        float v = a.x[e];
        if (EC) v = __fsub_rn(v, a.delta[e]);
        const uint8_t q = quantize1(v, p.lo, p.inv);
        dst[e - ebase] = q;
        if (EC) a.delta[e] = __fsub_rn(v, dequant1(q, p.lo, p.step));
      }
      if (i + 1 < g) {  // pass A of the next chunk shares this grid segment
        const int kn = (me + 2 + i) % g;
        size_t lo2, sz2;
        part_range(a.n, g, kn, lo2, sz2);
        const float2 r = minmax_span<EC>(a.x, a.delta, make_span(lo2, sz2), red);
        if (threadIdx.x == 0) a.partials[size_t(kn) * G + blockIdx.x] = r;
      }
    } else {  // identity: y = x (- delta) travels as fp32
      float4* d4 = reinterpret_cast<float4*>(dst);
      const float4* x4 = reinterpret_cast<const float4*>(a.x);
      float4* dl4 = reinterpret_cast<float4*>(a.delta);
      for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
        float4 v[UX];
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) {
            v[u] = __ldcs(x4 + gi);
            if (EC) v[u] = sub4(v[u], dl4[gi]);
          }
        }
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) {
            d4[gi - gbase] = v[u];
            if (a.check_finite)
              bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) && finite_f(v[u].w));
            if (EC) dl4[gi] = sub4(v[u], v[u]);
          }
        }
      }
      size_t e;
      if (edge_elem(sp, e)) {
        float v = a.x[e];
        if (EC) v = __fsub_rn(v, a.delta[e]);
        reinterpret_cast<float*>(dst)[e - ebase] = v;
        if (a.check_finite) bad |= !finite_f(v);
        if (EC) a.delta[e] = __fsub_rn(v, v);
      }
    }
    if (cta_arrive(a.cta_done + k)) red_release_sys_add(&hdr_of(a.win[k])->arrive1, 1ull);
    if (CODEC == kU8 && i + 1 < g) grid.sync();
  }

  // ------------------------------------------------ phase 2: owner reduce
  size_t mlo, msz;
  part_range(a.n, g, me, mlo, msz);
  const Span ms = make_span(mlo, msz);
  const size_t mg = mlo >> 2, me_e = mlo & ~size_t(3);
  WinHdr* mine = hdr_of(a.win[me]);
  if (threadIdx.x == 0)
    wait_geq(&mine->arrive1, (unsigned long long)g * a.epoch, a.timeout_ns, a.status);
  __syncthreads();
  const uint8_t* recv = a.win[me] + a.off_recv1;
  if (CODEC == kU8) {
    if (threadIdx.x < g) {
      const float2 h = __ldcg(&mine->hdr1[threadIdx.x]);
      s_lo[threadIdx.x] = h.x;
      s_step[threadIdx.x] = __fdiv_rn(__fsub_rn(h.y, h.x), 255.0f);
    }
    __syncthreads();
  }
  // fold of the g contributions for one aligned group (slot index gs)
  auto fold4 = [&](size_t gs) -> float4 {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int j = 0; j < g; ++j) {
      float4 d;
      if (CODEC == kU8) {
        const uint32_t c = __ldcg(reinterpret_cast<const uint32_t*>(recv + size_t(j) * a.slot_stride) + gs);
        d = dequant4(c, s_lo[j], s_step[j]);
      } else {
        d = __ldcg(reinterpret_cast<const float4*>(recv + size_t(j) * a.slot_stride) + gs);
      }
      a0 = __dadd_rn(a0, double(d.x));
      a1 = __dadd_rn(a1, double(d.y));
      a2 = __dadd_rn(a2, double(d.z));
      a3 = __dadd_rn(a3, double(d.w));
    }
    return make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2),
                       __double2float_rn(a3));
  };
  auto fold1 = [&](size_t es) -> float {
    double acc = 0.0;
    for (int j = 0; j < g; ++j) {
      float d;
      if (CODEC == kU8)
        d = dequant1((recv + size_t(j) * a.slot_stride)[es], s_lo[j], s_step[j]);
      else
        d = reinterpret_cast<const float*>(recv + size_t(j) * a.slot_stride)[es];
      acc = __dadd_rn(acc, double(d));
    }
    return __double2float_rn(acc);
  };
  auto eps4 = [&](size_t gi) -> float4 {  // epsilon is owned-length, unaligned
    const float* ep = a.eps + (4 * gi - mlo);
    return make_float4(ep[0], ep[1], ep[2], ep[3]);
  };
  auto set_eps4 = [&](size_t gi, float4 v) {
    float* ep = a.eps + (4 * gi - mlo);
    ep[0] = v.x;
    ep[1] = v.y;
    ep[2] = v.z;
    ep[3] = v.w;
  };
  float4* x4 = reinterpret_cast<float4*>(a.x);
  uint8_t* out2 = a.win[me] + a.off_out2;

  if (CODEC == kU8) {
    // pass 2A: y2 = (float)sum - eps ; (min, max) ; cache y2 when scratch
    float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
    float4* sc4 = reinterpret_cast<float4*>(a.scratch);
    for (size_t base = ms.g0 + t0; base < ms.g1; base += stride * UR) {
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const size_t gi = base + u * stride;
        if (gi < ms.g1) {
          float4 y = fold4(gi - mg);
          if (EC) y = sub4(y, eps4(gi));
          if (a.scratch) sc4[gi - mg] = y;
          lo = fmin_nan(lo, fmin_nan(fmin_nan(y.x, y.y), fmin_nan(y.z, y.w)));
          hi = fmax_nan(hi, fmax_nan(fmax_nan(y.x, y.y), fmax_nan(y.z, y.w)));
        }
      }
    }
    size_t e;
    if (edge_elem(ms, e)) {
      float y = fold1(e - me_e);
      if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
      if (a.scratch) a.scratch[e - me_e] = y;
      lo = fmin_nan(lo, y);
      hi = fmax_nan(hi, y);
    }
    const float2 r = block_minmax(lo, hi, red);
    if (threadIdx.x == 0) a.partials[size_t(g) * G + blockIdx.x] = r;
    grid.sync();
    // pass 2B: second Q, own payload decoded straight into x
    const float2 mm = reduce_partials(a.partials + size_t(g) * G, G, red);
    const U8Params p = u8_params(mm.x, mm.y);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      mine->hdr2 = mm;
      if (msz && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
    }
    uint32_t* o32 = reinterpret_cast<uint32_t*>(out2);
    for (size_t base = ms.g0 + t0; base < ms.g1; base += stride * UR) {
      float4 y[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const size_t gi = base + u * stride;
        if (gi < ms.g1) {
          if (a.scratch) {
            y[u] = __ldcg(sc4 + (gi - mg));
          } else {
            y[u] = fold4(gi - mg);
            if (EC) y[u] = sub4(y[u], eps4(gi));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const size_t gi = base + u * stride;
        if (gi < ms.g1) {
          const uint32_t q = quantize4(y[u], p.lo, p.inv);
          if (g > 1) o32[gi - mg] = q;
          const float4 d = dequant4(q, p.lo, p.step);
          __stcs(x4 + gi, d);
          if (EC) set_eps4(gi, sub4(y[u], d));
        }
      }
    }
    if (edge_elem(ms, e)) {
      float y;
      if (a.scratch) {
        y = a.scratch[e - me_e];
      } else {
        y = fold1(e - me_e);
        if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
      }
      const uint8_t q = quantize1(y, p.lo, p.inv);
      if (g > 1) out2[e - me_e] = q;
      const float d = dequant1(q, p.lo, p.step);
      a.x[e] = d;
      if (EC) a.eps[e - mlo] = __fsub_rn(y, d);
    }
  } else {
    // identity / full precision: the fold IS the result
    float4* o4 = reinterpret_cast<float4*>(out2);
    for (size_t base = ms.g0 + t0; base < ms.g1; base += stride * UR) {
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const size_t gi = base + u * stride;
        if (gi < ms.g1) {
          float4 y = fold4(gi - mg);
          if (EC) y = sub4(y, eps4(gi));
          if (a.check_finite)
            bad |= !(finite_f(y.x) && finite_f(y.y) && finite_f(y.z) && finite_f(y.w));
          if (EC) set_eps4(gi, sub4(y, y));
          if (g > 1) o4[gi - mg] = y;
          __stcs(x4 + gi, y);
        }
      }
    }
    size_t e;
    if (edge_elem(ms, e)) {
      float y = fold1(e - me_e);
      if (EC) y = __fsub_rn(y, a.eps[e - mlo]);
      if (a.check_finite) bad |= !finite_f(y);
      if (EC) a.eps[e - mlo] = __fsub_rn(y, y);
      if (g > 1) reinterpret_cast<float*>(out2)[e - me_e] = y;
      a.x[e] = y;
    }
  }
  if (bad) latch(a.status, kStatusNonFinite);
  if (g == 1) return;
  if (cta_arrive(a.cta_done + kMaxRanks)) st_release_sys(&mine->ready2, a.epoch);

  // ------------------------------------------------ phase 3: pull + decode
  for (int i = 0; i + 1 < g; ++i) {
    const int k = (me + 1 + i) % g;
    size_t lo, sz;
    part_range(a.n, g, k, lo, sz);
    const Span sp = make_span(lo, sz);
    const size_t gbase = lo >> 2, ebase = lo & ~size_t(3);
    WinHdr* hk = hdr_of(a.win[k]);
    if (threadIdx.x == 0) wait_geq(&hk->ready2, a.epoch, a.timeout_ns, a.status);
    __syncthreads();
    const uint8_t* src = a.win[k] + a.off_out2;
    if (CODEC == kU8) {
      const float2 h = ld_peer_f2(&hk->hdr2);
      const float lo8 = h.x, step = __fdiv_rn(__fsub_rn(h.y, h.x), 255.0f);
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(src);
      for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
        uint32_t c[UX];
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          c[u] = gi < sp.g1 ? ld_peer_u32(s32 + (gi - gbase)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) __stcs(x4 + gi, dequant4(c[u], lo8, step));
        }
      }
      size_t e;
      if (edge_elem(sp, e)) a.x[e] = dequant1(__ldcg(src + (e - ebase)), lo8, step);
    } else {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
        float4 c[UX];
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) c[u] = ld_peer_f4(s4 + (gi - gbase));
        }
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const size_t gi = base + u * stride;
          if (gi < sp.g1) __stcs(x4 + gi, c[u]);
        }
      }
      size_t e;
      if (edge_elem(sp, e)) a.x[e] = __ldcg(reinterpret_cast<const float*>(src) + (e - ebase));
    }
  }
}

// ------------------------------------------------------------ D_* kernel
template <int CODEC>
__global__ void __launch_bounds__(kThreads) decent_kernel(DecentArgs a) {
  __shared__ float2 red[32];
  __shared__ float s_lo[kMaxRanks], s_step[kMaxRanks];
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, me = a.me, p = a.parity;
  const size_t stride = size_t(G) * blockDim.x;
  const size_t t0 = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  WinHdr* mine = hdr_of(a.win[me]);
  uint8_t* mybuf = a.win[me] + a.off_dbuf;
  const Span sp = make_span(0, a.n);
  float4* x4 = reinterpret_cast<float4*>(a.x);
  int bad = 0;

  // The neighbours of two rounds ago must be done reading this buffer.
  if (threadIdx.x == 0 && a.expected_reads)
    wait_geq(&mine->dreads[p], a.expected_reads, a.timeout_ns, a.status);
  __syncthreads();

  // ----- publish: one encode of the whole bucket (collectives.cpp:266) or a stage copy
  if (CODEC == kU8) {
    const float2 r = minmax_span<false>(a.x, nullptr, sp, red);
    if (threadIdx.x == 0) a.partials[blockIdx.x] = r;
    grid.sync();
    const float2 mm = reduce_partials(a.partials, G, red);
    const U8Params q8 = u8_params(mm.x, mm.y);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      mine->dhdr[p] = mm;
      if (a.n && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
    }
    uint32_t* b32 = reinterpret_cast<uint32_t*>(mybuf);
    for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
      float4 v[UX];
#pragma unroll
      for (int u = 0; u < UX; ++u) {
        const size_t gi = base + u * stride;
        if (gi < sp.g1) v[u] = __ldcg(x4 + gi);
      }
#pragma unroll
      for (int u = 0; u < UX; ++u) {
        const size_t gi = base + u * stride;
        if (gi < sp.g1) b32[gi] = quantize4(v[u], q8.lo, q8.inv);
      }
    }
    size_t e;
    if (edge_elem(sp, e)) mybuf[e] = quantize1(a.x[e], q8.lo, q8.inv);
  } else {
    float4* b4 = reinterpret_cast<float4*>(mybuf);
    for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UX) {
      float4 v[UX];
#pragma unroll
      for (int u = 0; u < UX; ++u) {
        const size_t gi = base + u * stride;
        if (gi < sp.g1) v[u] = __ldcg(x4 + gi);
      }
#pragma unroll
      for (int u = 0; u < UX; ++u) {
        const size_t gi = base + u * stride;
        if (gi < sp.g1) {
          b4[gi] = v[u];
          if (a.check_finite)
            bad |= !(finite_f(v[u].x) && finite_f(v[u].y) && finite_f(v[u].z) && finite_f(v[u].w));
        }
      }
    }
    size_t e;
    if (edge_elem(sp, e)) {
      reinterpret_cast<float*>(mybuf)[e] = a.x[e];
      if (a.check_finite) bad |= !finite_f(a.x[e]);
    }
  }
  if (cta_arrive(a.cta_done + 0)) st_release_sys(&mine->dready[p], a.epoch);

  // ----- gather: wait for every neighbour (self included: our own CTAs)
  if (threadIdx.x == 0)
    for (int i = 0; i < a.nnb; ++i)
      wait_geq(&hdr_of(a.win[a.nbrs[i]])->dready[p], a.epoch, a.timeout_ns, a.status);
  __syncthreads();
  if (CODEC == kU8) {
    if (threadIdx.x < a.nnb) {
      const float2 h = ld_peer_f2(&hdr_of(a.win[a.nbrs[threadIdx.x]])->dhdr[p]);
      s_lo[threadIdx.x] = h.x;
      s_step[threadIdx.x] = __fdiv_rn(__fsub_rn(h.y, h.x), 255.0f);
    }
    __syncthreads();
  }
  const int nnb = a.nnb;
  for (size_t base = sp.g0 + t0; base < sp.g1; base += stride * UR) {
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int i = 0; i < nnb; ++i) {
          const int j = a.nbrs[i];
          const uint8_t* buf = a.win[j] + a.off_dbuf;
          float4 d;
          if (CODEC == kU8) {
            d = dequant4(ld_peer_u32(reinterpret_cast<const uint32_t*>(buf) + gi), s_lo[i], s_step[i]);
          } else {
            d = j == me ? __ldcg(x4 + gi) : ld_peer_f4(reinterpret_cast<const float4*>(buf) + gi);
          }
          a0 = __dadd_rn(a0, double(d.x));
          a1 = __dadd_rn(a1, double(d.y));
          a2 = __dadd_rn(a2, double(d.z));
          a3 = __dadd_rn(a3, double(d.w));
        }
        __stcs(x4 + gi, make_float4(__double2float_rn(__dmul_rn(a0, a.inv)),
                                    __double2float_rn(__dmul_rn(a1, a.inv)),
                                    __double2float_rn(__dmul_rn(a2, a.inv)),
                                    __double2float_rn(__dmul_rn(a3, a.inv))));
      }
    }
  }
  size_t e;
  if (edge_elem(sp, e)) {
    double acc = 0.0;
    for (int i = 0; i < nnb; ++i) {
      const int j = a.nbrs[i];
      const uint8_t* buf = a.win[j] + a.off_dbuf;
      const float d = CODEC == kU8 ? dequant1(__ldcg(buf + e), s_lo[i], s_step[i])
                                   : (j == me ? a.x[e] : __ldcg(reinterpret_cast<const float*>(buf) + e));
      acc = __dadd_rn(acc, double(d));
    }
    a.x[e] = __double2float_rn(__dmul_rn(acc, a.inv));
  }
  if (bad) latch(a.status, kStatusNonFinite);
  // ----- acknowledge the reads so each neighbour may reuse its buffer
  if (cta_arrive(a.cta_done + 1))
    for (int i = 0; i < nnb; ++i)
      if (a.nbrs[i] != me) red_release_sys_add(&hdr_of(a.win[a.nbrs[i]])->dreads[p], 1ull);
}

template <typename K, typename A>
int launch_coop(K kernel, const A& args, cudaStream_t s, int* grid_out) {
  static_assert(sizeof(A) < 4000, "kernel argument block too large");
  const int grid = persistent_grid(reinterpret_cast<const void*>(kernel), kThreads);
  A copy = args;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid),
                                          dim3(kThreads), params, 0, s));
  if (grid_out) *grid_out = grid;
  return B2_OK;
}

}  // namespace

int launch_central(const CentralArgs& a, int codec, bool ec, cudaStream_t s) {
  if (codec == kU8)
    return ec ? launch_coop(central_kernel<kU8, true>, a, s, nullptr)
              : launch_coop(central_kernel<kU8, false>, a, s, nullptr);
  return ec ? launch_coop(central_kernel<kIdentity, true>, a, s, nullptr)
            : launch_coop(central_kernel<kIdentity, false>, a, s, nullptr);
}

int launch_decent(const DecentArgs& a, int codec, cudaStream_t s) {
  return codec == kU8 ? launch_coop(decent_kernel<kU8>, a, s, nullptr)
                      : launch_coop(decent_kernel<kIdentity>, a, s, nullptr);
}

int max_persistent_grid() { return sm_count() * 4; }

}  // namespace b2
