// small_central.cu -- latency path of C_LP_S / C_FP_S (scatter_reduce_lp /
// scatter_reduce_fp, collectives.cpp:42-163) for buckets that fit in the
// registers of one co-resident grid: the engine's 8 MiB buckets (2M floats,
// engine.hpp:58) and smaller.  The ring kernel (collectives.cu) pays a ring
// set-up, grid barriers between its phases and several cross-GPU round trips.
//
// Every rank launches the same grid over the same n, so CTA b owns the same
// elements of every chunk on every rank (4-element unit u = i / 4 of chunk
// k: thread gt = u mod T, register u / T), and the ranks synchronise PER CTA:
//
//   1  x of every chunk into registers; per-chunk (min, max) partials
//   2  grid barrier #1: every CTA reduces the g chunk headers (uint8)
//   3  encode chunk k into MY window's slot k (+ delta with EC), my header of
//      chunk k into my window, fence, one red per owner on its [me][b]
//   4  owner side: wait for every source's [j][b], fold my chunk's piece in
//      ascending rank order (own codes from registers, the others over
//      NVLink), y2 (- eps) in registers, second (min, max) partial
//   5  grid barrier #2: header 2; Q2 from registers into my out2 (+ eps),
//      decode my own chunk of x directly; header 2 into my window; one red
//      per rank on its [me][b] (second counter array)
//   6  gather: wait for every owner's [k][b], decode owner k's piece of out2
//
// Two grid barriers and two cross-GPU hand-offs per CTA.  Buffer reuse needs
// no acknowledgements (collectives.cu 4.6's argument): my slot k is rewritten
// in call t+1 only after I gathered owner k's out2 of call t, published after
// owner k's last read of my slot; owner k's out2 is rewritten in call t+1
// only after its fold of call t+1, which needs my codes of call t+1, which I
// produce after my gather of call t.  Bit-exact with the reference (the same
// element arithmetic as every other path).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "b2_host.h"
#include "collectives.cuh"

namespace b2 {
namespace {

namespace cg = cooperative_groups;

constexpr int kCThr = 256;
constexpr float kInfC = __builtin_huge_valf();

__device__ __forceinline__ WinHdr* chdr(uint8_t* w) { return reinterpret_cast<WinHdr*>(w); }

__device__ __forceinline__ void crange(size_t n, int g, int k, size_t& lo, size_t& sz) {
  const size_t base = n / size_t(g), extra = n % size_t(g), uk = size_t(k);
  lo = uk * base + (uk < extra ? uk : extra);
  sz = base + (uk < extra ? 1 : 0);
}

// (lo, hi) over the CTA, valid in every thread
__device__ __forceinline__ float2 cta_minmax(float lo, float hi, float2* wred) {
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) wred[w] = make_float2(lo, hi);
  __syncthreads();
  const float2 v = l < kCThr / 32 ? wred[l] : wred[0];
  return make_float2(warp_min_nan(v.x), warp_max_nan(v.y));
}

// up to 4 consecutive floats at p (v valid, 16-byte aligned when al)
__device__ __forceinline__ float4 ld4v(const float* p, int v, bool al) {
  if (v == 4 && al) return *reinterpret_cast<const float4*>(p);
  float4 r = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  r.x = p[0];
  if (v > 1) r.y = p[1];
  if (v > 2) r.z = p[2];
  if (v > 3) r.w = p[3];
  return r;
}
__device__ __forceinline__ void st4v(float* p, float4 r, int v, bool al) {
  if (v == 4 && al) {
    *reinterpret_cast<float4*>(p) = r;
    return;
  }
  p[0] = r.x;
  if (v > 1) p[1] = r.y;
  if (v > 2) p[2] = r.z;
  if (v > 3) p[3] = r.w;
}
__device__ __forceinline__ float4 fsub4(float4 a, float4 b) { return sub4(a, b); }
__device__ __forceinline__ void mm4(float4 v, int n, float& lo, float& hi) {
  lo = fmin_nan(lo, v.x);
  hi = fmax_nan(hi, v.x);
  if (n > 1) { lo = fmin_nan(lo, v.y); hi = fmax_nan(hi, v.y); }
  if (n > 2) { lo = fmin_nan(lo, v.z); hi = fmax_nan(hi, v.z); }
  if (n > 3) { lo = fmin_nan(lo, v.w); hi = fmax_nan(hi, v.w); }
}
__device__ __forceinline__ bool fin4(float4 v, int n) {
  bool f = finite_f(v.x);
  if (n > 1) f &= finite_f(v.y);
  if (n > 2) f &= finite_f(v.z);
  if (n > 3) f &= finite_f(v.w);
  return f;
}
__device__ __forceinline__ float4 dq4(uint32_t c, const SrcDecS& d) {
  return d.fast ? dequant4_fast(c, d.lo, d.step, d.c23) : dequant4(c, d.lo, d.step);
}
__device__ __forceinline__ SrcDecS src_dec(float2 h) {
  const U8Params q = u8_params(h.x, h.y);
  return SrcDecS{q.lo, q.step, q.c23, q.fastdec ? 1 : 0};
}
// quantize the valid lanes of v (e = global index of lane 0)
__device__ __forceinline__ uint32_t q4v(float4 v, int n, const U8Params& p, const Rounder& r, size_t e) {
  if (n == 4) return q4r(v, p.lo, p.inv, r, e);
  uint32_t c = q1r(v.x, p.lo, p.inv, r, e);
  if (n > 1) c |= uint32_t(q1r(v.y, p.lo, p.inv, r, e + 1)) << 8;
  if (n > 2) c |= uint32_t(q1r(v.z, p.lo, p.inv, r, e + 2)) << 16;
  return c;
}

// Element i of chunk k: unit u = i / 4 (4 consecutive elements), held by
// thread gt = u mod T as its register j = u / T.
template <int CODEC, bool EC, int G, int R>
__global__ void __launch_bounds__(kCThr) central_small_kernel(CentralArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ float2 wred[kCThr / 32];
  __shared__ int s_bad;
  __shared__ SrcDecS s_dec[G];
  constexpr bool U8 = CODEC == kU8;
  const int me = a.me, b = blockIdx.x, nb = gridDim.x;
  const size_t T = size_t(nb) * kCThr, gt = size_t(b) * kCThr + threadIdx.x;
  const size_t n = a.n;
  const unsigned long long ep = a.epoch;
  if (threadIdx.x == 0) s_bad = 0;
  unsigned long long* tr = a.trace ? a.trace + size_t(b) * kTraceSlots : nullptr;
  if (tr && threadIdx.x == 0) tr[kTrStart] = globaltimer();
  const Rounder r1 = make_rounder(U8 && a.sr_on, a.sr_seed, me, 1), r2 = make_rounder(U8 && a.sr_on, a.sr_seed, me, 2);
  const bool xal = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0;
  const bool dal = !EC || (reinterpret_cast<uintptr_t>(a.delta) & 15) == 0;
  size_t clo[G], csz[G];
#pragma unroll
  for (int k = 0; k < G; ++k) crange(n, G, k, clo[k], csz[k]);
  int bad = 0;
  // valid lanes of unit (k, j)
  auto nv = [&](int k, int j) -> int {
    const size_t i = 4 * (gt + size_t(j) * T);
    return i >= csz[k] ? 0 : (csz[k] - i >= 4 ? 4 : int(csz[k] - i));
  };
  // ---- 1: y = x (- delta) of every chunk into registers, per-chunk (min, max)
  float4 y[G][R];
  float plo[G], phi[G];
#pragma unroll
  for (int k = 0; k < G; ++k) {
    plo[k] = kInfC;
    phi[k] = -kInfC;
    const bool al = ((clo[k] & 3) == 0);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int v = nv(k, j);
      y[k][j] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (v) {
        const size_t e = clo[k] + 4 * (gt + size_t(j) * T);
        float4 t = ld4v(a.x + e, v, al && xal);
        if (EC) t = fsub4(t, ld4v(a.delta + e, v, al && dal));
        y[k][j] = t;
        mm4(t, v, plo[k], phi[k]);
        if (!U8 && a.check_finite) bad |= !fin4(t, v);
      }
    }
  }
  // ---- 2: the g chunk headers (uint8)
  float hlo[G], hhi[G];
  if (U8) {
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const float2 m = cta_minmax(plo[k], phi[k], wred);
      if (threadIdx.x == 0) a.partials[size_t(k) * nb + b] = m;
    }
    grid.sync();
#pragma unroll
    for (int k = 0; k < G; ++k) {
      float l = kInfC, h = -kInfC;
      for (unsigned c = threadIdx.x; c < unsigned(nb); c += kCThr) {
        const float2 v = __ldcg(a.partials + size_t(k) * nb + c);
        l = fmin_nan(l, v.x);
        h = fmax_nan(h, v.y);
      }
      const float2 m = cta_minmax(l, h, wred);
      hlo[k] = m.x;
      hhi[k] = m.y;
    }
  }
  if (tr && threadIdx.x == 0) tr[kTrP1FirstA] = globaltimer();
  // ---- 3: encode every chunk into my slot k; my headers; signal the owners
  uint32_t own[R];  // my codes of my own chunk (uint8): the self term of the fold
  WinHdr* mine = chdr(a.win[me]);
#pragma unroll
  for (int k = 0; k < G; ++k) {
    uint8_t* slot = a.win[me] + a.off_recv1 + size_t(k) * a.slot_stride;  // element i at slot + eb * i
    const bool al = ((clo[k] & 3) == 0);
    U8Params p{};
    if (U8) p = u8_params(hlo[k], hhi[k]);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int v = nv(k, j);
      const size_t u = gt + size_t(j) * T;
      if (k == me) own[j] = 0;
      if (!v) continue;
      const size_t e = clo[k] + 4 * u;
      if (U8) {
        const uint32_t c = q4v(y[k][j], v, p, r1, e);
        reinterpret_cast<uint32_t*>(slot)[u] = c;
        if (EC) st4v(a.delta + e, fsub4(y[k][j], dequant4(c, p)), v, al && dal);
        if (k == me) own[j] = c;
      } else {
        reinterpret_cast<float4*>(slot)[u] = y[k][j];
        if (EC) st4v(a.delta + e, fsub4(y[k][j], y[k][j]), v, al && dal);
      }
    }
    if (U8 && threadIdx.x == 0) mine->hdr1[k] = make_float2(hlo[k], hhi[k]);  // every CTA: the same value
  }
  __syncthreads();
  if (threadIdx.x < G && int(threadIdx.x) != me) {
    __threadfence();  // peers read my window through this GPU's L2
    red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[threadIdx.x] + a.off_sgate) +
                            size_t(me) * a.sgate_stride + b,
                        1ull);
  }
  if (tr && threadIdx.x == 0) tr[kTrP1Done] = globaltimer();
  // ---- 4: fold my chunk's piece once every source's CTA b is in
  if (threadIdx.x < G) {
    const int j = threadIdx.x;
    if (j != me)
      wait_geq(reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_sgate) + size_t(j) * a.sgate_stride + b,
               ep, a.timeout_ns, a.status);
    if (U8) s_dec[j] = src_dec(j == me ? make_float2(hlo[me], hhi[me]) : __ldcg(&chdr(a.win[j])->hdr1[me]));
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[kTrP2Ready] = globaltimer();
  const size_t mlo = clo[me];
  const bool mal = ((mlo & 3) == 0);
  const bool eal = !EC || (reinterpret_cast<uintptr_t>(a.eps) & 15) == 0;
  float4 y2[R];
  float lo2 = kInfC, hi2 = -kInfC;
  {
    // every remote word of the piece first: one NVLink round trip
    uint32_t cw[U8 ? R : 1][G];
    float4 fw[U8 ? 1 : R][U8 ? 1 : G];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (!nv(me, j)) continue;
      const size_t u = gt + size_t(j) * T;
#pragma unroll
      for (int s = 0; s < G; ++s) {
        if (s == me) continue;
        const uint8_t* slot = a.win[s] + a.off_recv1 + size_t(me) * a.slot_stride;
        if (U8)
          cw[U8 ? j : 0][s] = __ldcg(reinterpret_cast<const uint32_t*>(slot) + u);
        else
          fw[U8 ? 0 : j][U8 ? 0 : s] = __ldcg(reinterpret_cast<const float4*>(slot) + u);
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int v = nv(me, j);
      y2[j] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (!v) continue;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // kernels.cpp:14-16, ascending rank
#pragma unroll
      for (int s = 0; s < G; ++s) {
        float4 d;
        if (U8)
          d = dq4(s == me ? own[j] : cw[U8 ? j : 0][s], s_dec[s]);
        else
          d = s == me ? y[me][j] : fw[U8 ? 0 : j][U8 ? 0 : s];
        a0 = __dadd_rn(a0, double(d.x));
        a1 = __dadd_rn(a1, double(d.y));
        a2 = __dadd_rn(a2, double(d.z));
        a3 = __dadd_rn(a3, double(d.w));
      }
      float4 t = make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2),
                             __double2float_rn(a3));
      if (EC) t = fsub4(t, ld4v(a.eps + 4 * (gt + size_t(j) * T), v, eal));
      if (!U8 && a.check_finite) bad |= !fin4(t, v);
      y2[j] = t;
      mm4(t, v, lo2, hi2);
    }
  }
  // ---- 5: second header (uint8), Q2, my own chunk of x, publish
  U8Params p2{};
  if (U8) {
    const float2 m = cta_minmax(lo2, hi2, wred);
    if (threadIdx.x == 0) a.partials[size_t(kMaxRanks) * nb + b] = m;
    grid.sync();
    float l = kInfC, h = -kInfC;
    for (unsigned c = threadIdx.x; c < unsigned(nb); c += kCThr) {
      const float2 w = __ldcg(a.partials + size_t(kMaxRanks) * nb + c);
      l = fmin_nan(l, w.x);
      h = fmax_nan(h, w.y);
    }
    const float2 mm = cta_minmax(l, h, wred);
    p2 = u8_params(mm.x, mm.y);
    if (threadIdx.x == 0) {
      mine->hdr2 = mm;  // every CTA: the same value
      if (b == 0 && csz[me] && !(finite_f(mm.x) && finite_f(mm.y))) latch(a.status, kStatusNonFinite);
    }
    if (b == 0 && threadIdx.x < G) {
      const int k = threadIdx.x;
      if (csz[k] && !(finite_f(hlo[k]) && finite_f(hhi[k]))) latch(a.status, kStatusNonFinite);
    }
  }
  if (tr && threadIdx.x == 0) tr[kTrP2A] = globaltimer();
  uint8_t* out2 = a.win[me] + a.off_out2;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int v = nv(me, j);
    if (!v) continue;
    const size_t u = gt + size_t(j) * T;
    float4 d2;
    if (U8) {
      const uint32_t c = q4v(y2[j], v, p2, r2, mlo + 4 * u);
      reinterpret_cast<uint32_t*>(out2)[u] = c;
      d2 = dequant4(c, p2);
    } else {
      reinterpret_cast<float4*>(out2)[u] = y2[j];
      d2 = y2[j];
    }
    if (EC) st4v(a.eps + 4 * u, fsub4(y2[j], d2), v, eal);
    st4v(a.x + mlo + 4 * u, d2, v, mal && xal);
  }
  __syncthreads();
  if (threadIdx.x < G && int(threadIdx.x) != me) {
    __threadfence();
    red_relaxed_sys_add(reinterpret_cast<unsigned long long*>(a.win[threadIdx.x] + a.off_sgate2) +
                            size_t(me) * a.sgate_stride + b,
                        1ull);
  }
  if (tr && threadIdx.x == 0) tr[kTrP2Done] = globaltimer();
  // ---- 6: gather every other owner's piece of out2
  if (threadIdx.x < G) {
    const int k = threadIdx.x;
    if (k != me) {
      wait_geq(reinterpret_cast<const unsigned long long*>(a.win[me] + a.off_sgate2) + size_t(k) * a.sgate_stride + b,
               ep, a.timeout_ns, a.status);
      if (U8) s_dec[k] = src_dec(__ldcg(&chdr(a.win[k])->hdr2));
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[kTrP3First] = globaltimer();
  {
    uint32_t cw[U8 ? G : 1][R];
    float4 fw[U8 ? 1 : G][U8 ? 1 : R];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (k == me) continue;
      const uint8_t* src = a.win[k] + a.off_out2;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (!nv(k, j)) continue;
        const size_t u = gt + size_t(j) * T;
        if (U8)
          cw[U8 ? k : 0][j] = __ldcg(reinterpret_cast<const uint32_t*>(src) + u);
        else
          fw[U8 ? 0 : k][U8 ? 0 : j] = __ldcg(reinterpret_cast<const float4*>(src) + u);
      }
    }
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (k == me) continue;
      const bool al = ((clo[k] & 3) == 0) && xal;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int v = nv(k, j);
        if (!v) continue;
        const float4 d = U8 ? dq4(cw[U8 ? k : 0][j], s_dec[k]) : fw[U8 ? 0 : k][U8 ? 0 : j];
        st4v(a.x + clo[k] + 4 * (gt + size_t(j) * T), d, v, al);
      }
    }
  }
  if (bad) atomicOr(&s_bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_bad) latch(a.status, kStatusNonFinite);
    fail_epilogue(a.status);
    if (tr) tr[kTrEnd] = globaltimer();
  }
}

template <int CODEC, bool EC, int G, int R>
int try_small_c(const CentralArgs& a, cudaStream_t s, int sms) {
  const void* fn = reinterpret_cast<const void*>(central_small_kernel<CODEC, EC, G, R>);
  const int per_sm = occupancy(fn, kCThr);
  const int nsm = sms > 0 && sms < sm_count() ? sms : sm_count();
  const size_t cap = std::min<size_t>(size_t(nsm) * size_t(per_sm > 0 ? per_sm : 0), kSmallMaxGridD);
  const size_t maxchunk = (a.n + G - 1) / G, per_block = size_t(kCThr) * 4 * R;
  const size_t need = (maxchunk + per_block - 1) / per_block;
  if (per_sm < 1 || need > cap) return B2_ERR_UNSUPPORTED;
  // at least one CTA per SM: the loads of a small bucket spread over every SM
  const int grid = int(std::min<size_t>(cap, std::max<size_t>(need, size_t(nsm))));
  CentralArgs copy = a;
  void* params[] = {&copy};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kCThr), params, 0, s));
  return B2_OK;
}

// one 4-element unit per thread and chunk first (more CTAs share a small
// bucket), then about 64 registers of bucket per thread
template <int CODEC, bool EC, int G>
int small_c(const CentralArgs& a, cudaStream_t s, int sms) {
  constexpr int kBig = G <= 2 ? 8 : G <= 4 ? 4 : 2;
  const int rc = try_small_c<CODEC, EC, G, 1>(a, s, sms);
  return rc == B2_ERR_UNSUPPORTED ? try_small_c<CODEC, EC, G, kBig>(a, s, sms) : rc;
}

template <int CODEC, bool EC>
int small_c_g(const CentralArgs& a, cudaStream_t s, int sms) {
  switch (a.g) {
    case 2: return small_c<CODEC, EC, 2>(a, s, sms);
    case 3: return small_c<CODEC, EC, 3>(a, s, sms);
    case 4: return small_c<CODEC, EC, 4>(a, s, sms);
    case 5: return small_c<CODEC, EC, 5>(a, s, sms);
    case 6: return small_c<CODEC, EC, 6>(a, s, sms);
    case 7: return small_c<CODEC, EC, 7>(a, s, sms);
    case 8: return small_c<CODEC, EC, 8>(a, s, sms);
  }
  return B2_ERR_UNSUPPORTED;
}

}  // namespace

// C_* latency path (g >= 2, uint8 / identity); B2_ERR_UNSUPPORTED when the
// bucket exceeds the register capacity or B2_SMALL_C_MAX (the caller then
// takes the ring kernel).  The choice depends only on (n, g, SM count, SM
// budget), the same on every rank of a window; the path keeps its own call
// counter and counter arrays (comm.cu), so a budget change that switches a
// window between this kernel and the ring is safe (see the reuse argument
// above, which holds across the two protocols).
int launch_central_small(const CentralArgs& a, int codec, bool ec, cudaStream_t s, int sms) {
  static const size_t limit = [] {  // B2_SMALL_C_MAX=<elements> moves the cut-over (A/B runs)
    const char* e = getenv("B2_SMALL_C_MAX");
    return e ? std::min<size_t>(std::strtoull(e, nullptr, 10), kSmallCentralWin) : kSmallCentralMax;
  }();
  if (a.g < 2 || a.n > limit) return B2_ERR_UNSUPPORTED;
  if (codec == kU8) return ec ? small_c_g<kU8, true>(a, s, sms) : small_c_g<kU8, false>(a, s, sms);
  return ec ? small_c_g<kIdentity, true>(a, s, sms) : small_c_g<kIdentity, false>(a, s, sms);
}

}  // namespace b2
