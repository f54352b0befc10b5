// codec.cu -- the uniform8 ("MinMaxUInt8") codec on one GPU, bucket
// flatten/unflatten, and the synthetic-gradient generator.
//
// Reference: codec.cpp:40-80 (encode), 93-109 (decode), 125-137
// (compensate_encode); kernels.cpp:34-56 (minmax / quantize_u8 /
// dequantize_u8); tensor.cpp:46-68 (BucketArena::flatten).
//
// Encode is two passes over x because every code depends on the chunk-global
// (min, max): pass 1 reduces a NaN-propagating (min, max) per CTA (128-bit
// loads, redux.sync warp reduction) into two order-preserving u32 keys with
// one atomicMin/atomicMax per CTA; pass 2 re-reads x (from L2 when the chunk
// fits in the 126 MB L2) and emits 4 codes per 32-bit store.  HBM bytes per
// element: 4 (pass 1) + 4 (pass 2, 0 when L2-resident) + 1 (codes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include <cooperative_groups.h>

#include "b2_device.cuh"
#include "b2_host.h"
#include "ring.cuh"

namespace b2 {
namespace {

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned key_of(float f) {
  const unsigned b = __float_as_uint(f);
  return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float float_of(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

// Encode = ONE cooperative launch on the TMA ring (ring.cuh): pass A streams
// x (- delta) and reduces a NaN-propagating (min, max) per CTA into two
// order-preserving u32 keys (one atomicMin/atomicMax per CTA, hdr scratch
// words); a grid barrier finalises the header; pass B re-streams x in REVERSE
// tile order (its tail is still in L2, all of it when the chunk fits) and
// writes 4 codes per 32-bit store (+ delta / decoded with error feedback).
template <bool EC>
__global__ void __launch_bounds__(kRingThreads, 1) encode_ring_kernel(const float* __restrict__ x,
                                                                      float* __restrict__ delta, size_t n,
                                                                      uint8_t* __restrict__ codes, float* hdr,
                                                                      float* __restrict__ decoded) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red[32];
  cg::grid_group grid = cg::this_grid();
  Ring r;
  r.init(smem, nullptr, 0);
  unsigned* keys = reinterpret_cast<unsigned*>(hdr + 2);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    keys[0] = 0xffffffffu;
    keys[1] = 0u;
  }
  grid.sync();
  PassDesc p = PassDesc::make();
  p.s = 0;
  p.n = n;
  p.eb = 4;
  p.nsrc = EC ? 2 : 1;
  p.base[0] = reinterpret_cast<const uint8_t*>(x);
  if (EC) p.base[1] = reinterpret_cast<const uint8_t*>(delta);
  const int ct = r.ct;
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  r.run(p, [&](const uint8_t* st, size_t, size_t units, int T) {
    const float4* xs = reinterpret_cast<const float4*>(st);
    const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
    for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
      float4 v = xs[gi];
      if (EC) v = sub4(v, ds[gi]);
      lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
      hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
    }
  });
  r.edges(p, [&](size_t e) {
    float v = x[e];
    if (EC) v = __fsub_rn(v, delta[e]);
    lo = fmin_nan(lo, v);
    hi = fmax_nan(hi, v);
  });
  if (r.ct >= 0) {
    const float2 m = consumer_minmax(lo, hi, red);
    if (ct == 0) {
      if (m.x != m.x || m.y != m.y) {
        atomicMax(keys + 1, 0xffffffffu);  // NaN -> the max key decodes to NaN
      } else {
        atomicMin(keys + 0, key_of(m.x));
        atomicMax(keys + 1, key_of(m.y));
      }
    }
  }
  grid.sync();
  const float mlo = float_of(__ldcg(keys + 0)), mhi = float_of(__ldcg(keys + 1));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr[0] = mlo;
    hdr[1] = mhi;
  }
  const U8Params q = u8_params(mlo, mhi);
  p.reverse = true;
  r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int T) {
    const float4* xs = reinterpret_cast<const float4*>(st);
    const float4* ds = reinterpret_cast<const float4*>(st + size_t(T) * 64);
    uint32_t* c32 = reinterpret_cast<uint32_t*>(codes + e0);
    for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
      float4 y = xs[gi];
      if (EC) y = sub4(y, ds[gi]);
      const uint32_t c = quantize4(y, q.lo, q.inv);
      __stcs(c32 + gi, c);
      if (EC) {
        const float4 d = dequant4(c, q);
        reinterpret_cast<float4*>(delta)[(e0 >> 2) + gi] = sub4(y, d);
        if (decoded) __stcs(reinterpret_cast<float4*>(decoded) + (e0 >> 2) + gi, d);
      }
    }
  });
  r.edges(p, [&](size_t e) {
    float y = x[e];
    if (EC) y = __fsub_rn(y, delta[e]);
    const uint8_t c = quantize1(y, q.lo, q.inv);
    codes[e] = c;
    if (EC) {
      const float d = dequant1(c, q.lo, q.step);
      delta[e] = __fsub_rn(y, d);
      if (decoded) decoded[e] = d;
    }
  });
}

__global__ void __launch_bounds__(kRingThreads, 1) decode_ring_kernel(const uint8_t* __restrict__ codes,
                                                                      const float* hdr, size_t n,
                                                                      float* __restrict__ out) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring r;
  r.init(smem, nullptr, 0);
  const U8Params q = u8_params(hdr[0], hdr[1]);
  PassDesc p = PassDesc::make();
  p.s = 0;
  p.n = n;
  p.eb = 1;
  p.nsrc = 1;
  p.base[0] = codes;
  const int ct = r.ct;
  float4* o4 = reinterpret_cast<float4*>(out);
  r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int) {
    const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
    for (int gi = ct; gi < int(units * 4); gi += kConsumers) __stcs(o4 + (e0 >> 2) + gi, dequant4(cs[gi], q));
  });
  r.edges(p, [&](size_t e) { out[e] = dequant1(codes[e], q.lo, q.step); });
}

// ------------------------------------------------- small buckets (latency)
// For buckets that fit in the registers of one full-occupancy grid (the 4M
// config of BASELINE.json: 16 MB), encode is ONE pass over x: every thread
// loads its R float4 groups (coalesced: group gt + k*T), reduces a
// NaN-propagating (min, max) per CTA into a partial, one grid barrier, every
// CTA reduces the partials (same order everywhere -> same header), then
// quantizes from its registers.  HBM bytes: 4n + n, one grid sync, no ring
// set-up -- the TMA ring's pipeline never warms up on 3 tiles per SM.
constexpr int kSmallThreads = 256;
template <bool EC, int R>
__global__ void __launch_bounds__(kSmallThreads) encode_small_kernel(const float* __restrict__ x,
                                                                     float* __restrict__ delta, size_t n,
                                                                     uint8_t* __restrict__ codes, float* hdr,
                                                                     float* __restrict__ decoded,
                                                                     float2* __restrict__ partials) {
  cg::grid_group grid = cg::this_grid();
  __shared__ float2 wred[kSmallThreads / 32];
  const size_t T = size_t(gridDim.x) * kSmallThreads, gt = size_t(blockIdx.x) * kSmallThreads + threadIdx.x;
  const size_t ng = n >> 2;  // whole float4 groups; the (< 4) tail goes to the last thread
  // programmatic dependent launch (small_launch): the previous kernel on the
  // stream is complete and visible past this point; a no-op otherwise
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4 y[R];
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const size_t g = gt + size_t(k) * T;
    if (g < ng) {
      y[k] = __ldcs(x4 + g);
      if (EC) y[k] = sub4(y[k], reinterpret_cast<const float4*>(delta)[g]);
      lo = fmin_nan(lo, fmin_nan(fmin_nan(y[k].x, y[k].y), fmin_nan(y[k].z, y[k].w)));
      hi = fmax_nan(hi, fmax_nan(fmax_nan(y[k].x, y[k].y), fmax_nan(y[k].z, y[k].w)));
    }
  }
  float yt[3];
  const bool tail = gt == T - 1 && (n & 3);
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      float v = x[e];
      if (EC) v = __fsub_rn(v, delta[e]);
      yt[e - 4 * ng] = v;
      lo = fmin_nan(lo, v);
      hi = fmax_nan(hi, v);
    }
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) wred[w] = make_float2(lo, hi);
  __syncthreads();
  if (threadIdx.x < 32) {
    const float2 v = l < kSmallThreads / 32 ? wred[l] : wred[0];
    const float a = warp_min_nan(v.x), b = warp_max_nan(v.y);
    if (l == 0) partials[blockIdx.x] = make_float2(a, b);
  }
  grid.sync();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the decode may start launching
  lo = __int_as_float(0x7f800000);
  hi = -__int_as_float(0x7f800000);
  for (unsigned c = threadIdx.x; c < gridDim.x; c += kSmallThreads) {
    const float2 v = __ldcg(partials + c);
    lo = fmin_nan(lo, v.x);
    hi = fmax_nan(hi, v.y);
  }
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  __syncthreads();  // wred reuse
  if (l == 0) wred[w] = make_float2(lo, hi);
  __syncthreads();
  {
    const float2 v = l < kSmallThreads / 32 ? wred[l] : wred[0];
    lo = warp_min_nan(v.x);
    hi = warp_max_nan(v.y);
  }
  if (gt == 0) {
    hdr[0] = lo;
    hdr[1] = hi;
  }
  const U8Params q = u8_params(lo, hi);
  uint32_t* c32 = reinterpret_cast<uint32_t*>(codes);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const size_t g = gt + size_t(k) * T;
    if (g < ng) {
      const uint32_t c = quantize4(y[k], q.lo, q.inv);
      __stcs(c32 + g, c);
      if (EC) {
        const float4 d = dequant4(c, q);
        reinterpret_cast<float4*>(delta)[g] = sub4(y[k], d);
        if (decoded) __stcs(reinterpret_cast<float4*>(decoded) + g, d);
      }
    }
  }
  if (tail)
    for (size_t e = 4 * ng; e < n; ++e) {
      const uint8_t c = quantize1(yt[e - 4 * ng], q.lo, q.inv);
      codes[e] = c;
      if (EC) {
        const float d = dequant1(c, q.lo, q.step);
        delta[e] = __fsub_rn(yt[e - 4 * ng], d);
        if (decoded) decoded[e] = d;
      }
    }
}

// decode: V x 4 codes (V 32-bit loads, T apart) -> V float4 stores per
// thread, no ring.  V = 2 by default (measured in a graph at 4M: 3.8 us,
// against 4.5 us with V = 1 and 3.9 us with V = 4; tests/cpp/codec_timing.py).
template <int V>
__global__ void __launch_bounds__(kSmallThreads) decode_small_kernel(const uint8_t* __restrict__ codes,
                                                                     const float* hdr, size_t n,
                                                                     float* __restrict__ out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the encode's codes and header are complete
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const U8Params q = u8_params(hdr[0], hdr[1]);
  const size_t ng = n >> 2, T = size_t(gridDim.x) * kSmallThreads;
  const uint32_t* c32 = reinterpret_cast<const uint32_t*>(codes);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t g0 = size_t(blockIdx.x) * kSmallThreads + threadIdx.x; g0 < ng; g0 += V * T) {
    uint32_t c[V];
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (g0 + v * T < ng) c[v] = __ldcs(c32 + g0 + v * T);
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (g0 + v * T < ng) __stcs(o4 + g0 + v * T, dequant4(c[v], q));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (size_t e = 4 * ng; e < n; ++e) out[e] = dequant1(codes[e], q.lo, q.step);
}

__global__ void init_keys_kernel(float* hdr, size_t n) {
  unsigned* keys = reinterpret_cast<unsigned*>(hdr + 2);
  keys[0] = 0xffffffffu;
  keys[1] = 0u;
  if (n == 0) {  // empty input: header (0, 0), codec.cpp:52-57
    hdr[0] = 0.0f;
    hdr[1] = 0.0f;
  }
}

__global__ void pack_wire_kernel(const uint8_t* __restrict__ codes, const float* hdr, size_t n,
                                 uint8_t* __restrict__ wire) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < 8) {
    const uint32_t b = __float_as_uint(hdr[i >> 2]);
    wire[i] = static_cast<uint8_t>(b >> (8 * (i & 3)));
  }
  for (size_t k = i; k < n; k += size_t(gridDim.x) * blockDim.x) wire[8 + k] = codes[k];
}

__global__ void unpack_wire_kernel(const uint8_t* __restrict__ wire, size_t n,
                                   uint8_t* __restrict__ codes, float* hdr) {
  const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < 2) {
    uint32_t b = 0;
    for (int k = 0; k < 4; ++k) b |= uint32_t(wire[4 * i + k]) << (8 * k);
    hdr[i] = __uint_as_float(b);
  }
  for (size_t k = i; k < n; k += size_t(gridDim.x) * blockDim.x) codes[k] = wire[8 + k];
}

// ----------------------------------------------------------- flatten
constexpr int kFlatMax = 64;
struct FlatTable {
  const float* ptr[kFlatMax];
  size_t len[kFlatMax];
  size_t off[kFlatMax];
  int count;
  int to_arena;  // 1 = members -> arena (flatten), 0 = arena -> members
};

// One CTA-strided pass per member; each member's copy is split across the
// whole grid.  Vector path when both sides are 16-byte aligned.
__global__ void __launch_bounds__(kThreads) flatten_kernel(FlatTable t, float* arena) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int m = 0; m < t.count; ++m) {
    const float* src = t.to_arena ? t.ptr[m] : arena + t.off[m];
    float* dst = t.to_arena ? arena + t.off[m] : const_cast<float*>(t.ptr[m]);
    const size_t len = t.len[m];
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    if (vec) {
      const size_t nv = len >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (size_t i = tid; i < nv; i += stride) d4[i] = ld_stream(s4 + i);
      for (size_t i = (nv << 2) + tid; i < len; i += stride) dst[i] = src[i];
    } else {
      for (size_t i = tid; i < len; i += stride) dst[i] = src[i];
    }
  }
}

// ----------------------------------------------------------- synthetic
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__global__ void __launch_bounds__(kThreads) synth_kernel(float* x, size_t n, uint64_t seed,
                                                         uint64_t offset) {
  const uint64_t key = splitmix64(seed);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const uint64_t h = splitmix64(key + offset + i);
    const int32_t m = static_cast<int32_t>(h >> 40);
    x[i] = __fmul_rn(static_cast<float>(m - 8388608), 1.1920928955078125e-07f);
  }
}


// Codec::encode uniform8 with Rounding::stochastic (codec.cpp:67-78):
// level = floor(q) + (u < q - floor(q)), q = (x - min) * inv_step, clamped
// to [0, 255].  u is uniform in [0, 1) with 24 random bits (the resolution of
// std::uniform_real_distribution<float>) from a counter hash of (seed,
// element) instead of the host's mt19937 stream, so the levels are unbiased
// like the reference's (test_codec.cpp:175-192) but not the same draws.
// Runs after the nearest-rounding encode, whose header it reuses; a
// degenerate range keeps the all-zero codes (codec.cpp:62-64).
__global__ void u8_stochastic_kernel(const float* __restrict__ x, size_t n, uint8_t* __restrict__ codes,
                                     const float* __restrict__ hdr, uint64_t seed) {
  const float lo = hdr[0], hi = hdr[1];
  const float range = __fsub_rn(hi, lo);
  if (range == 0.0f) return;
  const float inv = __fdiv_rn(255.0f, range);
  const uint64_t key = splitmix64(seed);
  for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += size_t(gridDim.x) * blockDim.x) {
    const float q = __fmul_rn(__fsub_rn(x[e], lo), inv);
    const float fl = floorf(q);
    const float u = float(uint32_t(splitmix64(key + e) >> 40)) * 0x1p-24f;
    float level = __fadd_rn(fl, u < __fsub_rn(q, fl) ? 1.0f : 0.0f);
    level = level < 0.0f ? 0.0f : (level > 255.0f ? 255.0f : level);
    codes[e] = uint8_t(level);
  }
}

int grid_for(const void* f) { return persistent_grid(f, kThreads); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------- onebit
// Codec::encode onebit (codec.cpp:81-88): scale = (float)(sum |x| in fp64) /
// (float)n, bit k of the LE bit string = !signbit(x[k]) (kernels.cpp:26-32,
// 58-63); wire = [scale f32][ceil(n/8) bytes].  One thread per 32 elements
// (one 32-bit word of bits); per-block fp64 partials are summed by the last
// block in block order, so the result is deterministic -- but the fp64 sum's
// order differs from the reference's (scalar: sequential; AVX2: 4 lanes), so
// the scale equals the reference's whenever that sum is exact in fp64 (e.g.
// inputs on a common 2^-k grid) and is within one float rounding otherwise
// (the reference's own backends differ the same way).  A non-finite input
// makes the scale NaN: the reference throws (codec.cpp:24-27).
constexpr int kObThreads = 256;
__global__ void __launch_bounds__(kObThreads) onebit_encode_kernel(const float* __restrict__ x, size_t n,
                                                                  uint8_t* __restrict__ wire, double* partials,
                                                                  unsigned* counter) {
  __shared__ double red[kObThreads / 32];
  __shared__ int bad_s[kObThreads / 32];
  __shared__ bool last;
  const size_t nwords = (n + 31) / 32, nbytes = (n + 7) / 8;
  double acc = 0.0;
  int bad = 0;
  for (size_t w = size_t(blockIdx.x) * kObThreads + threadIdx.x; w < nwords; w += size_t(gridDim.x) * kObThreads) {
    const size_t e0 = 32 * w;
    unsigned bits = 0;
    if (e0 + 32 <= n) {
      const float4* x4 = reinterpret_cast<const float4*>(x + e0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = __ldcs(x4 + q);
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          bits |= (__float_as_uint(e[j]) >> 31 ? 0u : 1u) << (4 * q + j);
          acc = __dadd_rn(acc, fabs(double(e[j])));
          bad |= !finite_f(e[j]);
        }
      }
      *reinterpret_cast<unsigned*>(wire + 4 + 4 * w) = bits;
    } else {
      for (size_t k = e0; k < n; ++k) {
        const float v = x[k];
        bits |= (__float_as_uint(v) >> 31 ? 0u : 1u) << (k - e0);
        acc = __dadd_rn(acc, fabs(double(v)));
        bad |= !finite_f(v);
      }
      for (size_t b = 4 * w; b < nbytes; ++b) wire[4 + b] = uint8_t(bits >> (8 * (b - 4 * w)));
    }
  }
  // block: fp64 partial (fixed tree order) and the non-finite flag
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
    bad |= __shfl_down_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = acc;
    bad_s[threadIdx.x >> 5] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    int any = 0;
    for (int i = 0; i < kObThreads / 32; ++i) {
      sum = __dadd_rn(sum, red[i]);
      any |= bad_s[i];
    }
    partials[2 * blockIdx.x] = sum;
    partials[2 * blockIdx.x + 1] = any ? 1.0 : 0.0;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {  // the last block: partials in block order, then the scale
    __threadfence();
    double sum = 0.0;
    bool anybad = false;
    for (unsigned i = 0; i < gridDim.x; ++i) {
      sum = __dadd_rn(sum, __ldcg(partials + 2 * i));
      anybad |= __ldcg(partials + 2 * i + 1) != 0.0;
    }
    const float scale = n ? __fdiv_rn(__double2float_rn(sum), float(n)) : 0.0f;
    *reinterpret_cast<float*>(wire) = anybad ? __int_as_float(0x7fc00000) : scale;
    *counter = 0u;
  }
}

// Codec::decode onebit (codec.cpp:110-114, kernels.cpp:65-69)
__global__ void __launch_bounds__(kObThreads) onebit_decode_kernel(const uint8_t* __restrict__ wire, size_t n,
                                                                  float* __restrict__ out) {
  const float scale = *reinterpret_cast<const float*>(wire);
  const size_t nwords = (n + 31) / 32;
  for (size_t w = size_t(blockIdx.x) * kObThreads + threadIdx.x; w < nwords; w += size_t(gridDim.x) * kObThreads) {
    const size_t e0 = 32 * w;
    if (e0 + 32 <= n) {
      const unsigned bits = *reinterpret_cast<const unsigned*>(wire + 4 + 4 * w);
      float4* o4 = reinterpret_cast<float4*>(out + e0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 v;
        v.x = (bits >> (4 * q)) & 1u ? scale : -scale;
        v.y = (bits >> (4 * q + 1)) & 1u ? scale : -scale;
        v.z = (bits >> (4 * q + 2)) & 1u ? scale : -scale;
        v.w = (bits >> (4 * q + 3)) & 1u ? scale : -scale;
        __stcs(o4 + q, v);
      }
    } else {
      for (size_t k = e0; k < n; ++k) out[k] = (wire[4 + k / 8] >> (k % 8)) & 1u ? scale : -scale;
    }
  }
}

// compensate_encode (codec.cpp:125-137) for the identity and onebit codecs:
// y = x - delta (fp32), then delta = y - D(Q(y)).  Identity: Q is the copy,
// so delta = y - y (0, NaN for non-finite y) and `flag` records a non-finite
// y (the reference's encode throws, codec.cpp:24-27).
__global__ void identity_compensate_kernel(const float* __restrict__ x, float* __restrict__ delta, size_t n,
                                           float* __restrict__ y_out, int* flag) {
  int bad = 0;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float y = __fsub_rn(x[i], delta[i]);
    y_out[i] = y;
    delta[i] = __fsub_rn(y, y);
    bad |= !finite_f(y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}
// onebit, before the encode: y = x - delta into `y` (the caller's decoded buffer)
__global__ void sub_kernel(const float* __restrict__ x, const float* __restrict__ delta, size_t n,
                           float* __restrict__ y) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    y[i] = __fsub_rn(x[i], delta[i]);
}
// onebit, after the encode: D(Q(y)) = (y not negative ? s : -s) (kernels.cpp:65-69), delta = y - D(Q(y))
__global__ void onebit_residual_kernel(const uint8_t* __restrict__ wire, float* __restrict__ y_dec,
                                       float* __restrict__ delta, size_t n) {
  const float s = *reinterpret_cast<const float*>(wire);
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const float y = y_dec[i];
    const float d = (__float_as_uint(y) >> 31) ? -s : s;
    delta[i] = __fsub_rn(y, d);
    y_dec[i] = d;
  }
}

}  // namespace

// ------------------------------------------------------- shared host utils
static thread_local std::string t_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
}
const char* last_error() { return t_err.c_str(); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

int occupancy(const void* func, int threads, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(func, dev, threads, smem);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    per_sm = 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = per_sm;
  return per_sm;
}

int persistent_grid(const void* func, int threads, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  return sm_count() * per_sm;
}

}  // namespace b2

using namespace b2;

extern "C" {

const char* b2_last_error(void) { return b2::last_error(); }

// B2_NO_PDL=1: plain launches of the small codec kernels (A/B runs)
static bool pdl_on() {
  static const bool v = [] {
    const char* e = getenv("B2_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return v;
}

// per-device scratch of the small-bucket encode: one (min, max) partial per CTA
static float2* small_partials() {
  static std::mutex mu;
  static std::map<int, float2*> per_dev;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  float2*& p = per_dev[dev];
  if (!p && cudaMalloc(&p, sizeof(float2) * 16384) != cudaSuccess) p = nullptr;
  return p;
}

extern "C++" {
// The register-resident encode for buckets up to its capacity (grid x 256
// threads x R float4); returns B2_ERR_UNSUPPORTED above it.
template <bool EC, int R>
static int try_small_encode(const float* x, float* delta, size_t n, uint8_t* codes, float* hdr, float* decoded,
                            cudaStream_t s) {
  const void* fn = reinterpret_cast<const void*>(encode_small_kernel<EC, R>);
  const int per_sm = occupancy(fn, kSmallThreads);
  if (per_sm < 1) return B2_ERR_UNSUPPORTED;
  const size_t ng = n >> 2;
  const size_t per_block = size_t(kSmallThreads) * R;
  const size_t need = (ng + per_block - 1) / per_block;  // blocks for one group per register slot
  const size_t cap = size_t(sm_count()) * size_t(per_sm);
  if (need > cap || need > 16384) return B2_ERR_UNSUPPORTED;
  // enough CTAs to spread the loads over every SM, never more than co-resident
  const int grid = int(std::max<size_t>(std::min<size_t>(cap, std::max<size_t>(need, size_t(sm_count()))), 1));
  if (size_t(grid) * per_block < ng) return B2_ERR_UNSUPPORTED;
  float2* partials = small_partials();
  if (!partials) return B2_ERR_CUDA;
  void* params[] = {&x, &delta, &n, &codes, &hdr, &decoded, &partials};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the launch with the previous kernel's tail
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  B2_CUDA_TRY(cudaLaunchKernelExC(&cfg, fn, params));
  return B2_OK;
}

template <bool EC>
static int small_encode(const float* x, float* delta, size_t n, uint8_t* codes, float* hdr, float* decoded,
                        cudaStream_t s) {
  int rc = try_small_encode<EC, 2>(x, delta, n, codes, hdr, decoded, s);
  if (rc == B2_ERR_UNSUPPORTED) rc = try_small_encode<EC, 4>(x, delta, n, codes, hdr, decoded, s);
  if (rc == B2_ERR_UNSUPPORTED) rc = try_small_encode<EC, 8>(x, delta, n, codes, hdr, decoded, s);
  return rc;
}
}  // extern "C++"

static int launch_encode(const float* x, float* delta, size_t n, uint8_t* codes, float* hdr, float* decoded,
                         cudaStream_t s) {
  if (n == 0) {  // empty input: header (0, 0), codec.cpp:52-57
    init_keys_kernel<<<1, 1, 0, s>>>(hdr, n);
    B2_CUDA_TRY(cudaGetLastError());
    return B2_OK;
  }
  const int rc = delta ? small_encode<true>(x, delta, n, codes, hdr, decoded, s)
                       : small_encode<false>(x, delta, n, codes, hdr, decoded, s);
  if (rc != B2_ERR_UNSUPPORTED) return rc;
  const void* fn = delta ? reinterpret_cast<const void*>(encode_ring_kernel<true>)
                         : reinterpret_cast<const void*>(encode_ring_kernel<false>);
  B2_CUDA_TRY(ensure_ring_smem(fn));
  void* params[] = {&x, &delta, &n, &codes, &hdr, &decoded};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(sm_count()), dim3(kRingThreads), params, kRingSmem, s));
  return B2_OK;
}

int b2_u8_encode(const float* x, size_t n, uint8_t* codes, float* hdr, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_encode: hdr is null");
  B2_REQUIRE(n == 0 || (x && codes), "b2_u8_encode: null buffer");
  B2_REQUIRE(n == 0 || aligned16(x), "b2_u8_encode: x must be 16-byte aligned");
  B2_REQUIRE(n == 0 || aligned16(codes), "b2_u8_encode: codes must be 16-byte aligned");
  return launch_encode(x, nullptr, n, codes, hdr, nullptr, static_cast<cudaStream_t>(stream));
}

int b2_u8_encode_stochastic(const float* x, size_t n, uint8_t* codes, float* hdr, uint64_t seed, void* stream) {
  int rc = b2_u8_encode(x, n, codes, hdr, stream);
  if (rc != B2_OK || n == 0) return rc;
  const int grid = int(std::min<size_t>((n + 255) / 256, size_t(sm_count()) * 8));
  u8_stochastic_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, codes, hdr, seed);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

// onebit scratch: per-block fp64 partials + the last-block counter, per device
// (per device AND stream: encodes on different streams may run concurrently)
static int onebit_scratch(double** partials, unsigned** counter, int grid, void* stream) {
  static std::mutex mu;
  static std::map<std::pair<int, void*>, std::pair<double*, unsigned*>> per_dev;
  int dev = 0;
  B2_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto& e = per_dev[{dev, stream}];
  if (!e.first) {
    B2_CUDA_TRY(cudaMalloc(&e.first, sizeof(double) * 2 * 4096));
    B2_CUDA_TRY(cudaMalloc(&e.second, sizeof(unsigned)));
    B2_CUDA_TRY(cudaMemset(e.second, 0, sizeof(unsigned)));
  }
  (void)grid;
  *partials = e.first;
  *counter = e.second;
  return B2_OK;
}

int b2_onebit_encode(const float* x, size_t n, uint8_t* wire, void* stream) {
  B2_REQUIRE(wire, "b2_onebit_encode: wire is null");
  B2_REQUIRE(n == 0 || x, "b2_onebit_encode: x is null");
  B2_REQUIRE(n == 0 || aligned16(x), "b2_onebit_encode: x must be 16-byte aligned");
  B2_REQUIRE(aligned16(wire), "b2_onebit_encode: wire must be 16-byte aligned");
  double* partials = nullptr;
  unsigned* counter = nullptr;
  const size_t nwords = (n + 31) / 32;
  const int grid = int(std::min<size_t>(std::max<size_t>((nwords + kObThreads - 1) / kObThreads, 1),
                                        size_t(sm_count()) * 4));
  int rc = onebit_scratch(&partials, &counter, grid, stream);
  if (rc) return rc;
  onebit_encode_kernel<<<grid, kObThreads, 0, static_cast<cudaStream_t>(stream)>>>(x, n, wire, partials, counter);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_onebit_decode(const uint8_t* wire, size_t n, float* out, void* stream) {
  B2_REQUIRE(wire, "b2_onebit_decode: wire is null");
  if (n == 0) return B2_OK;
  B2_REQUIRE(out, "b2_onebit_decode: out is null");
  B2_REQUIRE(aligned16(out), "b2_onebit_decode: out must be 16-byte aligned");
  B2_REQUIRE(aligned16(wire), "b2_onebit_decode: wire must be 16-byte aligned");
  const size_t nwords = (n + 31) / 32;
  const int grid = int(std::min<size_t>((nwords + kObThreads - 1) / kObThreads, size_t(sm_count()) * 4));
  onebit_decode_kernel<<<grid, kObThreads, 0, static_cast<cudaStream_t>(stream)>>>(wire, n, out);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_decode(const uint8_t* codes, const float* hdr, size_t n, float* out, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_decode: hdr is null");
  if (n == 0) return B2_OK;
  B2_REQUIRE(codes && out, "b2_u8_decode: null buffer");
  B2_REQUIRE(aligned16(out), "b2_u8_decode: out must be 16-byte aligned");
  B2_REQUIRE(aligned16(codes), "b2_u8_decode: codes must be 16-byte aligned");
  if (n <= (size_t(64) << 20)) {  // small buckets: one 32-bit load -> one float4 store per thread
    static const int V = [] {  // B2_DEC_V: codes-per-thread / 4 (A/B runs)
      const char* e = getenv("B2_DEC_V");
      const int v = e ? std::atoi(e) : 2;
      return v == 1 || v == 4 ? v : 2;
    }();
    const size_t ng = std::max<size_t>(n >> 2, 1);
    const int grid = int(std::min<size_t>((ng + V * kSmallThreads - 1) / (V * kSmallThreads),
                                          size_t(sm_count()) * 16));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_on() ? 1 : 0;
    if (V == 2)
      B2_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_small_kernel<2>, codes, hdr, n, out));
    else if (V == 4)
      B2_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_small_kernel<4>, codes, hdr, n, out));
    else
      B2_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_small_kernel<1>, codes, hdr, n, out));
    B2_CUDA_TRY(cudaGetLastError());
    return B2_OK;
  }
  B2_CUDA_TRY(ensure_ring_smem(reinterpret_cast<const void*>(decode_ring_kernel)));
  decode_ring_kernel<<<sm_count(), kRingThreads, kRingSmem, static_cast<cudaStream_t>(stream)>>>(codes, hdr, n,
                                                                                                  out);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_compensate_encode(const float* x, float* delta, size_t n, uint8_t* codes, float* hdr,
                            float* decoded, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_compensate_encode: hdr is null");
  B2_REQUIRE(n == 0 || (x && delta && codes), "b2_u8_compensate_encode: null buffer");
  B2_REQUIRE(n == 0 || (aligned16(x) && aligned16(delta) && aligned16(codes) && (!decoded || aligned16(decoded))),
             "b2_u8_compensate_encode: x, delta, codes, decoded must be 16-byte aligned");
  return launch_encode(x, delta, n, codes, hdr, decoded, static_cast<cudaStream_t>(stream));
}

static int elementwise_grid(size_t n) {
  return int(std::min<size_t>(std::max<size_t>((n + kThreads - 1) / kThreads, 1), size_t(sm_count()) * 8));
}

int b2_identity_compensate_encode(const float* x, float* delta, size_t n, float* y, int* nonfinite, void* stream) {
  B2_REQUIRE(nonfinite, "b2_identity_compensate_encode: nonfinite flag is null");
  if (n == 0) return B2_OK;
  B2_REQUIRE(x && delta && y, "b2_identity_compensate_encode: null buffer");
  identity_compensate_kernel<<<elementwise_grid(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      x, delta, n, y, nonfinite);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_onebit_compensate_encode(const float* x, float* delta, size_t n, uint8_t* wire, float* decoded,
                                void* stream) {
  B2_REQUIRE(wire && (n == 0 || (x && delta && decoded)), "b2_onebit_compensate_encode: null buffer");
  B2_REQUIRE(n == 0 || aligned16(decoded), "b2_onebit_compensate_encode: decoded must be 16-byte aligned");
  auto s = static_cast<cudaStream_t>(stream);
  if (n) {
    sub_kernel<<<elementwise_grid(n), kThreads, 0, s>>>(x, delta, n, decoded);
    B2_CUDA_TRY(cudaGetLastError());
  }
  int rc = b2_onebit_encode(decoded, n, wire, stream);
  if (rc || n == 0) return rc;
  onebit_residual_kernel<<<elementwise_grid(n), kThreads, 0, s>>>(wire, decoded, delta, n);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_pack_wire(const uint8_t* codes, const float* hdr, size_t n, uint8_t* wire, void* stream) {
  B2_REQUIRE(hdr && wire && (n == 0 || codes), "b2_u8_pack_wire: null buffer");
  const int blocks = n > 0 ? static_cast<int>((n + kThreads - 1) / kThreads) : 1;
  pack_wire_kernel<<<blocks < 1024 ? blocks : 1024, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      codes, hdr, n, wire);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_unpack_wire(const uint8_t* wire, size_t n, uint8_t* codes, float* hdr, void* stream) {
  B2_REQUIRE(hdr && wire && (n == 0 || codes), "b2_u8_unpack_wire: null buffer");
  const int blocks = n > 0 ? static_cast<int>((n + kThreads - 1) / kThreads) : 1;
  unpack_wire_kernel<<<blocks < 1024 ? blocks : 1024, kThreads, 0,
                       static_cast<cudaStream_t>(stream)>>>(wire, n, codes, hdr);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

static int flatten_impl(const float* const* ptrs, const size_t* lens, int count, float* arena,
                        int to_arena, cudaStream_t s) {
  B2_REQUIRE(count > 0, "flatten: empty tensor list");
  B2_REQUIRE(arena && ptrs && lens, "flatten: null argument");
  size_t off = 0;
  for (int i = 0; i < count; ++i) {
    B2_REQUIRE(lens[i] > 0, "flatten: zero-length tensor at position %d", i);
    B2_REQUIRE(ptrs[i], "flatten: null tensor at position %d", i);
  }
  for (int first = 0; first < count; first += kFlatMax) {
    FlatTable t{};
    t.count = (count - first) < kFlatMax ? (count - first) : kFlatMax;
    t.to_arena = to_arena;
    for (int i = 0; i < t.count; ++i) {
      t.ptr[i] = ptrs[first + i];
      t.len[i] = lens[first + i];
      t.off[i] = off;
      off += lens[first + i];
    }
    flatten_kernel<<<grid_for((const void*)flatten_kernel), kThreads, 0, s>>>(t, arena);
    B2_CUDA_TRY(cudaGetLastError());
  }
  return B2_OK;
}

int b2_bucket_flatten(const float* const* srcs, const size_t* lens, int count, float* arena,
                      void* stream) {
  return flatten_impl(srcs, lens, count, arena, 1, static_cast<cudaStream_t>(stream));
}

int b2_bucket_unflatten(const float* arena, float* const* dsts, const size_t* lens, int count,
                        void* stream) {
  return flatten_impl(const_cast<const float* const*>(dsts), lens, count, const_cast<float*>(arena), 0,
                      static_cast<cudaStream_t>(stream));
}

int b2_fill_synthetic(float* x, size_t n, uint64_t seed, uint64_t offset, void* stream) {
  if (n == 0) return B2_OK;
  B2_REQUIRE(x, "b2_fill_synthetic: null buffer");
  synth_kernel<<<grid_for((const void*)synth_kernel), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      x, n, seed, offset);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

}  // extern "C"
