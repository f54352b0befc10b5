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

#include <mutex>
#include <vector>

#include "b2_device.cuh"
#include "b2_host.h"

namespace b2 {
namespace {

constexpr int U = 4;  // 4 x 16-byte loads in flight per thread per iteration

__device__ __forceinline__ unsigned key_of(float f) {
  const unsigned b = __float_as_uint(f);
  return b ^ ((b >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ float float_of(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

// Pass 1: per-CTA (min, max) of y = x (- delta), folded into keys[0..1].
template <bool EC>
__global__ void __launch_bounds__(kThreads) minmax_keys_kernel(const float* __restrict__ x,
                                                               const float* __restrict__ delta,
                                                               size_t n, unsigned* keys) {
  __shared__ float2 red[32];
  const Span sp = make_span(0, n);
  float lo = __int_as_float(0x7f800000), hi = -__int_as_float(0x7f800000);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* d4 = reinterpret_cast<const float4*>(delta);
  for (size_t base = sp.g0 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; base < sp.g1;
       base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) {
        v[u] = ld_stream(x4 + gi);
        if (EC) v[u] = sub4(v[u], ld_stream(d4 + gi));
      } else {
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * stride < sp.g1) {
        lo = fmin_nan(lo, fmin_nan(fmin_nan(v[u].x, v[u].y), fmin_nan(v[u].z, v[u].w)));
        hi = fmax_nan(hi, fmax_nan(fmax_nan(v[u].x, v[u].y), fmax_nan(v[u].z, v[u].w)));
      }
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 8) {  // unaligned head / tail
    const size_t e = threadIdx.x < 4 ? sp.s + threadIdx.x : sp.tail_begin + (threadIdx.x - 4);
    const bool in = threadIdx.x < 4 ? e < sp.head_end : e < sp.s + sp.n;
    if (in) {
      float v = x[e];
      if (EC) v = __fsub_rn(v, delta[e]);
      lo = fmin_nan(lo, v);
      hi = fmax_nan(hi, v);
    }
  }
  const float2 r = block_minmax(lo, hi, red);
  if (threadIdx.x == 0) {
    if (r.x != r.x || r.y != r.y) {
      atomicMax(keys + 1, 0xffffffffu);  // NaN -> the max key decodes to NaN
    } else {
      atomicMin(keys + 0, key_of(r.x));
      atomicMax(keys + 1, key_of(r.y));
    }
  }
}

// Pass 2: codes = Q(y); with EC also delta = y - D(Q(y)) and decoded.
template <bool EC>
__global__ void __launch_bounds__(kThreads) quantize_kernel(const float* __restrict__ x,
                                                            float* __restrict__ delta, size_t n,
                                                            uint8_t* __restrict__ codes, float* hdr,
                                                            float* __restrict__ decoded) {
  const unsigned* keys = reinterpret_cast<const unsigned*>(hdr + 2);
  const float lo = float_of(__ldcg(keys + 0)), hi = float_of(__ldcg(keys + 1));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hdr[0] = lo;
    hdr[1] = hi;
  }
  const U8Params p = u8_params(lo, hi);
  const Span sp = make_span(0, n);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* d4 = reinterpret_cast<float4*>(delta);
  uint32_t* c4 = reinterpret_cast<uint32_t*>(codes);
  for (size_t base = sp.g0 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; base < sp.g1;
       base += stride * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) {
        v[u] = ld_stream(x4 + gi);
        if (EC) v[u] = sub4(v[u], d4[gi]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) {
        const uint32_t q = quantize4(v[u], p.lo, p.inv);
        st_stream(c4 + gi, q);
        if (EC) {
          const float4 d = dequant4(q, p.lo, p.step);
          d4[gi] = sub4(v[u], d);
          if (decoded) st_stream(reinterpret_cast<float4*>(decoded) + gi, d);
        }
      }
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 8) {
    const size_t e = threadIdx.x < 4 ? sp.s + threadIdx.x : sp.tail_begin + (threadIdx.x - 4);
    const bool in = threadIdx.x < 4 ? e < sp.head_end : e < sp.s + sp.n;
    if (in) {
      float v = x[e];
      if (EC) v = __fsub_rn(v, delta[e]);
      const uint8_t q = quantize1(v, p.lo, p.inv);
      codes[e] = q;
      if (EC) {
        const float d = dequant1(q, p.lo, p.step);
        delta[e] = __fsub_rn(v, d);
        if (decoded) decoded[e] = d;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) decode_kernel(const uint8_t* __restrict__ codes,
                                                          const float* hdr, size_t n,
                                                          float* __restrict__ out) {
  const float lo = hdr[0], hi = hdr[1];
  const float step = __fdiv_rn(__fsub_rn(hi, lo), 255.0f);
  const Span sp = make_span(0, n);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  const uint32_t* c4 = reinterpret_cast<const uint32_t*>(codes);
  float4* o4 = reinterpret_cast<float4*>(out);
  for (size_t base = sp.g0 + size_t(blockIdx.x) * blockDim.x + threadIdx.x; base < sp.g1;
       base += stride * U) {
    uint32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t gi = base + u * stride;
      c[u] = gi < sp.g1 ? ld_stream(c4 + gi) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t gi = base + u * stride;
      if (gi < sp.g1) st_stream(o4 + gi, dequant4(c[u], lo, step));
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < 8) {
    const size_t e = threadIdx.x < 4 ? sp.s + threadIdx.x : sp.tail_begin + (threadIdx.x - 4);
    const bool in = threadIdx.x < 4 ? e < sp.head_end : e < sp.s + sp.n;
    if (in) out[e] = dequant1(codes[e], lo, step);
  }
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

int grid_for(const void* f) { return persistent_grid(f, kThreads); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

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

int b2_u8_encode(const float* x, size_t n, uint8_t* codes, float* hdr, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_encode: hdr is null");
  B2_REQUIRE(n == 0 || (x && codes), "b2_u8_encode: null buffer");
  B2_REQUIRE(n == 0 || aligned16(x), "b2_u8_encode: x must be 16-byte aligned");
  B2_REQUIRE(n == 0 || (reinterpret_cast<uintptr_t>(codes) & 3) == 0,
             "b2_u8_encode: codes must be 4-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  init_keys_kernel<<<1, 1, 0, s>>>(hdr, n);
  if (n) {
    minmax_keys_kernel<false><<<grid_for((const void*)minmax_keys_kernel<false>), kThreads, 0, s>>>(
        x, nullptr, n, reinterpret_cast<unsigned*>(hdr + 2));
    quantize_kernel<false><<<grid_for((const void*)quantize_kernel<false>), kThreads, 0, s>>>(
        x, nullptr, n, codes, hdr, nullptr);
  }
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_decode(const uint8_t* codes, const float* hdr, size_t n, float* out, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_decode: hdr is null");
  if (n == 0) return B2_OK;
  B2_REQUIRE(codes && out, "b2_u8_decode: null buffer");
  B2_REQUIRE(aligned16(out), "b2_u8_decode: out must be 16-byte aligned");
  B2_REQUIRE((reinterpret_cast<uintptr_t>(codes) & 3) == 0,
             "b2_u8_decode: codes must be 4-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  decode_kernel<<<grid_for((const void*)decode_kernel), kThreads, 0, s>>>(codes, hdr, n, out);
  B2_CUDA_TRY(cudaGetLastError());
  return B2_OK;
}

int b2_u8_compensate_encode(const float* x, float* delta, size_t n, uint8_t* codes, float* hdr,
                            float* decoded, void* stream) {
  B2_REQUIRE(hdr, "b2_u8_compensate_encode: hdr is null");
  B2_REQUIRE(n == 0 || (x && delta && codes), "b2_u8_compensate_encode: null buffer");
  B2_REQUIRE(n == 0 || (aligned16(x) && aligned16(delta) && (!decoded || aligned16(decoded))),
             "b2_u8_compensate_encode: x, delta, decoded must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  init_keys_kernel<<<1, 1, 0, s>>>(hdr, n);
  if (n) {
    minmax_keys_kernel<true><<<grid_for((const void*)minmax_keys_kernel<true>), kThreads, 0, s>>>(
        x, delta, n, reinterpret_cast<unsigned*>(hdr + 2));
    quantize_kernel<true><<<grid_for((const void*)quantize_kernel<true>), kThreads, 0, s>>>(
        x, delta, n, codes, hdr, decoded);
  }
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
