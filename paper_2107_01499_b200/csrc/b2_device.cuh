// b2_device.cuh -- device-side building blocks shared by every kernel.
//
// Exact-arithmetic rules (SURVEY.md 7 "Hard parts"): the reference compiles
// without FMA (kernels_avx2.cpp:36,122), uses IEEE division and
// round-half-even, and accumulates in double from +0.0 in ascending rank
// order.  Every float op below is an explicit _rn intrinsic so nvcc cannot
// contract or reassociate it.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b2 {

constexpr int kThreads = 512;     // threads per CTA for every persistent kernel
constexpr int kMaxRanks = 8;
// 16-byte units per arrival region of a gated pass (ring.cuh PassDesc::gate)
constexpr int kGateUnits = 2048;

// ------------------------------------------------------------ float helpers

// min/max with NaN propagation (PTX min.NaN / max.NaN): a NaN anywhere in the
// chunk survives to the header, which is how non-finite input is detected
// without a separate check_finite pass (codec.cpp:24-27).  +-Inf survive as
// the min or max themselves.
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ bool finite_f(float v) {
  return (__float_as_uint(v) & 0x7f800000u) != 0x7f800000u;
}

// Warp-wide NaN-propagating min/max via redux.sync (sm_100a, needs
// -gencode arch=compute_100a,code=sm_100a).
__device__ __forceinline__ float warp_min_nan(float v) {
  float r;
  asm volatile("redux.sync.min.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float warp_max_nan(float v) {
  float r;
  asm volatile("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// Block-wide (lo, hi) reduction; result valid in every thread.
__device__ __forceinline__ float2 block_minmax(float lo, float hi, float2* smem /*[32]*/) {
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) smem[w] = make_float2(lo, hi);
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float2 v = l < nw ? smem[l] : smem[0];
  lo = warp_min_nan(v.x);
  hi = warp_max_nan(v.y);
  return make_float2(lo, hi);
}

// ------------------------------------------------ uniform8 element math
// quantize_u8 (kernels.cpp:43-50): q = clamp(nearbyint((x - lo) * inv), 0, 255)
// with one rounding per operation.  Clamping first and then adding 1.5*2^23
// rounds half-to-even exactly like nearbyintf for |v| <= 255 and leaves the
// level in the low byte; NaN clamps to 0 (the x86 scalar path also yields 0),
// +Inf to 255.  Everything stays on the FMA/ALU pipes (no F2I).
__device__ __forceinline__ uint32_t level_bits(float x, float lo, float inv) {
  float v = __fmul_rn(__fsub_rn(x, lo), inv);
  v = fminf(fmaxf(v, 0.0f), 255.0f);
  return __float_as_uint(__fadd_rn(v, 12582912.0f));  // low byte = level
}
__device__ __forceinline__ uint8_t quantize1(float x, float lo, float inv) {
  return static_cast<uint8_t>(level_bits(x, lo, inv) & 0xffu);
}
__device__ __forceinline__ uint32_t quantize4(float4 v, float lo, float inv) {
  const uint32_t a = level_bits(v.x, lo, inv), b = level_bits(v.y, lo, inv);
  const uint32_t c = level_bits(v.z, lo, inv), d = level_bits(v.w, lo, inv);
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Stochastic rounding inside the collectives (Codec{uniform8,
// Rounding::stochastic}, codec.cpp:67-78): level = floor(q) + (u < q -
// floor(q)), clamped to [0, 255], u uniform in [0, 1) with 24 random bits
// (std::uniform_real_distribution<float>'s resolution) from a counter hash of
// (per-call key, element index) -- the reference draws u from the caller's
// host mt19937 stream, so only the distribution (unbiased levels) is shared.
struct Rounder {
  unsigned long long key;  // 0 with on == false
  bool on;
};
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// per call, rank and encode phase (1: the first encode, 2: the owner's second)
__device__ __forceinline__ Rounder make_rounder(bool on, unsigned long long seed, int rank, int phase) {
  return Rounder{on ? mix64(seed ^ mix64((unsigned long long)(rank + 1) * 0x100000001b3ULL + (unsigned long long)phase))
                    : 0ull,
                 on};
}
__device__ __forceinline__ uint32_t level_sr(float x, float lo, float inv, unsigned long long key, size_t e) {
  const float q = __fmul_rn(__fsub_rn(x, lo), inv);
  const float fl = floorf(q);
  const float u = float(uint32_t(mix64(key + e) >> 40)) * 0x1p-24f;
  float level = __fadd_rn(fl, u < __fsub_rn(q, fl) ? 1.0f : 0.0f);
  level = fminf(fmaxf(level, 0.0f), 255.0f);  // NaN -> 0 like the nearest path
  return uint32_t(level);
}
// quantize with the call's rounding; e = index of the (first) element
__device__ __forceinline__ uint8_t q1r(float x, float lo, float inv, const Rounder& r, size_t e) {
  return r.on ? uint8_t(level_sr(x, lo, inv, r.key, e)) : quantize1(x, lo, inv);
}
__device__ __forceinline__ uint32_t q4r(float4 v, float lo, float inv, const Rounder& r, size_t e) {
  if (!r.on) return quantize4(v, lo, inv);
  return level_sr(v.x, lo, inv, r.key, e) | (level_sr(v.y, lo, inv, r.key, e + 1) << 8) |
         (level_sr(v.z, lo, inv, r.key, e + 2) << 16) | (level_sr(v.w, lo, inv, r.key, e + 3) << 24);
}

// dequantize_u8 (kernels.cpp:52-56): lo + (float)q * step, rounded multiply
// then rounded add.  (float)q via the 2^23 magic: PRMT + FADD, exact.
template <int K>
__device__ __forceinline__ float level_f(uint32_t codes) {
  return __fsub_rn(__uint_as_float(__byte_perm(codes, 0x4B000000u, 0x7440 | K)), 8388608.0f);
}
__device__ __forceinline__ float dequant1(uint8_t q, float lo, float step) {
  return __fadd_rn(lo, __fmul_rn(static_cast<float>(q), step));
}
__device__ __forceinline__ float4 dequant4(uint32_t c, float lo, float step) {
  float4 r;
  r.x = __fadd_rn(lo, __fmul_rn(level_f<0>(c), step));
  r.y = __fadd_rn(lo, __fmul_rn(level_f<1>(c), step));
  r.z = __fadd_rn(lo, __fmul_rn(level_f<2>(c), step));
  r.w = __fadd_rn(lo, __fmul_rn(level_f<3>(c), step));
  return r;
}

// Codec parameters from a (min, max) header (codec.cpp:61,66,106).
struct U8Params {
  float lo, inv, step;
  float c23;        // -(2^23 * step), exact: lets one FFMA produce fl32(q * step)
  bool fastdec;     // c23 and (2^23 + 255) * step are finite -> dequant via FFMA
  bool degenerate;  // range == 0: all codes 0 (codec.cpp:62-64)
};
__device__ __forceinline__ U8Params u8_params(float lo, float hi) {
  U8Params p;
  const float range = __fsub_rn(hi, lo);
  p.lo = lo;
  p.degenerate = (range == 0.0f);
  p.inv = p.degenerate ? 0.0f : __fdiv_rn(255.0f, range);
  p.step = __fdiv_rn(range, 255.0f);
  p.c23 = __fmul_rn(-8388608.0f, p.step);
  p.fastdec = fabsf(p.step) < 0x1p100f;  // also false for NaN / Inf
  return p;
}

// dequant with the parameters above.  Fast form: (2^23 + q) is the magic
// float m (PRMT only); fma(m, step, -2^23 step) = round((2^23 + q) step -
// 2^23 step) = round(q * step) -- the exact product rounded ONCE, i.e. the
// reference's rounded multiply -- then the rounded add.  3 ops per element.
template <int K>
__device__ __forceinline__ float magic_q(uint32_t codes) {
  return __uint_as_float(__byte_perm(codes, 0x4B000000u, 0x7440 | K));
}
__device__ __forceinline__ float4 dequant4_fast(uint32_t c, float lo, float step, float c23) {
  float4 r;
  r.x = __fadd_rn(lo, __fmaf_rn(magic_q<0>(c), step, c23));
  r.y = __fadd_rn(lo, __fmaf_rn(magic_q<1>(c), step, c23));
  r.z = __fadd_rn(lo, __fmaf_rn(magic_q<2>(c), step, c23));
  r.w = __fadd_rn(lo, __fmaf_rn(magic_q<3>(c), step, c23));
  return r;
}
__device__ __forceinline__ float4 dequant4(uint32_t c, const U8Params& p) {
  return p.fastdec ? dequant4_fast(c, p.lo, p.step, p.c23) : dequant4(c, p.lo, p.step);
}
__device__ __forceinline__ float dequant1(uint8_t q, const U8Params& p) { return dequant1(q, p.lo, p.step); }

__device__ __forceinline__ float4 sub4(float4 a, float4 b) {
  return make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z),
                     __fsub_rn(a.w, b.w));
}

// ------------------------------------------------------------- memory ops
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {  // read-once data
  return __ldcs(p);
}
template <typename T>
__device__ __forceinline__ void st_stream(T* p, T v) {
  __stcs(p, v);
}
// Peer (NVLink) data: bypass L1 so a line cached earlier in this kernel can
// never be returned stale after a flag acquire.
__device__ __forceinline__ uint32_t ld_peer_u32(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ float4 ld_peer_f4(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ float2 ld_peer_f2(const float2* p) { return __ldcg(p); }

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Status bits latched into the communicator's mapped status word.
enum : int { kStatusNonFinite = 1, kStatusTimeout = 2 };

// Failure context of one window (device memory, built by the communicator):
// the mapped host status word and every rank's poison word (WinHdr::poison).
// A rendezvous timeout POISONS the window on every rank before this rank
// publishes anything else: a late peer that passes its (cumulative) waits and
// consumes data published after the timeout sees the poison at its kernel end
// (fail_epilogue) and latches B2_ERR_TIMEOUT instead of returning success; the
// host then refuses every further launch on the communicator (comm.cu).
struct Fail {
  int* host;                             // mapped host status word
  unsigned long long* mine;              // my window's poison word
  unsigned long long* peer[kMaxRanks];   // every rank's poison word (peer-mapped; [me] == mine)
  int n;
};

__device__ __forceinline__ void latch(Fail* f, int bit) {
  atomicOr_system(f->host, bit);
  if (bit & kStatusTimeout) {
    for (int j = 0; j < f->n; ++j)
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(f->peer[j]), "l"(1ull) : "memory");
    __threadfence_system();  // the poison is visible before anything this rank publishes later
  }
}
__device__ __forceinline__ bool poisoned(const Fail* f) {
  return *reinterpret_cast<volatile unsigned long long*>(f->mine) != 0ull;
}

// Spin until *flag >= target (acquire, system scope) or the timeout expires.
// Returns false on timeout (status latched, every rank's window poisoned) so
// the caller can fall through instead of hanging the GPU; a window that is
// already poisoned (by this rank or a peer) fails every wait at once.
__device__ __forceinline__ bool wait_geq(const unsigned long long* flag, unsigned long long target,
                                         unsigned long long timeout_ns, Fail* f) {
  if (ld_acquire_sys(flag) >= target) return true;
  const unsigned long long t0 = globaltimer();
  unsigned ns = 32;
  while (ld_acquire_sys(flag) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (poisoned(f)) {
      atomicOr_system(f->host, kStatusTimeout);
      return false;
    }
    if (globaltimer() - t0 > timeout_ns) {
      latch(f, kStatusTimeout);
      return false;
    }
  }
  return true;
}

// Kernel epilogue (one thread per CTA, after the CTA's last wait): a poison
// set by a peer that timed out in this call turns the call into an error.
__device__ __forceinline__ void fail_epilogue(Fail* f) {
  if (f && poisoned(f)) atomicOr_system(f->host, kStatusTimeout);
}

// --------------------------------------------------- work decomposition
// A range [s, s+n) of a 16-byte-aligned fp32 buffer splits into an unaligned
// head (< 4 elements), a body of aligned 4-element groups and a tail.
struct Span {
  size_t s, n;          // element range
  size_t g0, g1;        // body groups [g0, g1): elements [4*g0, 4*g1)
  size_t head_end;      // head = [s, head_end)
  size_t tail_begin;    // tail = [tail_begin, s+n)
};
__host__ __device__ __forceinline__ Span make_span(size_t s, size_t n) {
  Span sp;
  sp.s = s;
  sp.n = n;
  const size_t e = s + n;
  size_t a = (s + 3) & ~size_t(3);
  if (a > e) a = e;
  size_t b = e & ~size_t(3);
  if (b < a) b = a;
  sp.head_end = a;
  sp.tail_begin = b;
  sp.g0 = a >> 2;
  sp.g1 = b >> 2;
  return sp;
}

}  // namespace b2
