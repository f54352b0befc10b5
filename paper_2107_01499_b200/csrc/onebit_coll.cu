// onebit_coll.cu -- C_LP_S with the onebit codec: the aggregation the
// reference's 1-bit Adam runs on its momentum every compressed step
// (algorithms.cpp:141-148 -> aggregate_centralized -> c_lp_s with
// Codec{onebit} and the bucket's ErrorState).
//
// Same structure as scatter_reduce_lp (collectives.cpp:91-163), one
// cooperative launch per call:
//   phase 1  every chunk k of (x - delta): sign bits (kernels.cpp:58-63) are
//            stored straight into owner k's window slot [me] over NVLink while
//            the fp64 sum |y| (kernels.cpp:26-32) accumulates; grid barrier;
//            scale_k = (float)sum / (float)n_k (codec.cpp:81-88) goes to the
//            slot header, then one release per owner.  With error feedback a
//            second local pass writes delta = y - D(P) (codec.cpp:125-137).
//   phase 2  (owner) fold D(P_j) in fp64, ranks ascending (collectives.cpp:
//            125-142), y2 = (float)acc - eps, sign bits + fp64 sum |y2| into
//            my out2, grid barrier, scale2, publish; eps = y2 - D(P2).
//   phase 3  every owner's out2 decoded into x (collectives.cpp:154-161).
//
// Layout: a warp tile is 1024 consecutive chunk elements moved as 16-byte
// quads (see encode_tile); one __ballot_sync per element column gives a
// 32-bit sign word, decode transposes the tile's 32 words once.  The words
// of a tile are one 128 B line.
//
// Exactness: signs, the ascending fp64 fold and every fp32 expression are
// the reference's.  The fp64 |y| sums are summed in a fixed tree order, not
// sequentially, so a scale can differ from the reference's by one float
// rounding when the fp64 sum is inexact (the reference's scalar and AVX2
// backends differ the same way); on inputs whose fp64 sums are exact the
// whole result is bit-identical (tests/mp_parity.py).
#include <cooperative_groups.h>

#include "b2_host.h"
#include "collectives.cuh"

namespace cg = cooperative_groups;

namespace b2 {
namespace {

constexpr int kThr = 256;
constexpr int kWarps = kThr / 32;
constexpr size_t kTile = 1024;  // elements per warp tile = 32 sign words

__device__ __forceinline__ void chunk_range(size_t n, int g, int k, size_t& lo, size_t& sz) {
  const size_t base = n / size_t(g), extra = n % size_t(g), uk = size_t(k);  // collectives.cpp:167-175
  lo = uk * base + (uk < extra ? uk : extra);
  sz = base + (uk < extra ? 1 : 0);
}

// Block sum in a fixed order (warp tree, then warps ascending); result on thread 0.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) s = __dadd_rn(s, red[i]);
  __syncthreads();
  return s;
}

// Every CTA reduces the same partials in the same order -> the same scale,
// returned to every thread of the CTA.
__device__ __forceinline__ float scale_of(const double* partials, size_t nk, double* red) {
  double v = 0.0;
  for (unsigned c = threadIdx.x; c < gridDim.x; c += kThr) v = __dadd_rn(v, __ldcg(partials + c));
  const double s = block_sum(v, red);
  if (threadIdx.x == 0) red[0] = s;
  __syncthreads();
  const double all = red[0];
  __syncthreads();
  return nk ? __fdiv_rn(__double2float_rn(all), float(nk)) : 0.0f;  // codec.cpp:82-83
}

// 32x32 bit transpose across a warp: lane i holds row word i on entry and
// column i on exit (bit r of the result = bit i of lane r's word).  Block
// swap at 16, then recursively within the 16x16, 8x8, ... blocks.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int sft = 16 >> i;
    const uint32_t m = masks[i];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
    x = (lane & sft) ? (x & ~m) | ((y & ~m) >> sft) : (x & m) | ((y & m) << sft);
  }
  return x;
}

__device__ __forceinline__ float sign_value(float y, float s) {  // D(Q(y)) for onebit
  return (__float_as_uint(y) >> 31) ? -s : s;
}

// G = the number of ranks (compile time: the fold's bit gathering unrolls).

// Internal sign-word layout of a 1024-element tile: lane l holds elements
// 128q + 4l + c (q = 0..7, c = 0..3) -- one 16-byte load per q -- and word
// 4q + c collects, in bit l, the sign of element 128q + 4l + c.  The words
// live only in the collectives' windows (b2_onebit_encode alone emits
// sign_pack's wire order), so the layout follows the 16-byte accesses.
__device__ __forceinline__ float comp(const float4& v, int c) {
  return c == 0 ? v.x : c == 1 ? v.y : c == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int c, float f) {
  if (c == 0) v.x = f; else if (c == 1) v.y = f; else if (c == 2) v.z = f; else v.w = f;
}
// elements [e, e+4) of p (zero past n); vec: p is 16-byte aligned
template <bool STREAM>
__device__ __forceinline__ float4 ld_quad(const float* p, size_t e, size_t n, bool vec) {
  if (vec && e + 4 <= n) {
    const float4* q = reinterpret_cast<const float4*>(p + e);
    return STREAM ? __ldcs(q) : __ldcg(q);
  }
  float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (e < n) v.x = p[e];
  if (e + 1 < n) v.y = p[e + 1];
  if (e + 2 < n) v.z = p[e + 2];
  if (e + 3 < n) v.w = p[e + 3];
  return v;
}
__device__ __forceinline__ void st_quad(float* p, size_t e, size_t n, bool vec, float4 v) {
  if (vec && e + 4 <= n) {
    __stcs(reinterpret_cast<float4*>(p + e), v);
    return;
  }
  if (e < n) p[e] = v.x;
  if (e + 1 < n) p[e + 1] = v.y;
  if (e + 2 < n) p[e + 2] = v.z;
  if (e + 3 < n) p[e + 3] = v.w;
}
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Sign word of this lane (word index = lane) for tile [base, base+1024) of
// y = x - d (d null: y = x), accumulating sum |y| in fp64 (kernels.cpp:26-32).
template <bool EC>
__device__ __forceinline__ uint32_t encode_tile(const float* x, const float* d, size_t base, size_t n, bool vec,
                                                int lane, double& acc) {
  float4 v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const size_t e = base + 128 * q + 4 * lane;
    v[q] = ld_quad<true>(x, e, n, vec);
    if (EC) {  // codec.cpp:131
      const float4 dq = ld_quad<true>(d, e, n, vec);
      v[q] = make_float4(__fsub_rn(v[q].x, dq.x), __fsub_rn(v[q].y, dq.y), __fsub_rn(v[q].z, dq.z),
                         __fsub_rn(v[q].w, dq.w));
    }
  }
  const bool full = base + kTile <= n;
  uint32_t word = 0;
  double acc_odd = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float y = comp(v[q], c);  // +0 past n: no |y|
      const bool in = full || base + 128 * q + 4 * lane + c < n;
      const uint32_t b = __ballot_sync(0xffffffffu, in && !(__float_as_uint(y) >> 31));
      if (lane == 4 * q + c) word = b;
      if (c & 1)
        acc_odd = __dadd_rn(acc_odd, fabs(double(y)));
      else
        acc = __dadd_rn(acc, fabs(double(y)));
    }
  }
  acc = __dadd_rn(acc, acc_odd);
  return word;
}

// Valid-bit mask of word `lane` of a tile with rem elements left.
__device__ __forceinline__ uint32_t valid_mask(size_t rem, int lane) {
  if (rem >= kTile) return 0xffffffffu;
  const size_t off = 128 * size_t(lane >> 2) + (lane & 3);
  if (rem <= off) return 0u;
  const size_t cnt = (rem - off + 3) / 4;
  return cnt >= 32 ? 0xffffffffu : (1u << cnt) - 1u;
}

template <int G, bool EC>
__global__ void __launch_bounds__(kThr) onebit_central_kernel(OnebitArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kWarps];
  __shared__ float sc[kMaxRanks];
  __shared__ float fold_tab[1 << kMaxRanks];
  __shared__ float s_in[kMaxRanks];
  __shared__ int bad_s;
  const int lane = threadIdx.x & 31;
  const size_t warp = (size_t(blockIdx.x) * kThr + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * kThr) >> 5;
  constexpr int g = G;
  const int me = a.me;
  WinHdr* myhdr = reinterpret_cast<WinHdr*>(a.win[me]);
  if (threadIdx.x == 0) bad_s = 0;
  int bad = 0;

  // ---- phase 1: signs of y = x - delta to the owners, fp64 sum |y| per chunk
  for (int i = 0; i < g; ++i) {
    const int k = (me + 1 + i) % g;  // peers first, my own chunk last
    size_t lo, nk;
    chunk_range(a.n, g, k, lo, nk);
    uint32_t* dst = reinterpret_cast<uint32_t*>(a.win[k] + a.off_recv1 + size_t(me) * a.slot_stride + 16);
    const float* xk = a.x + lo;
    const float* dk = EC ? a.delta + lo : nullptr;
    const bool vec = aligned16(xk) && (!EC || aligned16(dk));
    double acc = 0.0;
    for (size_t t = warp; t * kTile < nk; t += nwarps)
      dst[t * 32 + lane] = encode_tile<EC>(xk, dk, t * kTile, nk, vec, lane, acc);
    bad |= !isfinite(acc);  // finite |y| cannot overflow an fp64 sum
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) a.partials[size_t(k) * gridDim.x + blockIdx.x] = s;
  }
  // my NVLink stores precede CTA 0's release below (cumulativity through the barrier)
  __syncthreads();
  if (threadIdx.x == 0) fence_acq_rel_sys();
  grid.sync();
  for (int k = 0; k < g; ++k) {
    size_t lo, nk;
    chunk_range(a.n, g, k, lo, nk);
    const float s = scale_of(a.partials + size_t(k) * gridDim.x, nk, red);
    if (threadIdx.x == 0) sc[k] = s;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (threadIdx.x < g) {
      const int k = threadIdx.x;
      *reinterpret_cast<float*>(a.win[k] + a.off_recv1 + size_t(me) * a.slot_stride) = sc[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_acq_rel_sys();
      for (int k = 0; k < g; ++k) red_relaxed_sys_add(&reinterpret_cast<WinHdr*>(a.win[k])->arrive1, 1ull);
    }
  }
  if (EC) {  // delta = y - D(Q(y)), local (codec.cpp:135)
    for (int k = 0; k < g; ++k) {
      size_t lo, nk;
      chunk_range(a.n, g, k, lo, nk);
      const float s = sc[k];
      for (size_t e = size_t(blockIdx.x) * kThr + threadIdx.x; e < nk; e += size_t(gridDim.x) * kThr) {
        const float y = __fsub_rn(__ldcs(a.x + lo + e), a.delta[lo + e]);
        a.delta[lo + e] = __fsub_rn(y, sign_value(y, s));
      }
    }
  }

  // ---- phase 2 (owner of chunk me): fold, second compression
  size_t mlo, mn;
  chunk_range(a.n, g, me, mlo, mn);
  if (threadIdx.x == 0) wait_geq(&myhdr->arrive1, a.epoch * unsigned(g), a.timeout_ns, a.status);
  __syncthreads();
  const uint32_t* src[G];
#pragma unroll
  for (int j = 0; j < G; ++j)
    src[j] = reinterpret_cast<const uint32_t*>(a.win[me] + a.off_recv1 + size_t(j) * a.slot_stride + 16);
  if (threadIdx.x < g)
    s_in[threadIdx.x] = __ldcg(reinterpret_cast<const float*>(a.win[me] + a.off_recv1 + size_t(threadIdx.x) * a.slot_stride));
  __syncthreads();
  // D(P_j) is +-s_j, so (float)(sum_j ascending in fp64) depends only on the
  // g sign bits: one table of 2^g values, each folded exactly as
  // collectives.cpp:125-142 folds an element (kernels.cpp:14-16).
  for (int idx = threadIdx.x; idx < (1 << g); idx += kThr) {
    double acc = 0.0;
    for (int j = 0; j < g; ++j) acc = __dadd_rn(acc, double(((idx >> j) & 1) ? s_in[j] : -s_in[j]));
    fold_tab[idx] = __double2float_rn(acc);
  }
  __syncthreads();
  uint32_t* out2 = reinterpret_cast<uint32_t*>(a.win[me] + a.off_out2 + 16);
  if constexpr (!EC && G <= 4) {
    // Without epsilon the second payload is a boolean function of the g sign
    // words: every one of the 2^g sign patterns (minterms) is a word mask;
    // its popcount counts the elements whose y2 is fold_tab[pattern], so
    // sum |y2| = sum_pattern count * |fold_tab| (exact products in fp64).
    uint32_t cnt[1 << G];
#pragma unroll
    for (int p = 0; p < (1 << G); ++p) cnt[p] = 0;
    for (size_t t = warp; t * kTile < mn; t += nwarps) {
      const uint32_t valid = valid_mask(mn - t * kTile, lane);
      uint32_t w[G];
#pragma unroll
      for (int j = 0; j < G; ++j) w[j] = __ldcg(src[j] + t * 32 + lane);
      uint32_t word = 0;
#pragma unroll
      for (int p = 0; p < (1 << G); ++p) {
        uint32_t m = valid;
#pragma unroll
        for (int j = 0; j < G; ++j) m &= ((p >> j) & 1) ? w[j] : ~w[j];
        cnt[p] += __popc(m);
        if (!(__float_as_uint(fold_tab[p]) >> 31)) word |= m;  // sign_pack of y2
      }
      out2[t * 32 + lane] = word;
    }
    double acc2 = 0.0;
#pragma unroll
    for (int p = 0; p < (1 << G); ++p) {
      acc2 = __dadd_rn(acc2, double(cnt[p]) * fabs(double(fold_tab[p])));
      bad |= cnt[p] && !finite_f(fold_tab[p]);
    }
    const double s = block_sum(acc2, red);
    if (threadIdx.x == 0) a.partials[size_t(g) * gridDim.x + blockIdx.x] = s;
  } else {
    double acc2 = 0.0;
    for (size_t t = warp; t * kTile < mn; t += nwarps) {
      const size_t base = t * kTile;
      const bool full = base + kTile <= mn;
      uint32_t col[G];  // lane l: bit 4q+c = rank j's sign of element 128q + 4l + c
#pragma unroll
      for (int j = 0; j < G; ++j) col[j] = transpose32(__ldcg(src[j] + t * 32 + lane), lane);
      uint32_t word = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const size_t e = base + 128 * q + 4 * lane;
        float4 ev = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (EC) ev = ld_quad<false>(a.eps, e, mn, true);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int k = 4 * q + c;
          const bool in = full || e + c < mn;
          uint32_t idx = 0;
#pragma unroll
          for (int j = 0; j < G; ++j) idx |= ((col[j] >> k) & 1u) << j;
          float y2 = fold_tab[idx];
          if (EC) {
            y2 = __fsub_rn(y2, comp(ev, c));  // compensate_encode with epsilon
            set_comp(ev, c, y2);              // stash y2 until scale2 is known
          }
          if (!in) y2 = 0.0f;
          const uint32_t b = __ballot_sync(0xffffffffu, in && !(__float_as_uint(y2) >> 31));
          if (lane == k) word = b;
          acc2 = __dadd_rn(acc2, fabs(double(y2)));
        }
        if (EC) st_quad(a.eps, e, mn, true, ev);
      }
      out2[t * 32 + lane] = word;
    }
    bad |= !isfinite(acc2);
    const double s = block_sum(acc2, red);
    if (threadIdx.x == 0) a.partials[size_t(g) * gridDim.x + blockIdx.x] = s;
  }
  if (bad) atomicOr(&bad_s, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (bad_s) latch(a.status, kStatusNonFinite);  // codec.cpp:24-27 (the reference throws)
    fence_acq_rel_sys();
  }
  grid.sync();
  const float s2 = scale_of(a.partials + size_t(g) * gridDim.x, mn, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __stcg(reinterpret_cast<float*>(a.win[me] + a.off_out2), s2);
    fence_acq_rel_sys();
    st_release_sys(&myhdr->ready2, a.epoch);  // publish (collectives.cpp:150-151)
  }
  if (EC) {  // epsilon = y2 - D(Q(y2))
    for (size_t e = size_t(blockIdx.x) * kThr + threadIdx.x; e < mn; e += size_t(gridDim.x) * kThr) {
      const float y2 = __ldcg(a.eps + e);  // stashed by another CTA: read through L2
      a.eps[e] = __fsub_rn(y2, sign_value(y2, s2));
    }
  }

  // ---- phase 3: decode every owner's second payload into x
  for (int i = 0; i < g; ++i) {
    const int k = (me + i) % g;  // my own (local) first
    size_t lo, nk;
    chunk_range(a.n, g, k, lo, nk);
    if (threadIdx.x == 0) wait_geq(&reinterpret_cast<WinHdr*>(a.win[k])->ready2, a.epoch, a.timeout_ns, a.status);
    __syncthreads();
    const float s = __ldcg(reinterpret_cast<const float*>(a.win[k] + a.off_out2));
    const uint32_t* bits = reinterpret_cast<const uint32_t*>(a.win[k] + a.off_out2 + 16);
    float* xk = a.x + lo;
    const bool vec = aligned16(xk);
    for (size_t t = warp; t * kTile < nk; t += nwarps) {
      const size_t base = t * kTile;
      const uint32_t col = transpose32(__ldcg(bits + t * 32 + lane), lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o;
#pragma unroll
        for (int c = 0; c < 4; ++c) set_comp(o, c, ((col >> (4 * q + c)) & 1u) ? s : -s);  // kernels.cpp:65-69
        st_quad(xk, base + 128 * q + 4 * lane, nk, vec, o);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) fail_epilogue(a.status);
}


// ---------------------------------------------------------------- D_LP_S
// d_lp_s with Codec{onebit} (collectives.cpp:260-288): one encode of the
// whole bucket (one scale), x' = (float)((sum_{j in N, ascending} (double)
// D(P_j)) * inv).  D(P_j) = +-s_j, so x' is a function of the |N| sign bits:
// a 2^|N| table folded exactly as the reference folds one element.
template <int NB>
__global__ void __launch_bounds__(kThr) onebit_decent_kernel(OnebitDecentArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kWarps];
  __shared__ float tab[1 << NB];
  __shared__ float s_nb[NB];
  const int lane = threadIdx.x & 31;
  const size_t warp = (size_t(blockIdx.x) * kThr + threadIdx.x) >> 5;
  const size_t nwarps = (size_t(gridDim.x) * kThr) >> 5;
  const size_t n = a.n;
  const int p = a.parity;
  WinHdr* myhdr = reinterpret_cast<WinHdr*>(a.win[a.me]);
  uint8_t* mine = a.win[a.me] + a.off_dbuf;

  // my dbuf[p] is free once the neighbours of two calls ago have read it
  if (threadIdx.x == 0) wait_geq(&myhdr->dreads[p], a.expected_reads, a.timeout_ns, a.status);
  __syncthreads();

  // encode: sign words into my window, fp64 sum |x| (kernels.cpp:26-32, 58-63)
  uint32_t* bits = reinterpret_cast<uint32_t*>(mine + 16);
  double acc = 0.0;
  for (size_t t = warp; t * kTile < n; t += nwarps)
    bits[t * 32 + lane] = encode_tile<false>(a.x, nullptr, t * kTile, n, true, lane, acc);
  const bool bad = !isfinite(acc);  // finite |x| cannot overflow an fp64 sum
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) a.partials[blockIdx.x] = s;
  if (__syncthreads_or(bad) && threadIdx.x == 0) latch(a.status, kStatusNonFinite);  // codec.cpp:24-27
  if (threadIdx.x == 0) fence_acq_rel_sys();  // my sign words precede CTA 0's publication
  grid.sync();
  const float scale = scale_of(a.partials, n, red);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __stcg(reinterpret_cast<float*>(mine), scale);
    fence_acq_rel_sys();
    st_release_sys(&myhdr->dready[p], a.epoch);
  }

  // gather the neighbours' payloads (self included), fold by table
  if (threadIdx.x < NB) {
    const uint8_t* w = a.win[a.nbrs[threadIdx.x]] + a.off_dbuf;
    wait_geq(&reinterpret_cast<const WinHdr*>(a.win[a.nbrs[threadIdx.x]])->dready[p], a.epoch, a.timeout_ns,
             a.status);
    s_nb[threadIdx.x] = __ldcg(reinterpret_cast<const float*>(w));
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < (1 << NB); idx += kThr) {
    double f = 0.0;
    for (int i = 0; i < NB; ++i) f = __dadd_rn(f, double(((idx >> i) & 1) ? s_nb[i] : -s_nb[i]));
    tab[idx] = __double2float_rn(__dmul_rn(f, a.inv));  // collectives.cpp:282-286
  }
  __syncthreads();
  const uint32_t* src[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) src[i] = reinterpret_cast<const uint32_t*>(a.win[a.nbrs[i]] + a.off_dbuf + 16);
  for (size_t t = warp; t * kTile < n; t += nwarps) {
    const size_t base = t * kTile;
    uint32_t col[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) col[i] = transpose32(__ldcg(src[i] + t * 32 + lane), lane);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 o;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t idx = 0;
#pragma unroll
        for (int i = 0; i < NB; ++i) idx |= ((col[i] >> (4 * q + c)) & 1u) << i;
        set_comp(o, c, tab[idx]);
      }
      st_quad(a.x, base + 128 * q + 4 * lane, n, true, o);
    }
  }
  // my reads of the neighbours' windows are done: one credit to each of them
  __syncthreads();
  if (threadIdx.x == 0) fence_acq_rel_sys();
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x < NB && a.nbrs[threadIdx.x] != a.me)
    red_release_sys_add(&reinterpret_cast<WinHdr*>(a.win[a.nbrs[threadIdx.x]])->dreads[p], 1ull);
  if (threadIdx.x == 0) fail_epilogue(a.status);
}
}  // namespace

template <int G>
const void* onebit_fn(bool ec) {
  return ec ? reinterpret_cast<const void*>(onebit_central_kernel<G, true>)
            : reinterpret_cast<const void*>(onebit_central_kernel<G, false>);
}

int launch_onebit_central(const OnebitArgs& a, bool ec, cudaStream_t s, int sms) {
  const void* fn = nullptr;
  switch (a.g) {
    case 1: fn = onebit_fn<1>(ec); break;
    case 2: fn = onebit_fn<2>(ec); break;
    case 3: fn = onebit_fn<3>(ec); break;
    case 4: fn = onebit_fn<4>(ec); break;
    case 5: fn = onebit_fn<5>(ec); break;
    case 6: fn = onebit_fn<6>(ec); break;
    case 7: fn = onebit_fn<7>(ec); break;
    case 8: fn = onebit_fn<8>(ec); break;
    default: set_error("onebit c_lp_s: %d ranks (1..%d supported)", a.g, kMaxRanks); return B2_ERR_INVALID;
  }
  const int grid = budget_grid(persistent_grid(fn, kThr), sms);
  OnebitArgs args = a;
  void* params[] = {&args};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThr), params, 0, s));
  return B2_OK;
}

int launch_onebit_decent(const OnebitDecentArgs& a, cudaStream_t s, int sms) {
  const void* fn = nullptr;
  switch (a.nnb) {
    case 1: fn = reinterpret_cast<const void*>(onebit_decent_kernel<1>); break;
    case 2: fn = reinterpret_cast<const void*>(onebit_decent_kernel<2>); break;
    case 3: fn = reinterpret_cast<const void*>(onebit_decent_kernel<3>); break;
    case 4: fn = reinterpret_cast<const void*>(onebit_decent_kernel<4>); break;
    case 5: fn = reinterpret_cast<const void*>(onebit_decent_kernel<5>); break;
    case 6: fn = reinterpret_cast<const void*>(onebit_decent_kernel<6>); break;
    case 7: fn = reinterpret_cast<const void*>(onebit_decent_kernel<7>); break;
    case 8: fn = reinterpret_cast<const void*>(onebit_decent_kernel<8>); break;
    default: set_error("onebit d_lp_s: %d neighbours (1..%d supported)", a.nnb, kMaxRanks); return B2_ERR_INVALID;
  }
  const int grid = budget_grid(persistent_grid(fn, kThr), sms);
  OnebitDecentArgs args = a;
  void* params[] = {&args};
  B2_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThr), params, 0, s));
  return B2_OK;
}

// bytes of one onebit window slot for chunks of at most maxchunk elements
size_t onebit_slot_bytes(size_t maxchunk) {
  const size_t words = (maxchunk + kTile - 1) / kTile * 32;
  return (16 + 4 * words + 255) / 256 * 256;
}

}  // namespace b2
