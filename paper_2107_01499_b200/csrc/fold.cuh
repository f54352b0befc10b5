// fold.cuh -- the owner-side reduction of g decoded contributions:
// acc = ((0.0 + d_0) + d_1) + ... in fp64, ascending source order, rounded
// to fp32 once (kernels.cpp:14-16 add_f64; collectives.cpp:127-142).  This is
// the compute hot spot of phase 2: every term needs an F2F.F64.F32 (16/clk/SM
// on B200, measured by tests/cpp/probe.cu), so the loop is written for ILP.
#pragma once

#include "b2_device.cuh"
#include "collectives.cuh"

namespace b2 {

// Exact fp32 -> fp64 widening without the XU pipe: reinterpret the float's
// sign/exponent/mantissa as a double whose exponent field holds the FLOAT
// bias, i.e. the double equals f * 2^-896 exactly for every finite f
// (normal, subnormal, +-0).  Two ALU ops for the high word, one for the low.
__device__ __forceinline__ double widen_scaled(float f) {
  const int b = __float_as_int(f);
  return __hiloint2double(static_cast<int>(static_cast<unsigned>(b >> 3) & 0x8FFFFFFFu),
                          static_cast<int>(static_cast<unsigned>(b) << 29));
}
// acc + (double)f with ONE rounding: the product widen_scaled(f) * 2^896 is
// exact (power-of-two scaling back to f), so the fused multiply-add rounds
// exactly like __dadd_rn(acc, double(f)) -- including 0.0 + (-0.0) = +0.0.
// Valid for finite f only; callers route non-finite data to the F2F path.
__device__ __forceinline__ double add_widen(double acc, float f) {
  return __fma_rn(widen_scaled(f), 0x1p896, acc);
}

// fp64 ascending fold of nsrc decoded contributions of one group
template <int CODEC>
__device__ __forceinline__ float4 fold_group(const uint8_t* st, int gi, int nsrc, int T, const float* lo,
                                             const float* step) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int j = 0; j < nsrc; ++j) {
    float4 d;
    if (CODEC == kU8) {
      const uint32_t c = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16)[gi];
      d = dequant4(c, lo[j], step[j]);
    } else {
      d = reinterpret_cast<const float4*>(st + size_t(j) * T * 64)[gi];
    }
    a0 = __dadd_rn(a0, double(d.x));
    a1 = __dadd_rn(a1, double(d.y));
    a2 = __dadd_rn(a2, double(d.z));
    a3 = __dadd_rn(a3, double(d.w));
  }
  return make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2),
                     __double2float_rn(a3));
}


// Fast fold of two groups (8 independent fp64 chains in flight per thread)
// with the XU-free widening.  Requires every decoded term to be finite:
// uint8 sources whose header bounds |d| below FLT_MAX (fold_fast_ok) decode
// to finite values by construction.
template <int CODEC>
__device__ __forceinline__ void fold_group2_fast(const uint8_t* st, int gi0, int gi1, int nsrc, int T,
                                                 const float* lo, const float* step, float4& r0, float4& r1) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  for (int j = 0; j < nsrc; ++j) {
    float4 d, e;
    if (CODEC == kU8) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16);
      const uint32_t c0 = cs[gi0], c1 = cs[gi1];
      d = dequant4(c0, lo[j], step[j]);
      e = dequant4(c1, lo[j], step[j]);
    } else {
      const float4* fs = reinterpret_cast<const float4*>(st + size_t(j) * T * 64);
      d = fs[gi0];
      e = fs[gi1];
    }
    a0 = add_widen(a0, d.x);
    b0 = add_widen(b0, e.x);
    a1 = add_widen(a1, d.y);
    b1 = add_widen(b1, e.y);
    a2 = add_widen(a2, d.z);
    b2 = add_widen(b2, e.z);
    a3 = add_widen(a3, d.w);
    b3 = add_widen(b3, e.w);
  }
  r0 = make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2), __double2float_rn(a3));
  r1 = make_float4(__double2float_rn(b0), __double2float_rn(b1), __double2float_rn(b2), __double2float_rn(b3));
}

// A uint8 source's decoded values lo + q*step (q <= 255) are finite -- and so
// take the fast widening -- when its header is finite and |lo| + 256 step
// stays well inside the float range.
__device__ __forceinline__ bool fold_fast_ok(float lo, float step) {
  return finite_f(lo) && finite_f(step) && __fadd_rn(fabsf(lo), __fmul_rn(256.0f, step)) < 1.0e38f;
}

// Two groups per call: 8 independent fp64 chains in flight per thread, so the
// conversion/FP64 pipe always has ready work (the single-group fold is
// latency-bound on its 4 DADD chains with 16 consumer warps per SM).
template <int CODEC>
__device__ __forceinline__ void fold_group2(const uint8_t* st, int gi0, int gi1, int nsrc, int T,
                                            const float* lo, const float* step, float4& r0, float4& r1) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  for (int j = 0; j < nsrc; ++j) {
    float4 d, e;
    if (CODEC == kU8) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16);
      const uint32_t c0 = cs[gi0], c1 = cs[gi1];
      d = dequant4(c0, lo[j], step[j]);
      e = dequant4(c1, lo[j], step[j]);
    } else {
      const float4* fs = reinterpret_cast<const float4*>(st + size_t(j) * T * 64);
      d = fs[gi0];
      e = fs[gi1];
    }
    a0 = __dadd_rn(a0, double(d.x));
    b0 = __dadd_rn(b0, double(e.x));
    a1 = __dadd_rn(a1, double(d.y));
    b1 = __dadd_rn(b1, double(e.y));
    a2 = __dadd_rn(a2, double(d.z));
    b2 = __dadd_rn(b2, double(e.z));
    a3 = __dadd_rn(a3, double(d.w));
    b3 = __dadd_rn(b3, double(e.w));
  }
  r0 = make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2), __double2float_rn(a3));
  r1 = make_float4(__double2float_rn(b0), __double2float_rn(b1), __double2float_rn(b2), __double2float_rn(b3));
}

// Table form: D_j(q) pre-widened to fp64 once per source (256 entries), so
// the per-element F2F disappears; costs one LDS.64 with data-dependent banks.
__device__ __forceinline__ float4 fold_group_tab(const uint8_t* st, int gi, int nsrc, int T,
                                                 const double* tab /* [nsrc][256] */) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int j = 0; j < nsrc; ++j) {
    const uint32_t c = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16)[gi];
    const double* t = tab + j * 256;
    a0 = __dadd_rn(a0, t[c & 0xffu]);
    a1 = __dadd_rn(a1, t[(c >> 8) & 0xffu]);
    a2 = __dadd_rn(a2, t[(c >> 16) & 0xffu]);
    a3 = __dadd_rn(a3, t[c >> 24]);
  }
  return make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2), __double2float_rn(a3));
}

// Per-source decode constants for the owner / neighbour folds.
struct SrcDec {
  float lo, step, c23;
};

// The production fold: two groups (8 fp64 chains) per call, NSRC known at
// compile time (fully unrolled), FFMA dequant and XU-free widening.  Exact
// when every source's header allows the fast forms (fold_fast_ok +
// U8Params::fastdec); otherwise callers use fold_group2.
// inv != 1 scales the fp64 sums before the single rounding (D_*: average).
// Identity sources may hold non-finite values; `special` reports them so the
// caller can redo the group with the exact F2F fold.
// Two terms, no scaling: (float)((0.0 + (double)d0) + (double)d1) is the
// correctly rounded fp32 sum d0 + d1 -- binary64 has 53 >= 2*24 + 2 bits, so
// rounding the exact sum to binary64 and then to binary32 equals rounding it
// once (double rounding is innocuous at that precision) -- except that the
// fp64 fold starts from +0.0 and so turns (-0) + (-0) into +0: + 0.0f
// reproduces that.  Two FADDs per element instead of two widenings, two DFMAs
// and an F2F.  Holds for every input, non-finite included.
__device__ __forceinline__ float sum2_exact(float d0, float d1) { return __fadd_rn(__fadd_rn(d0, d1), 0.0f); }

template <int NSRC, int CODEC>
__device__ __forceinline__ void fold2_fast(const uint8_t* st, int gi0, int gi1, int T, const SrcDec* dec,
                                           double inv, float4& r0, float4& r1, bool& special) {
  if (NSRC == 2 && inv == 1.0) {
    float4 d[2], e[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (CODEC == kU8) {
        const uint32_t* cs = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16);
        const SrcDec q = dec[j];
        d[j] = dequant4_fast(cs[gi0], q.lo, q.step, q.c23);
        e[j] = dequant4_fast(cs[gi1], q.lo, q.step, q.c23);
      } else {
        const float4* fs = reinterpret_cast<const float4*>(st + size_t(j) * T * 64);
        d[j] = fs[gi0];
        e[j] = fs[gi1];
      }
    }
    r0 = make_float4(sum2_exact(d[0].x, d[1].x), sum2_exact(d[0].y, d[1].y), sum2_exact(d[0].z, d[1].z),
                     sum2_exact(d[0].w, d[1].w));
    r1 = make_float4(sum2_exact(e[0].x, e[1].x), sum2_exact(e[0].y, e[1].y), sum2_exact(e[0].z, e[1].z),
                     sum2_exact(e[0].w, e[1].w));
    special = false;
    return;
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
  bool sp = false;
#pragma unroll
  for (int j = 0; j < NSRC; ++j) {
    float4 d, e;
    if (CODEC == kU8) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16);
      const uint32_t c0 = cs[gi0], c1 = cs[gi1];
      const SrcDec q = dec[j];
      d = dequant4_fast(c0, q.lo, q.step, q.c23);
      e = dequant4_fast(c1, q.lo, q.step, q.c23);
    } else {
      const float4* fs = reinterpret_cast<const float4*>(st + size_t(j) * T * 64);
      d = fs[gi0];
      e = fs[gi1];
      sp |= !(fabsf(d.x) <= 3.4028235e38f) | !(fabsf(d.y) <= 3.4028235e38f) | !(fabsf(d.z) <= 3.4028235e38f) |
            !(fabsf(d.w) <= 3.4028235e38f) | !(fabsf(e.x) <= 3.4028235e38f) | !(fabsf(e.y) <= 3.4028235e38f) |
            !(fabsf(e.z) <= 3.4028235e38f) | !(fabsf(e.w) <= 3.4028235e38f);
    }
    a0 = add_widen(a0, d.x);
    b0 = add_widen(b0, e.x);
    a1 = add_widen(a1, d.y);
    b1 = add_widen(b1, e.y);
    a2 = add_widen(a2, d.z);
    b2 = add_widen(b2, e.z);
    a3 = add_widen(a3, d.w);
    b3 = add_widen(b3, e.w);
  }
  if (inv != 1.0) {
    a0 = __dmul_rn(a0, inv);
    a1 = __dmul_rn(a1, inv);
    a2 = __dmul_rn(a2, inv);
    a3 = __dmul_rn(a3, inv);
    b0 = __dmul_rn(b0, inv);
    b1 = __dmul_rn(b1, inv);
    b2 = __dmul_rn(b2, inv);
    b3 = __dmul_rn(b3, inv);
  }
  r0 = make_float4(__double2float_rn(a0), __double2float_rn(a1), __double2float_rn(a2), __double2float_rn(a3));
  r1 = make_float4(__double2float_rn(b0), __double2float_rn(b1), __double2float_rn(b2), __double2float_rn(b3));
  special = sp;
}

// Exact reference fold of one group with F2F widening (any data, any
// header): the fallback of fold2_fast.
template <int CODEC>
__device__ __forceinline__ float4 fold1_exact(const uint8_t* st, int gi, int nsrc, int T, const SrcDec* dec,
                                              double inv) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int j = 0; j < nsrc; ++j) {
    float4 d;
    if (CODEC == kU8)
      d = dequant4(reinterpret_cast<const uint32_t*>(st + size_t(j) * T * 16)[gi], dec[j].lo, dec[j].step);
    else
      d = reinterpret_cast<const float4*>(st + size_t(j) * T * 64)[gi];
    a0 = __dadd_rn(a0, double(d.x));
    a1 = __dadd_rn(a1, double(d.y));
    a2 = __dadd_rn(a2, double(d.z));
    a3 = __dadd_rn(a3, double(d.w));
  }
  return make_float4(__double2float_rn(__dmul_rn(a0, inv)), __double2float_rn(__dmul_rn(a1, inv)),
                     __double2float_rn(__dmul_rn(a2, inv)), __double2float_rn(__dmul_rn(a3, inv)));
}

// Runtime source count -> compile-time unrolled fold.
// `fast` (CTA-uniform) selects the fast forms; the exact fold is used when a
// header forbids them or an identity group holds non-finite values.
template <int CODEC>
__device__ __forceinline__ void fold2(int nsrc, bool fast, const uint8_t* st, int gi0, int gi1, int T,
                                      const SrcDec* dec, double inv, float4& r0, float4& r1) {
  bool special = !fast;
  if (fast) {
    switch (nsrc) {
      case 1: fold2_fast<1, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 2: fold2_fast<2, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 3: fold2_fast<3, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 4: fold2_fast<4, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 5: fold2_fast<5, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 6: fold2_fast<6, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      case 7: fold2_fast<7, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
      default: fold2_fast<8, CODEC>(st, gi0, gi1, T, dec, inv, r0, r1, special); break;
    }
  }
  if (special) {
    r0 = fold1_exact<CODEC>(st, gi0, nsrc, T, dec, inv);
    r1 = fold1_exact<CODEC>(st, gi1, nsrc, T, dec, inv);
  }
}

}  // namespace b2
