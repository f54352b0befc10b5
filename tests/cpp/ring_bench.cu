// ring_bench.cu -- the product's Ring/PassDesc streaming machinery in
// isolation: read-only (min/max) and read+write (quantize -> codes) passes over
// x at several sizes, to find where the collective's x passes lose bandwidth.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I../../include \
//        -I../../paper_2107_01499_b200/csrc -o ring_bench ring_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ring.cuh"

using namespace b2;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);             \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// MODE 0: minmax only; 1: quantize -> codes (1 B/elem write); 2: two passes
// (minmax then quantize, reversed) over the same range; 3: decode codes -> x
// write.  sched != null: dynamic tile scheduling (the collectives' default).
template <int MODE>
__global__ void __launch_bounds__(kRingThreads, 1) ring_kernel(float* x, uint8_t* codes, size_t n, float2* out,
                                                               int* status, unsigned long long* sched) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red[32];
  __shared__ PassDesc s_p[2];
  __shared__ PassDesc s_q[4];  // MODE 7: four quarter passes
  Ring r;
  r.init(smem, status, 1000000000ull, sched);
  if (threadIdx.x == 0) {
    PassDesc p = PassDesc::make();
    p.n = n;
    p.eb = MODE == 3 ? 1 : 4;
    p.base[0] = MODE == 3 ? codes : reinterpret_cast<const uint8_t*>(x);
    s_p[0] = p;
    p.reverse = true;
    s_p[1] = p;
    for (int i = 0; i < 4; ++i) {
      s_q[i] = s_p[0];
      s_q[i].s = n / 4 * i;
      s_q[i].n = n / 4;
    }
  }
  __syncthreads();
  float lo = 1e30f, hi = -1e30f;
  const int ct = r.ct;
  if (MODE == 0 || MODE == 2) {
    r.run(s_p[0], [&](const uint8_t* st, size_t, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        const float4 v = xs[gi];
        lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
        hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
      }
    });
  }
  if (MODE == 1 || MODE == 2) {
    r.run(s_p[MODE == 2 ? 1 : 0], [&](const uint8_t* st, size_t e0, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      uint32_t* c32 = reinterpret_cast<uint32_t*>(codes + e0);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) c32[gi] = quantize4(xs[gi], -1.0f, 127.5f);
    });
  }
  if (MODE == 7) {  // the C_LP_S phase-1A shape: four chunk passes interleaved
    r.run_multi(s_q, 4, [&](int, const uint8_t* st, size_t, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        const float4 v = xs[gi];
        lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
        hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
      }
    });
  }
  if (MODE == 5 || MODE == 6) {  // split mode: pipe A quantizes (10 warps, 3 stages), pipe B idle
    r.split_begin();
    const int gct = r.gct, gn = r.gn;
    r.stream_split(
        s_p, 1,
        [&](int, const uint8_t* st, size_t e0, size_t units, int) {
          const float4* xs = reinterpret_cast<const float4*>(st);
          uint32_t* c32 = reinterpret_cast<uint32_t*>(codes + e0);
          if (MODE == 6) r.slot_acquire();
          for (int gi = gct; gi < int(units * 4); gi += gn) c32[gi] = quantize4(xs[gi], -1.0f, 127.5f);
          if (MODE == 6) r.slot_commit(nullptr, 0u);
        },
        [](int) {}, s_p, 0, [&](int, const uint8_t*, size_t, size_t, int) {}, [](int) {});
    if (MODE == 6 && r.group_a()) {
      r.slot_acquire();
      r.slot_commit(nullptr, 0u, true);
    }
    if (MODE == 6 && r.storer && (threadIdx.x & 31) == 0) r.signal_loop();
    r.split_end();
  }
  if (MODE == 3) {
    r.run(s_p[0], [&](const uint8_t* st, size_t e0, size_t units, int) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
      float4* x4 = reinterpret_cast<float4*>(x + e0);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers)
        __stcs(x4 + gi, dequant4_fast(cs[gi], -1.0f, 0.0078431f, -65793.0f));
    });
  }
  if (ct >= 0) {
    const float2 m = consumer_minmax(lo, hi, red);
    if (ct == 0) out[blockIdx.x] = m;
  }
  r.finish(reinterpret_cast<unsigned*>(sched + 64));
}

// plain LDG baseline: grid-stride float4 loads, 8 in flight per thread
__global__ void __launch_bounds__(512) ldg_minmax(const float4* x, size_t n4, float2* out) {
  float lo = 1e30f, hi = -1e30f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      lo = fmin_nan(lo, fmin_nan(fmin_nan(v[u].x, v[u].y), fmin_nan(v[u].z, v[u].w)));
      hi = fmax_nan(hi, fmax_nan(fmax_nan(v[u].x, v[u].y), fmax_nan(v[u].z, v[u].w)));
    }
  }
  for (; i < n4; i += stride) {
    const float4 v = x[i];
    lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
    hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
  }
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + threadIdx.x / 32] = make_float2(lo, hi);
}

float run_ldg(const float* x, size_t n, float2* out, int nsm, int per_sm, int reps) {
  auto go = [&] { ldg_minmax<<<nsm * per_sm, 512>>>(reinterpret_cast<const float4*>(x), n / 4, out); };
  go();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) go();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

float* g_cold[4] = {};  // when set: launches rotate over 4 inputs (> L2 each), so every read is cold

template <int MODE>
float run(float* x, uint8_t* c, size_t n, float2* out, int* st, int nsm, int reps, unsigned long long* sched) {
  CK(cudaFuncSetAttribute(ring_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  unsigned long long* sc = sched;
  void* args[] = {&x, &c, &n, &out, &st, &sc};
  int launch = 0;
  auto go = [&] {
    if (g_cold[0]) x = g_cold[launch++ % 4];
    CK(cudaLaunchCooperativeKernel((const void*)ring_kernel<MODE>, dim3(nsm), dim3(kRingThreads), args, kRingSmem, 0));
  };
  go();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) go();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t nmax = 100000000;
  float* x;
  uint8_t* c;
  float2* out;
  int* st;
  CK(cudaMalloc(&x, nmax * 4));
  CK(cudaMalloc(&c, nmax));
  CK(cudaMalloc(&out, 8 * 1024 * 64));
  CK(cudaMalloc(&st, 4));
  CK(cudaMemset(x, 0, nmax * 4));
  printf("ring: %d stages x %d B\n", kStages, kStageBytes);
  for (int per_sm : {2, 4}) {
    const size_t n = 100000000;
    const float t = run_ldg(x, n, out, nsm, per_sm, 10);
    printf("LDG minmax n=%zu, %d CTAs/SM: %.1f us (%.0f GB/s)\n", n, per_sm, t * 1e3, n * 4.0 / 1e6 / t);
  }
  unsigned long long* sched;
  CK(cudaMalloc(&sched, 65 * 8));
  CK(cudaMemset(sched, 0, 65 * 8));
  unsigned long long* endc = sched;  // static runs still need a valid end counter
  for (int k = 0; k < 4; ++k) {
    CK(cudaMalloc(&g_cold[k], nmax * 4));
    CK(cudaMemset(g_cold[k], 0, nmax * 4));
  }
  {
    const size_t n = nmax;
    const double mb = n * 4.0 / 1e6;
    float t0 = run<0>(x, c, n, out, st, nsm, 12, sched);
    float t7 = run<7>(x, c, n, out, st, nsm, 12, sched);
    float t1 = run<1>(x, c, n, out, st, nsm, 12, sched);
    printf("COLD (4 rotating 400 MB inputs, dynamic): minmax %.1f us (%.0f GB/s) | 4 chunk passes %.1f us | quantize "
           "%.1f us\n", t0 * 1e3, mb / t0, t7 * 1e3, t1 * 1e3);
    g_cold[0] = nullptr;
  }
  for (int dyn = 0; dyn < 2; ++dyn) {
    unsigned long long* sc = dyn ? sched : nullptr;
    (void)endc;
    printf("launch n=1000 (%s): %.1f us\n", dyn ? "dynamic" : "static", run<0>(x, c, 1000, out, st, nsm, 20, sc) * 1e3);
    for (size_t n : {size_t(25000000), size_t(100000000)}) {
      const double mb = n * 4.0 / 1e6;
      float t0 = run<0>(x, c, n, out, st, nsm, 10, sc);
      float t1 = run<1>(x, c, n, out, st, nsm, 10, sc);
      float t2 = run<2>(x, c, n, out, st, nsm, 10, sc);
      float t3 = run<3>(x, c, n, out, st, nsm, 10, sc);
      float t5 = run<5>(x, c, n, out, st, nsm, 10, sc);
      float t7 = run<7>(x, c, n, out, st, nsm, 10, sc);
      printf("  minmax as 4 interleaved chunk passes: %.1f us\n", t7 * 1e3);
      float t6 = run<6>(x, c, n, out, st, nsm, 10, sc);
      printf("  split pipe A quantize (10 warps, 3 stages): %.1f us; + credits/signaller: %.1f us\n", t5 * 1e3,
             t6 * 1e3);
      printf("%s n=%zu (%.0f MB x): minmax %.1f us (%.0f GB/s) | quantize %.1f us (%.0f GB/s) | minmax+quantize(rev) "
             "%.1f us | decode %.1f us (%.0f GB/s)\n",
             dyn ? "dynamic" : "static ", n, mb, t0 * 1e3, mb / t0, t1 * 1e3, (n * 5.0 / 1e6) / t1, t2 * 1e3,
             t3 * 1e3, (n * 5.0 / 1e6) / t3);
    }
  }
  return 0;
}
