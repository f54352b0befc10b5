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
// (minmax then quantize) over the same range; 3: decode codes -> x write
template <int MODE>
__global__ void __launch_bounds__(kRingThreads, 1) ring_kernel(float* x, uint8_t* codes, size_t n, float2* out,
                                                               int* status) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float2 red[32];
  Ring r;
  r.init(smem, status, 1000000000ull);
  PassDesc p;
  p.s = 0;
  p.n = n;
  p.eb = MODE == 3 ? 1 : 4;
  p.nsrc = 1;
  p.base[0] = MODE == 3 ? codes : reinterpret_cast<const uint8_t*>(x);
  float lo = 1e30f, hi = -1e30f;
  const int ct = r.ct;
  if (MODE == 0 || MODE == 2) {
    r.run(p, [&](const uint8_t* st, size_t, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) {
        const float4 v = xs[gi];
        lo = fmin_nan(lo, fmin_nan(fmin_nan(v.x, v.y), fmin_nan(v.z, v.w)));
        hi = fmax_nan(hi, fmax_nan(fmax_nan(v.x, v.y), fmax_nan(v.z, v.w)));
      }
    });
  }
  if (MODE == 1 || MODE == 2) {
    r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(st);
      uint32_t* c32 = reinterpret_cast<uint32_t*>(codes + e0);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers) c32[gi] = quantize4(xs[gi], -1.0f, 127.5f);
    });
  }
  if (MODE == 3) {
    r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int) {
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(st);
      float4* x4 = reinterpret_cast<float4*>(x + e0);
      for (int gi = ct; gi < int(units * 4); gi += kConsumers)
        __stcs(x4 + gi, dequant4_fast(cs[gi], -1.0f, 0.0078431f, -65793.0f));
    });
  }
  if (!r.producer) {
    const float2 m = consumer_minmax(lo, hi, red);
    if (ct == 0) out[blockIdx.x] = m;
  }
}

template <int MODE>
float run(float* x, uint8_t* c, size_t n, float2* out, int* st, int nsm, int reps) {
  CK(cudaFuncSetAttribute(ring_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  ring_kernel<MODE><<<nsm, kRingThreads, kRingSmem>>>(x, c, n, out, st);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) ring_kernel<MODE><<<nsm, kRingThreads, kRingSmem>>>(x, c, n, out, st);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

template <int MODE>
float run_coop(float* x, uint8_t* c, size_t n, float2* out, int* st, int nsm, int reps) {
  CK(cudaFuncSetAttribute(ring_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  void* args[] = {&x, &c, &n, &out, &st};
  auto go = [&] {
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
  CK(cudaMalloc(&out, 8 * 1024));
  CK(cudaMalloc(&st, 4));
  CK(cudaMemset(x, 0, nmax * 4));
  for (size_t n : {size_t(1000), size_t(100000000)}) {
    printf("launch n=%zu: regular %.1f us, cooperative %.1f us\n", n, run<0>(x, c, n, out, st, nsm, 20) * 1e3,
           run_coop<0>(x, c, n, out, st, nsm, 20) * 1e3);
  }
  for (size_t n : {size_t(12500000), size_t(25000000), size_t(50000000), size_t(100000000)}) {
    const double mb = n * 4.0 / 1e6;
    float t0 = run<0>(x, c, n, out, st, nsm, 10);
    float t1 = run<1>(x, c, n, out, st, nsm, 10);
    float t2 = run<2>(x, c, n, out, st, nsm, 10);
    float t3 = run<3>(x, c, n, out, st, nsm, 10);
    printf("n=%zu (%.0f MB x): minmax %.1f us (%.0f GB/s) | quantize %.1f us (%.0f GB/s) | minmax+quantize %.1f us | "
           "decode %.1f us (%.0f GB/s)\n",
           n, mb, t0 * 1e3, mb / t0, t1 * 1e3, (n * 5.0 / 1e6) / t1, t2 * 1e3, t3 * 1e3, (n * 5.0 / 1e6) / t3);
  }
  return 0;
}
