// fold_bench.cu -- single-GPU microbenchmark of the phase-2 owner fold
// (g uint8 contributions -> fp64 ascending fold -> fp32), streamed through
// the same TMA ring as the product kernel, to choose the fold variant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I../../include \
//        -I../../paper_2107_01499_b200/csrc -o fold_bench fold_bench.cu
//   ./fold_bench <g> <variant 0=group,1=group2,2=table> [elements]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fold.cuh"
#include "ring.cuh"

using namespace b2;

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);                              \
      exit(1);                                                                                  \
    }                                                                                           \
  } while (0)

template <int VAR>
__global__ void __launch_bounds__(kRingThreads, 1) fold_kernel(const uint8_t* codes, size_t slot, int g, size_t n,
                                                                float* out, int* status) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float s_lo[kMaxRanks], s_step[kMaxRanks];
  __shared__ double s_tab[kMaxRanks * 256];
  __shared__ SrcDec s_dec[kMaxRanks];
  Ring r;
  r.init(smem, status, 1000000000ull);
  if (threadIdx.x < kMaxRanks) {
    s_lo[threadIdx.x] = -1.0f + 0.01f * threadIdx.x;
    s_step[threadIdx.x] = __fdiv_rn(__fsub_rn(1.0f, s_lo[threadIdx.x]), 255.0f);
    const U8Params q = u8_params(s_lo[threadIdx.x], 1.0f);
    s_dec[threadIdx.x] = SrcDec{q.lo, q.step, q.c23};
  }
  __syncthreads();
  for (int i = threadIdx.x; i < g * 256; i += blockDim.x)
    s_tab[i] = double(dequant1(uint8_t(i & 255), s_lo[i >> 8], s_step[i >> 8]));
  __syncthreads();
  PassDesc p = PassDesc::make();
  p.s = 0;
  p.n = n;
  p.eb = 1;
  p.nsrc = g;
  for (int j = 0; j < g; ++j) p.base[j] = codes + j * slot;
  const int ct = r.ct;
  float4* x4 = reinterpret_cast<float4*>(out);
  r.run(p, [&](const uint8_t* st, size_t e0, size_t units, int T) {
    const int ng = int(units * 4);
    if (VAR == 1 || VAR == 3) {
      for (int gi = ct; gi < ng; gi += 2 * kConsumers) {
        const int g1 = gi + kConsumers < ng ? gi + kConsumers : gi;
        float4 a, b;
        if (VAR == 1)
          fold_group2<kU8>(st, gi, g1, g, T, s_lo, s_step, a, b);
        else
          fold2<kU8>(g, true, st, gi, g1, T, s_dec, 1.0, a, b);
        __stcs(x4 + (e0 >> 2) + gi, a);
        if (g1 != gi) __stcs(x4 + (e0 >> 2) + g1, b);
      }
    } else {
      for (int gi = ct; gi < ng; gi += kConsumers) {
        const float4 y = VAR == 2 ? fold_group_tab(st, gi, g, T, s_tab) : fold_group<kU8>(st, gi, g, T, s_lo, s_step);
        __stcs(x4 + (e0 >> 2) + gi, y);
      }
    }
  });
}

int main(int argc, char** argv) {
  const int g = argc > 1 ? atoi(argv[1]) : 2;
  const int var = argc > 2 ? atoi(argv[2]) : 0;
  const size_t n = argc > 3 ? strtoull(argv[3], 0, 10) : 100000000ull / g;
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t slot = (n + 255) / 256 * 256;
  uint8_t* codes;
  float* out;
  int* status;
  CK(cudaMalloc(&codes, slot * g));
  CK(cudaMalloc(&out, n * 4));
  CK(cudaMalloc(&status, 4));
  std::vector<uint8_t> h(slot * g);
  for (size_t i = 0; i < h.size(); ++i) h[i] = uint8_t((i * 2654435761u) >> 13);
  CK(cudaMemcpy(codes, h.data(), h.size(), cudaMemcpyHostToDevice));
  auto launch = [&] {
    if (var == 0) fold_kernel<0><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, out, status);
    if (var == 1) fold_kernel<1><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, out, status);
    if (var == 2) fold_kernel<2><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, out, status);
    if (var == 3) fold_kernel<3><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, out, status);
  };
  CK(cudaFuncSetAttribute(fold_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  CK(cudaFuncSetAttribute(fold_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  CK(cudaFuncSetAttribute(fold_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  CK(cudaFuncSetAttribute(fold_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
  if (var == 9) {  // exactness check of the fast fold vs the F2F fold on the same data
    float *o1, *o2;
    CK(cudaMalloc(&o1, n * 4));
    CK(cudaMalloc(&o2, n * 4));
    fold_kernel<0><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, o1, status);
    fold_kernel<3><<<nsm, kRingThreads, kRingSmem>>>(codes, slot, g, n, o2, status);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned> h1(n), h2(n);
    CK(cudaMemcpy(h1.data(), o1, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), o2, n * 4, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < n; ++i) bad += h1[i] != h2[i];
    printf("fold g=%d exactness fast vs f2f: %zu mismatches of %zu\n", g, bad, n);
    return bad != 0;
  }
  launch();
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  for (int i = 0; i < 5; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  ms /= 5;
  const double bytes = double(n) * g + 4.0 * n;
  printf("fold g=%d var=%d n=%zu: %.1f us, %.2f Gelem-src/s (%.2f per clk per SM @1.9GHz), %.0f GB/s\n", g, var, n,
         ms * 1e3, double(n) * g / ms / 1e6, double(n) * g / (ms * 1e-3) / nsm / 1.9e9, bytes / ms / 1e6);
  return 0;
}
