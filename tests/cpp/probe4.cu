// probe4.cu -- NVSwitch ceilings with every GPU active at once (one process,
// one host thread per GPU, peer access enabled):
//   push  : GPU r stores into GPU (r+s)%G for shift s (STG.128 / STG.32)
//   pull  : GPU r TMA-reads from GPU (r+s)%G
//   a2a   : GPU r stores 1/(G-1) of the bytes to every peer at once
// Prints aggregate per-GPU GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2107_01499_b200/csrc -o probe4 probe4.cu -lpthread
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

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

template <int W>  // bytes per lane per store: 4 or 16
__global__ void push_kernel(uint8_t* const* dst, int ndst, size_t bytes_per_dst) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (int d = 0; d < ndst; ++d) {
    if (W == 16) {
      uint4* p = reinterpret_cast<uint4*>(dst[d]);
      for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < bytes_per_dst / 16; i += stride)
        p[i] = make_uint4(unsigned(i), 1, 2, 3);
    } else {
      uint32_t* p = reinterpret_cast<uint32_t*>(dst[d]);
      for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < bytes_per_dst / 4; i += stride)
        p[i] = unsigned(i);
    }
  }
}

// a2a push: interleave destinations at 32 KB granularity
__global__ void a2a_kernel(uint8_t* const* dst, int ndst, size_t bytes_per_dst) {
  const size_t chunk = 32768, nch = bytes_per_dst / chunk;
  for (size_t c = blockIdx.x; c < nch * ndst; c += gridDim.x) {
    uint4* p = reinterpret_cast<uint4*>(dst[c % ndst] + (c / ndst) * chunk);
    for (int i = threadIdx.x; i < int(chunk / 16); i += blockDim.x) p[i] = make_uint4(unsigned(i), 1, 2, 3);
  }
}

__global__ void __launch_bounds__(kRingThreads, 1) pull_kernel(const uint8_t* src, size_t bytes, float* out, int* st) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring r;
  r.init(smem, st, 1000000000ull);
  PassDesc p = PassDesc::make();
  p.s = 0;
  p.n = bytes;
  p.eb = 1;
  p.nsrc = 1;
  p.base[0] = src;
  float acc = 0.f;
  r.run(p, [&](const uint8_t* s, size_t, size_t units, int) {
    const uint32_t* c = reinterpret_cast<const uint32_t*>(s);
    for (int gi = r.ct; gi < int(units * 4); gi += kConsumers) acc += float(c[gi] & 1);
  });
  if (acc == 12345.f) out[0] = acc;
}

int main(int argc, char** argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G < 2) {
    printf("needs >= 2 GPUs\n");
    return 0;
  }
  const size_t bytes = size_t(256) << 20;  // per transfer
  std::vector<uint8_t*> buf(G);
  std::vector<float*> outs(G);
  std::vector<int*> sts(G);
  int nsm = 0;
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d));
    CK(cudaMalloc(&buf[d], bytes));
    CK(cudaMemset(buf[d], 1, bytes));
    CK(cudaMalloc(&outs[d], 64));
    CK(cudaMalloc(&sts[d], 64));
    CK(cudaFuncSetAttribute(pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
    for (int e = 0; e < G; ++e)
      if (e != d) CK(cudaDeviceEnablePeerAccess(e, 0));
  }
  auto timed = [&](auto launch) {  // all GPUs concurrently, max time
    std::vector<float> ms(G);
    std::vector<std::thread> th;
    for (int d = 0; d < G; ++d)
      th.emplace_back([&, d] {
        CK(cudaSetDevice(d));
        launch(d);
        CK(cudaDeviceSynchronize());
      });
    for (auto& t : th) t.join();
    th.clear();
    for (int d = 0; d < G; ++d)
      th.emplace_back([&, d] {
        CK(cudaSetDevice(d));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a));
        for (int i = 0; i < 3; ++i) launch(d);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms[d], a, b));
        ms[d] /= 3;
      });
    for (auto& t : th) t.join();
    float mx = 0;
    for (float v : ms) mx = v > mx ? v : mx;
    return mx;
  };
  std::vector<uint8_t**> dsts(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&dsts[d], sizeof(uint8_t*) * 8));
  }
  for (int s = 1; s < G; ++s) {
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      uint8_t* p = buf[(d + s) % G];
      CK(cudaMemcpy(dsts[d], &p, sizeof(p), cudaMemcpyHostToDevice));
    }
    float t16 = timed([&](int d) { push_kernel<16><<<nsm * 4, 512>>>(dsts[d], 1, bytes); });
    float t4 = timed([&](int d) { push_kernel<4><<<nsm * 4, 512>>>(dsts[d], 1, bytes); });
    float tp = timed([&](int d) {
      pull_kernel<<<nsm, kRingThreads, kRingSmem>>>(buf[(d + s) % G], bytes, outs[d], sts[d]);
    });
    printf("G=%d shift %d: push STG.128 %.0f GB/s, push STG.32 %.0f GB/s, TMA pull %.0f GB/s (per GPU)\n", G, s,
           bytes / t16 / 1e6, bytes / t4 / 1e6, bytes / tp / 1e6);
  }
  if (G > 2) {
    const size_t per = bytes / (G - 1) / 32768 * 32768;
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      std::vector<uint8_t*> v;
      for (int s = 1; s < G; ++s) v.push_back(buf[(d + s) % G]);
      CK(cudaMemcpy(dsts[d], v.data(), sizeof(uint8_t*) * v.size(), cudaMemcpyHostToDevice));
    }
    float ta = timed([&](int d) { a2a_kernel<<<nsm * 4, 512>>>(dsts[d], G - 1, per); });
    printf("G=%d all-to-all push (32 KB interleave): %.0f GB/s egress per GPU\n", G, per * (G - 1) / ta / 1e6);
  }
  return 0;
}
