// probe.cu -- hardware probes that informed the kernel design.
//
//   probe cvt            : F2F.F64.F32 + DADD vs integer-path conversion throughput
//   probe hbm            : streaming read bandwidth, LDG.128 vs cp.async.bulk ring
//   probe peer           : (needs 2 GPUs, one process) peer LDG.128 / STG.128 /
//                          cp.async.bulk from peer memory, bandwidth + correctness
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__global__ void cvt_f2f(const float* x, double* out, int iters) {
  float v = x[threadIdx.x & 31] + threadIdx.x;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < iters; ++i) {
    a0 = __dadd_rn(a0, double(v));
    a1 = __dadd_rn(a1, double(__fadd_rn(v, 1.0f)));
    a2 = __dadd_rn(a2, double(__fadd_rn(v, 2.0f)));
    a3 = __dadd_rn(a3, double(__fadd_rn(v, 3.0f)));
    v = __fadd_rn(v, 0.5f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

__device__ __forceinline__ double f2d_int(float f) {
  const unsigned b = __float_as_uint(f);
  const unsigned e = (b >> 23) & 0xff;
  unsigned hi = ((b >> 3) & 0x0fffffffu) + 0x38000000u;
  hi |= (b & 0x80000000u);
  hi = e ? hi : (b & 0x80000000u);
  const unsigned lo = e ? (b << 29) : 0u;
  return __hiloint2double(hi, lo);
}

__global__ void cvt_int(const float* x, double* out, int iters) {
  float v = x[threadIdx.x & 31] + threadIdx.x;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int i = 0; i < iters; ++i) {
    a0 = __dadd_rn(a0, f2d_int(v));
    a1 = __dadd_rn(a1, f2d_int(__fadd_rn(v, 1.0f)));
    a2 = __dadd_rn(a2, f2d_int(__fadd_rn(v, 2.0f)));
    a3 = __dadd_rn(a3, f2d_int(__fadd_rn(v, 3.0f)));
    v = __fadd_rn(v, 0.5f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

__global__ void ldg_read(const float4* x, size_t n4, float* out) {
  float acc = 0;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += stride * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i + u * stride < n4 ? __ldcs(x + i + u * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void stg_write(float4* y, size_t n4) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4; i += stride)
    y[i] = make_float4(1, 2, 3, float(i & 7));
}

// ---------------------------------------------------- cp.async.bulk ring read
constexpr int STAGES = 6, STAGE = 32768;
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(544) ring_read(const char* x, size_t bytes, float* out, float* copy_out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + STAGES;
  unsigned char* buf = sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NC = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t ntiles = bytes / STAGE;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      unsigned ph = 0;
      for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(empty + s, ph ^ 1);
        mbar_expect(full + s, STAGE);
        bulk_g2s(buf + size_t(s) * STAGE, x + t * STAGE, STAGE, full + s);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  float acc = 0;
  int s = 0;
  unsigned ph = 0;
  const int ct = threadIdx.x - 32;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(full + s, ph);
    const float4* b4 = reinterpret_cast<const float4*>(buf + size_t(s) * STAGE);
    for (int i = ct; i < STAGE / 16; i += NC * 32) {
      float4 v = b4[i];
      acc += v.x + v.y + v.z + v.w;
      if (copy_out) reinterpret_cast<float4*>(copy_out)[t * (STAGE / 16) + i] = v;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);
    if (++s == STAGES) { s = 0; ph ^= 1; }
  }
  if (acc == 12345.f) out[0] = acc;
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / reps;
}

int main(int argc, char** argv) {
  const char* mode = argc > 1 ? argv[1] : "cvt";
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int ring_smem = 128 + STAGES * STAGE;
  CK(cudaFuncSetAttribute(ring_read, cudaFuncAttributeMaxDynamicSharedMemorySize, ring_smem));
  if (!strcmp(mode, "cvt")) {
    float* x;
    double* out;
    CK(cudaMalloc(&x, 128));
    CK(cudaMemset(x, 0, 128));
    CK(cudaMalloc(&out, sizeof(double) * nsm * 4 * 512));
    const int iters = 4096;
    const double ops = double(nsm) * 4 * 512 * iters * 4;
    float t1 = time_ms([&] { cvt_f2f<<<nsm * 4, 512>>>(x, out, iters); });
    float t2 = time_ms([&] { cvt_int<<<nsm * 4, 512>>>(x, out, iters); });
    printf("cvt: F2F+DADD %.3f ms -> %.1f Gcvt/s (%.2f per clk per SM @1.9GHz); INT+DADD %.3f ms -> %.1f G/s\n", t1,
           ops / t1 / 1e6, ops / t1 / 1e6 / nsm / 1.9, t2, ops / t2 / 1e6);
  } else if (!strcmp(mode, "hbm")) {
    const size_t bytes = size_t(1) << 31;  // 2 GiB
    char* x;
    float* out;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMemset(x, 1, bytes));
    CK(cudaMalloc(&out, 64));
    for (int bpsm : {1, 2, 4}) {
      float t = time_ms([&] { ldg_read<<<nsm * bpsm, 512>>>((const float4*)x, bytes / 16, out); });
      printf("hbm: LDG.128 read grid=%dx512: %.1f GB/s\n", nsm * bpsm, bytes / t / 1e6);
    }
    float t = time_ms([&] { ring_read<<<nsm, 544, ring_smem>>>(x, bytes, out, nullptr); });
    printf("hbm: cp.async.bulk ring read (6x32KB, 1 CTA/SM): %.1f GB/s\n", bytes / t / 1e6);
    t = time_ms([&] { stg_write<<<nsm * 4, 512>>>((float4*)x, bytes / 16); });
    printf("hbm: STG.128 write: %.1f GB/s\n", bytes / t / 1e6);
  } else if (!strcmp(mode, "peer")) {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
      printf("peer: needs 2 GPUs\n");
      return 0;
    }
    const size_t bytes = size_t(1) << 30;
    char *x0, *x1, *y0;
    float* out;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&x1, bytes));
    CK(cudaMemset(x1, 0, bytes));
    {
      std::vector<float> h(1 << 20);
      for (size_t i = 0; i < h.size(); ++i) h[i] = float(i % 1000);
      CK(cudaMemcpy(x1, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    }
    CK(cudaSetDevice(0));
    CK(cudaMalloc(&x0, bytes));
    CK(cudaMalloc(&y0, bytes));
    CK(cudaMalloc(&out, 64));
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, 0, 1));
    printf("peer: can access %d\n", can);
    CK(cudaDeviceEnablePeerAccess(1, 0));
    float t = time_ms([&] { ldg_read<<<nsm * 4, 512>>>((const float4*)x1, bytes / 16, out); });
    printf("peer: LDG.128 read from GPU1: %.1f GB/s\n", bytes / t / 1e6);
    t = time_ms([&] { stg_write<<<nsm * 4, 512>>>((float4*)x1, bytes / 16); });
    printf("peer: STG.128 write to GPU1: %.1f GB/s\n", bytes / t / 1e6);
    // restore pattern, then TMA read from peer and verify the first MiB
    CK(cudaSetDevice(1));
    {
      std::vector<float> h(1 << 20);
      for (size_t i = 0; i < h.size(); ++i) h[i] = float(i % 1000);
      CK(cudaMemcpy(x1, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
      CK(cudaDeviceSynchronize());
    }
    CK(cudaSetDevice(0));
    ring_read<<<nsm, 544, ring_smem>>>(x1, size_t(1) << 22, out, (float*)y0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> h(1 << 20);
    CK(cudaMemcpy(h.data(), y0, h.size() * 4, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (size_t i = 0; i < h.size(); ++i) bad += h[i] != float(i % 1000);
    printf("peer: cp.async.bulk from peer memory: %s (%zu mismatches)\n", bad ? "WRONG" : "correct", bad);
    t = time_ms([&] { ring_read<<<nsm, 544, ring_smem>>>(x1, bytes, out, nullptr); });
    printf("peer: cp.async.bulk ring read from GPU1: %.1f GB/s\n", bytes / t / 1e6);
    t = time_ms([&] { CK(cudaMemcpyPeerAsync(x0, 0, x1, 1, bytes)); });
    printf("peer: cudaMemcpyPeer GPU1->GPU0: %.1f GB/s\n", bytes / t / 1e6);
  }
  return 0;
}
