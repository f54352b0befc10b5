// mc_probe.cu -- is NVSwitch multicast (NVLS) usable here, and how fast is an
// allgather that PUSHES each GPU's slice once through a multicast mapping
// (multimem.st) compared with every GPU PULLING the other slices from its
// peers (ld.global over NVLink)?  One process, one host thread per GPU.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mc_probe mc_probe.cu -lcuda -lpthread
//   ./mc_probe [MB per GPU slice, default 25]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e_ = (x);                                                  \
    if (e_ != cudaSuccess) {                                               \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);         \
      exit(1);                                                             \
    }                                                                      \
  } while (0)
#define CU(x)                                                              \
  do {                                                                     \
    CUresult r_ = (x);                                                     \
    if (r_ != CUDA_SUCCESS) {                                              \
      const char* s_ = nullptr;                                            \
      cuGetErrorString(r_, &s_);                                           \
      printf("CU %s (%d) at %d\n", s_ ? s_ : "?", int(r_), __LINE__);      \
      exit(2);                                                             \
    }                                                                      \
  } while (0)

// GPU r writes slice r of the multicast buffer: every GPU's copy receives it
__global__ void mc_push(float4* mc, size_t slice_v4, int r) {
  float4* p = mc + size_t(r) * slice_v4;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < slice_v4; i += size_t(gridDim.x) * blockDim.x) {
    const float4 v = make_float4(float(r), float(i & 1023), 1.f, 2.f);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
  }
}
// GPU r pulls every other slice from the owner's unicast buffer into its own copy
struct Peers {
  const float4* src[8];
};
__global__ void pull(Peers ps, float4* mine, size_t slice_v4, int g, int r) {
  for (int s = 1; s < g; ++s) {
    const int k = (r + s) % g;
    const float4* q = ps.src[k] + size_t(k) * slice_v4;
    float4* d = mine + size_t(k) * slice_v4;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < slice_v4; i += size_t(gridDim.x) * blockDim.x)
      d[i] = __ldcg(q + i);
  }
}

int main(int argc, char** argv) {
  const size_t slice = size_t(argc > 1 ? atoi(argv[1]) : 25) << 20;
  CU(cuInit(0));
  int g = 0;
  CK(cudaGetDeviceCount(&g));
  if (g < 2) {
    printf("{\"error\": \"needs >= 2 GPUs\"}\n");
    return 0;
  }
  int mc_ok = 0;
  CUdevice dev0;
  CU(cuDeviceGet(&dev0, 0));
  cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev0);
  printf("multicast supported attribute: %d, gpus %d\n", mc_ok, g);
  if (!mc_ok) return 0;
  const size_t want = slice * size_t(g);
  CUmulticastObjectProp mp{};
  mp.numDevices = unsigned(g);
  mp.size = want;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (want + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < g; ++d) {
    CUdevice dv;
    CU(cuDeviceGet(&dv, d));
    CU(cuMulticastAddDevice(mc, dv));
  }
  std::vector<float4*> uc(g), mcp(g);
  for (int d = 0; d < g; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFree(0));
    for (int e = 0; e < g; ++e)
      if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaGetLastError();
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ugran = 0;
    CU(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle mh;
    CU(cuMemCreate(&mh, size, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mh, 0, size, 0));
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr up, mptr;
    CU(cuMemAddressReserve(&up, size, ugran, 0, 0));
    CU(cuMemMap(up, size, 0, mh, 0));
    CU(cuMemSetAccess(up, size, &ad, 1));
    CU(cuMemAddressReserve(&mptr, size, gran, 0, 0));
    CU(cuMemMap(mptr, size, 0, mc, 0));
    CU(cuMemSetAccess(mptr, size, &ad, 1));
    uc[d] = reinterpret_cast<float4*>(up);
    mcp[d] = reinterpret_cast<float4*>(mptr);
  }
  // peers read each other's unicast buffers (pull comparison)
  for (int d = 0; d < g; ++d) {
    CK(cudaSetDevice(d));
    std::vector<CUmemAccessDesc> ads;
    for (int e = 0; e < g; ++e) {
      CUmemAccessDesc ad{};
      ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ad.location.id = e;
      ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      ads.push_back(ad);
    }
    CU(cuMemSetAccess(reinterpret_cast<CUdeviceptr>(uc[d]), size, ads.data(), ads.size()));
  }
  const size_t slice_v4 = slice / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int mode = 0; mode < 2; ++mode) {
    for (int grid_mult : {1, 2, 4}) {
      std::vector<float> ms(g);
      std::vector<std::thread> th;
      for (int d = 0; d < g; ++d)
        th.emplace_back([&, d] {
          CK(cudaSetDevice(d));
          cudaStream_t s;
          CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
          cudaEvent_t a, b;
          CK(cudaEventCreate(&a));
          CK(cudaEventCreate(&b));
          Peers ps{};
          for (int e = 0; e < g; ++e) ps.src[e] = uc[e];
          for (int it = 0; it < 6; ++it) {
            if (it == 3) CK(cudaEventRecord(a, s));
            if (mode == 0)
              mc_push<<<sms * grid_mult, 512, 0, s>>>(mcp[d], slice_v4, d);
            else
              pull<<<sms * grid_mult, 512, 0, s>>>(ps, uc[d], slice_v4, g, d);
          }
          CK(cudaEventRecord(b, s));
          CK(cudaEventSynchronize(b));
          float t = 0;
          CK(cudaEventElapsedTime(&t, a, b));
          ms[d] = t / 3;
        });
      for (auto& t : th) t.join();
      float mx = 0;
      for (float v : ms) mx = v > mx ? v : mx;
      const double ingress = double(slice) * (g - 1);
      printf("{\"mode\": \"%s\", \"g\": %d, \"grid\": %d, \"slice_MB\": %.1f, \"us\": %.1f, \"ingress_GBps\": %.1f}\n",
             mode == 0 ? "multicast_push" : "pull_ldg", g, sms * grid_mult, slice / 1048576.0, mx * 1e3,
             ingress / (mx * 1e-3) / 1e9);
    }
  }
  // check: after the multicast pushes every copy holds every slice
  CK(cudaSetDevice(0));
  for (int d = 0; d < g; ++d) {
    CK(cudaSetDevice(d));
    mc_push<<<sms, 512>>>(mcp[d], slice_v4, d);
    CK(cudaDeviceSynchronize());
  }
  int bad = 0;
  for (int d = 0; d < g; ++d) {
    std::vector<float4> h(slice_v4 * g);
    CK(cudaSetDevice(d));
    CK(cudaMemcpy(h.data(), uc[d], slice * g, cudaMemcpyDeviceToHost));
    for (int k = 0; k < g; ++k)
      for (size_t i = 0; i < slice_v4; i += 997)
        if (h[k * slice_v4 + i].x != float(k) || h[k * slice_v4 + i].y != float(i & 1023)) ++bad;
  }
  printf("{\"check\": \"%s\", \"bad\": %d}\n", bad ? "FAIL" : "ok", bad);
  return 0;
}
