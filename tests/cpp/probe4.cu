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

struct PullArgs {
  const uint8_t* src[8];
  int nsrc;
  float4* out;  // non-null: decode-like expansion, 4 fp32 per code byte written here (like phase 3)
};
// pull `bytes` in total: nsrc sources of bytes/nsrc each, one tile = nsrc
// bulk copies of 32 KB / nsrc (the fold's tile shape)
__global__ void __launch_bounds__(kRingThreads, 1) pull_kernel(PullArgs pa, size_t bytes, float* out, int* st) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ PassDesc sp;
  Ring r;
  r.init(smem, st, 1000000000ull);
  if (threadIdx.x == 0) {
    sp = PassDesc::make();
    sp.n = bytes / pa.nsrc;
    sp.eb = 1;
    sp.nsrc = pa.nsrc;
    for (int j = 0; j < pa.nsrc; ++j) sp.base[j] = pa.src[j];
  }
  __syncthreads();
  const PassDesc& p = sp;
  float acc = 0.f;
  r.run(p, [&](const uint8_t* s, size_t e0, size_t units, int T) {
    const uint32_t* c = reinterpret_cast<const uint32_t*>(s);
    if (pa.out) {  // every source's codes -> fp32 at (source slice, e0)
      for (int j = 0; j < pa.nsrc; ++j)
        for (int gi = r.ct; gi < int(units * 4); gi += kConsumers) {
          const uint32_t q = c[j * T * 4 + gi];
          __stcs(pa.out + (size_t(j) * (bytes / pa.nsrc) / 4 + e0 / 4 + gi),
                 make_float4(float(q & 255), float((q >> 8) & 255), float((q >> 16) & 255), float(q >> 24)));
        }
    } else {
      for (int gi = r.ct; gi < int(units * 4); gi += kConsumers) acc += float(c[gi] & 1);
    }
  });
  if (acc == 12345.f) out[0] = acc;
}

// 1B-like traffic: stream x (G chunks interleaved, reversed) and push the
// quantized codes of chunk i to GPU (d+1+i)%G with STG (MODE 0); MODE 1 =
// the x stream only; MODE 2 = the pushes only (codes from registers).
struct MixArgs {
  const float* x;
  size_t n;
  uint8_t* dst[8];  // codes destination per chunk pass (already offset by chunk start)
  int G;
};
template <int MODE>
__global__ void __launch_bounds__(kRingThreads, 1) mix_kernel(MixArgs a, unsigned long long* sched, int* st) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ PassDesc ps[8];
  Ring r;
  r.init(smem, st, 1000000000ull, sched);
  if (threadIdx.x == 0) {
    const size_t per = a.n / a.G;
    for (int i = 0; i < a.G; ++i) {
      ps[i] = PassDesc::make();
      ps[i].s = per * i;
      ps[i].n = per;
      ps[i].base[0] = reinterpret_cast<const uint8_t*>(a.x);
      ps[i].reverse = true;
    }
  }
  __syncthreads();
  const size_t per = a.n / a.G;
  if (MODE == 2) {
    if (r.ct >= 0) {
      const size_t ng = per / 4;  // 4-code groups per chunk
      for (size_t gi = size_t(blockIdx.x) * kConsumers + r.ct; gi < ng * a.G; gi += size_t(gridDim.x) * kConsumers) {
        const int i = int(gi % a.G);
        reinterpret_cast<uint32_t*>(a.dst[i])[gi / a.G] = unsigned(gi);
      }
    }
  } else {
    float acc = 0.f;
    r.run_multi(ps, a.G, [&](int i, const uint8_t* s, size_t e0, size_t units, int) {
      const float4* xs = reinterpret_cast<const float4*>(s);
      uint32_t* d = reinterpret_cast<uint32_t*>(a.dst[i] + (e0 - per * i));
      for (int gi = r.ct; gi < int(units * 4); gi += kConsumers) {
        const uint32_t q = quantize4(xs[gi], -1.0f, 127.5f);
        if (MODE == 0)
          d[gi] = q;
        else
          acc += float(q & 1);
      }
    });
    if (acc == 12345.f) st[1] = 1;
  }
  r.finish(reinterpret_cast<unsigned*>(sched + 64));
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
      PullArgs pa{};
      pa.src[0] = buf[(d + s) % G];
      pa.nsrc = 1;
      pull_kernel<<<nsm, kRingThreads, kRingSmem>>>(pa, bytes, outs[d], sts[d]);
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
  {  // fold-shaped pulls: G sources per tile (1 local + G-1 peers), 32 KB / G per copy
    for (int ns : {1, 2, 4}) {
      float t = timed([&](int d) {
        PullArgs pa{};
        pa.nsrc = ns;
        for (int j = 0; j < ns; ++j) pa.src[j] = buf[(d + 1) % G] + j * (bytes / ns);
        pull_kernel<<<nsm, kRingThreads, kRingSmem>>>(pa, bytes, outs[d], sts[d]);
      });
      printf("G=%d pull from 1 peer, %d copies of %d KB per tile: %.0f GB/s\n", G, ns, 32 / ns, bytes / t / 1e6);
    }
    float t = timed([&](int d) {
      PullArgs pa{};
      pa.nsrc = G;
      for (int j = 0; j < G; ++j) pa.src[j] = buf[(d + j) % G];  // j == 0: local
      pull_kernel<<<nsm, kRingThreads, kRingSmem>>>(pa, bytes, outs[d], sts[d]);
    });
    printf("G=%d fold-shaped pull (1 local + %d peers per tile): %.0f GB/s remote ingress\n", G, G - 1,
           bytes * (G - 1) / G / t / 1e6);
    std::vector<float4*> outs4(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMalloc(&outs4[d], bytes * 4));
    }
    float t2 = timed([&](int d) {
      PullArgs pa{};
      pa.nsrc = G;
      pa.out = outs4[d];
      for (int j = 0; j < G; ++j) pa.src[j] = buf[(d + j) % G];
      pull_kernel<<<nsm, kRingThreads, kRingSmem>>>(pa, bytes, outs[d], sts[d]);
    });
    printf("G=%d fold-shaped pull + 4x local fp32 writes (phase-3 shape): %.0f GB/s remote ingress, %.0f GB/s "
           "written\n", G, bytes * (G - 1) / G / t2 / 1e6, bytes * 4.0 / t2 / 1e6);
  }
  {  // the C_LP_S phase-1B traffic mix at 100M fp32 per GPU
    const size_t n = 100000000;
    std::vector<float*> xs(G);
    std::vector<uint8_t*> recv(G);
    std::vector<unsigned long long*> sch(G);
    for (int d = 0; d < G; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaMalloc(&xs[d], n * 4));
      CK(cudaMemset(xs[d], 0, n * 4));
      CK(cudaMalloc(&recv[d], n));  // G slots of n/G codes
      CK(cudaMalloc(&sch[d], 65 * 8));
      CK(cudaMemset(sch[d], 0, 65 * 8));
      CK(cudaFuncSetAttribute(mix_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
      CK(cudaFuncSetAttribute(mix_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
      CK(cudaFuncSetAttribute(mix_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingSmem));
    }
    std::vector<MixArgs> ma(G);
    const size_t per = n / G;
    for (int d = 0; d < G; ++d) {
      ma[d].x = xs[d];
      ma[d].n = n;
      ma[d].G = G;
      for (int i = 0; i < G; ++i) {
        const int k = (d + 1 + i) % G;
        ma[d].dst[i] = recv[k] + per * d;  // owner k, slot d
      }
    }
    float t0 = timed([&](int d) { mix_kernel<0><<<nsm, kRingThreads, kRingSmem>>>(ma[d], sch[d], sts[d]); });
    float t1 = timed([&](int d) { mix_kernel<1><<<nsm, kRingThreads, kRingSmem>>>(ma[d], sch[d], sts[d]); });
    float t2 = timed([&](int d) { mix_kernel<2><<<nsm, kRingThreads, kRingSmem>>>(ma[d], sch[d], sts[d]); });
    printf("G=%d 1B mix (100M fp32/GPU): read x + push codes %.1f us | read x only %.1f us | push codes only %.1f us "
           "(%.0f GB/s egress)\n",
           G, t0 * 1e3, t1 * 1e3, t2 * 1e3, per * (G - 1) / t2 / 1e6);
  }
  return 0;
}
