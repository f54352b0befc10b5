// nvl_probe.cpp -- every GPU of the box runs `calls` back-to-back primitive
// calls on a device-resident bucket, one host thread per GPU in ONE process
// (so that `ncu --devices 0` can read device 0's NVLink / DRAM counters of a
// collective launch while the other GPUs run it unprofiled).
//
//   nvl_probe <prim: c_lp_s|c_fp_s|d_lp_s|d_fp_s> <elements> <calls> [gpus]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rcomm_b200/rcomm_b200.hpp"

using namespace rcomm::b200;

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s <prim> <elements> <calls> [gpus]\n", argv[0]);
    return 2;
  }
  const std::string prim = argv[1];
  const size_t n = std::strtoull(argv[2], nullptr, 10);
  const int calls = std::atoi(argv[3]);
  int g = 0;
  cudaGetDeviceCount(&g);
  if (argc > 4) g = std::min(g, std::atoi(argv[4]));
  if (g < 1) return 1;
  ThreadGroup tg(g);
  std::vector<std::thread> th;
  std::vector<int> rc(g, 0);
  for (int r = 0; r < g; ++r)
    th.emplace_back([&, r] {
      try {
        cudaSetDevice(r);
        B200Endpoint ep(r, g, r, tg.allgather(r));
        float* x = nullptr;
        cudaMalloc(&x, n * sizeof(float));
        b2_fill_synthetic(x, n, 2026 + r, 0, ep.stream());
        std::vector<int> nb;
        for (int j : {(r + g - 1) % g, r, (r + 1) % g})
          if (std::find(nb.begin(), nb.end(), j) == nb.end()) nb.push_back(j);
        std::sort(nb.begin(), nb.end());
        for (int i = 0; i < calls; ++i) {
          int s = B2_OK;
          if (prim == "c_lp_s")
            s = b2_c_lp_s(ep.handle(), x, n, B2_CODEC_UNIFORM8, nullptr, 0, nullptr, 0, 1, ep.stream());
          else if (prim == "c_fp_s")
            s = b2_c_fp_s(ep.handle(), x, n, 1, ep.stream());
          else if (prim == "d_lp_s")
            s = b2_d_lp_s(ep.handle(), x, n, nb.data(), int(nb.size()), B2_CODEC_UNIFORM8, B2_REDUCE_AVERAGE, 1,
                          ep.stream());
          else
            s = b2_d_fp_s(ep.handle(), x, n, nb.data(), int(nb.size()), B2_REDUCE_AVERAGE, 1, ep.stream());
          if (s != B2_OK) throw Error(s, b2_last_error());
        }
        ep.sync();
        int d = 0;
        std::vector<int> all(g);
        tg.allgather(r)(&d, sizeof d, all.data());  // nobody frees a window a peer still reads
        cudaFree(x);
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
        rc[r] = 1;
      }
    });
  for (auto& t : th) t.join();
  for (int v : rc)
    if (v) return 1;
  std::printf("{\"prim\": \"%s\", \"elements\": %zu, \"calls\": %d, \"gpus\": %d, \"ok\": true}\n", prim.c_str(), n,
              calls, g);
  return 0;
}
