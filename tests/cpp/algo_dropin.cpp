// algo_dropin.cpp -- the reference's OWN training algorithms
// (/root/reference/proj/src/algorithms.cpp, compiled unmodified) driven for k
// steps over g workers, once on the reference's CPU SimCluster and once with
// the B200 primitives linked in place of collectives.cpp
// (paper_2107_01499_b200/host/rcomm_link.cpp).  The same source builds both
// binaries (paper_2107_01499_b200/build.py build_dropin):
//
//   algo_dropin_ref   -DDROPIN_REF: SimCluster + fast_profile, collectives.cpp
//   algo_dropin_b200  rcomm::NvlEndpoint per GPU (thread per GPU), rcomm_link.cpp
//
//   ./algo_dropin_{ref,b200} <algorithm> <workers> <steps> <out_prefix>
//
// Each worker writes its final parameters (all buckets, bucket order) to
// <out_prefix>_rank<r>.bin; tests/test_gpu_dropin.py compares the two runs
// bit for bit, in the style of acceptance.cpp:741-795 (sim vs tcp params).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "rcomm/algorithms.hpp"
#include "rcomm/engine.hpp"
#include "rcomm/tensor.hpp"
#include "rcomm/transport.hpp"
#ifndef DROPIN_REF
#include "rcomm_b200/rcomm_link.hpp"
#endif

using namespace rcomm;

namespace {

// deterministic uniform [-1, 1) values, 24-bit grid (splitmix64)
float synth(std::uint64_t seed, std::uint64_t i) {
  std::uint64_t z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return static_cast<float>(static_cast<std::int64_t>(z >> 40) - (1 << 23)) / static_cast<float>(1 << 23);
}

const std::vector<std::size_t> kLayers0 = {1000, 37, 70001, 5, 250000, 4096, 33333};
// B2_DROPIN_SCALE=<k>: every layer k times larger (the ring kernels' sizes)
std::vector<std::size_t> layers() {
  const char* e = std::getenv("B2_DROPIN_SCALE");
  const std::size_t k = e ? std::strtoull(e, nullptr, 10) : 1;
  std::vector<std::size_t> v = kLayers0;
  for (auto& n : v) n *= (k > 0 ? k : 1);
  return v;
}
const std::vector<std::size_t> kLayers = layers();

void worker(Endpoint& ep, AlgorithmName algo, int steps, const std::string& out) {
  const int r = ep.rank();
  // buckets of two consecutive layers (backward order, like the engine's packing)
  std::vector<std::vector<FlatTensor>> params, grads;
  std::vector<Bucket> buckets;
  for (std::size_t b = 0; 2 * b < kLayers.size(); ++b) {
    Bucket bk;
    bk.id = b;
    std::vector<FlatTensor*> pp, gg;
    params.emplace_back();
    grads.emplace_back();
    params.back().reserve(2);
    grads.back().reserve(2);
    for (std::size_t l = 2 * b; l < std::min(kLayers.size(), 2 * b + 2); ++l) {
      std::vector<float> init(kLayers[l]);
      for (std::size_t i = 0; i < init.size(); ++i) init[i] = 0.5f * synth(100 + l, i);  // identical replicas
      params.back().emplace_back("p" + std::to_string(l), std::vector<std::size_t>{kLayers[l]}, init);
      grads.back().emplace_back("g" + std::to_string(l), std::vector<std::size_t>{kLayers[l]},
                                std::vector<float>(kLayers[l], 0.0f));
      bk.layers.push_back(l);
      bk.elements += kLayers[l];
    }
    for (auto& t : params.back()) pp.push_back(&t);
    for (auto& t : grads.back()) gg.push_back(&t);
    bk.params = BucketArena::flatten(pp);
    bk.grads = BucketArena::flatten(gg);
    bk.trigger_layer = bk.layers.back();
    buckets.push_back(std::move(bk));
  }
  AlgoParams p;
  p.gamma = 0.05;
  p.warmup_steps = 2;
  p.topology.kind = TopologyKind::ring;
  p.topology.n = ep.world_size();
  p.rng_seed = 1234u + static_cast<std::uint32_t>(r);
  EngineOptions opts;
  auto comm = make_algorithm(algo, p);
  comm->setup(buckets, ep, opts);
  double now = 0.0;
  for (int s = 0; s < steps; ++s) {
    for (auto& b : buckets) {  // this worker's gradients of step s
      auto g = b.grads.span();
      for (std::size_t i = 0; i < g.size(); ++i)
        g[i] = synth(7000 + 1000ull * static_cast<std::uint64_t>(s) + 10ull * static_cast<std::uint64_t>(r) + b.id, i);
    }
    for (auto& b : buckets) now = comm->run(now, b, ep, opts);
    comm->end_iteration(ep);
  }
  std::ofstream f(out + "_rank" + std::to_string(r) + ".bin", std::ios::binary);
  for (auto& b : buckets)
    f.write(reinterpret_cast<const char*>(b.params.data()), static_cast<std::streamsize>(4 * b.params.size()));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s <algorithm> <workers> <steps> <out_prefix>\n", argv[0]);
    return 2;
  }
  const AlgorithmName algo = algorithm_from_string(argv[1]);
  const int world = std::atoi(argv[2]), steps = std::atoi(argv[3]);
  const std::string out = argv[4];
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(world));
  std::vector<std::thread> th;
#ifdef DROPIN_REF
  NetworkProfile prof;
  prof.intra_node = {0.0, 1e12};
  prof.inter_node = {0.0, 1e12};
  SimCluster cluster(world, prof);
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        worker(cluster.endpoint(r), algo, steps, out);
      } catch (...) {
        errs[static_cast<std::size_t>(r)] = std::current_exception();
        cluster.close();
      }
    });
#else
  // B2_DEVICES=<d>: rank r on GPU r % d (several ranks per GPU, each with its
  // own stream; with B2_SM_BUDGET=<148/(ranks per GPU)> their cooperative
  // kernels are co-resident) -- how tests/cpp/g8_emulation.py runs 8 ranks
  // on a 4-GPU box.  B2_TIMEOUT_MS bounds every rendezvous.
  const int ndev = std::getenv("B2_DEVICES") ? std::atoi(std::getenv("B2_DEVICES")) : world;
  const int budget = std::getenv("B2_SM_BUDGET") ? std::atoi(std::getenv("B2_SM_BUDGET")) : 0;
  const int tmo = std::getenv("B2_TIMEOUT_MS") ? std::atoi(std::getenv("B2_TIMEOUT_MS")) : 0;
  NvlThreadGroup tg(world);
  for (int r = 0; r < world; ++r)
    th.emplace_back([&, r] {
      try {
        NvlEndpoint ep(r, world, r % (ndev > 0 ? ndev : world), tg.allgather(r));
        if (budget > 0) b2_comm_set_sm_budget(ep.handle(), budget);
        if (tmo > 0) b2_comm_set_timeout_ms(ep.handle(), static_cast<std::uint64_t>(tmo));
        worker(ep, algo, steps, out);
        // a peer may still be pulling my last payload: nobody frees its
        // windows before everybody is done (the allgather is a barrier)
        int d = 0;
        std::vector<int> all(static_cast<std::size_t>(world));
        tg.allgather(r)(&d, sizeof d, all.data());
      } catch (...) {
        errs[static_cast<std::size_t>(r)] = std::current_exception();
      }
    });
#endif
  for (auto& t : th) t.join();
  int rc = 0;
  for (int r = 0; r < world; ++r)
    if (errs[static_cast<std::size_t>(r)]) {
      try {
        std::rethrow_exception(errs[static_cast<std::size_t>(r)]);
      } catch (const std::exception& e) {
        std::fprintf(stderr, "rank %d: %s\n", r, e.what());
      }
      rc = 1;
    }
  if (!rc) std::printf("{\"algorithm\": \"%s\", \"workers\": %d, \"steps\": %d, \"ok\": true}\n", argv[1], world, steps);
  return rc;
}
