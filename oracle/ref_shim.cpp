// ref_shim.cpp -- C entry points into the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles the reference's own translation units in place
// from /root/reference/proj/src (kernels, kernels_avx2, tensor, codec,
// collectives, sim_transport) together with this file into
// oracle/_ref/librcomm_ref.so.  Nothing here re-implements the algorithm: each
// function drives the reference's public API (collectives.hpp, codec.hpp)
// through its own SimCluster + fast_profile harness, exactly like
// tests/test_collectives.cpp:14-39 does, so the outputs ARE the reference's.
//
// Used by: tests/golden/make_golden.py (fixture generation), the CPU parity
// tests, and bench.py --impl reference / cpu_baseline (timing).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "rcomm/codec.hpp"
#include "rcomm/collectives.hpp"
#include "rcomm/kernels.hpp"
#include "rcomm/tensor.hpp"
#include "rcomm/transport.hpp"

using namespace rcomm;

namespace {

thread_local std::string g_err;

NetworkProfile fast_profile() {  // test_collectives.cpp:14-19
  NetworkProfile p;
  p.intra_node = {0.0, 1e12};
  p.inter_node = {0.0, 1e12};
  return p;
}

template <typename F>
void run_workers(SimCluster& cluster, int n, F fn) {  // test_collectives.cpp:23-39
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errors(static_cast<std::size_t>(n));
  for (int r = 0; r < n; ++r)
    threads.emplace_back([&, r] {
      try {
        fn(cluster.endpoint(r), r);
      } catch (...) {
        errors[static_cast<std::size_t>(r)] = std::current_exception();
        cluster.close();
      }
    });
  for (auto& t : threads) t.join();
  for (auto& e : errors)
    if (e) std::rethrow_exception(e);
}

template <typename F>
int guarded(F fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

Codec make_codec(int kind) {
  return Codec{kind == 0 ? CodecKind::identity : kind == 2 ? CodecKind::onebit : CodecKind::uniform8,
               Rounding::nearest};
}

Topology make_topo(int kind, int n, std::uint64_t seed) {
  Topology t;
  t.kind = kind == 0 ? TopologyKind::ring
                     : (kind == 1 ? TopologyKind::random : TopologyKind::full);
  t.n = n;
  t.seed = seed;
  return t;
}

std::uint64_t splitmix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void synth(float* x, std::size_t n, std::uint64_t seed) {  // = orc_synth
  const std::uint64_t key = splitmix64(seed);
  for (std::size_t i = 0; i < n; ++i) {
    const std::uint64_t h = splitmix64(key + i);
    const std::int32_t m = static_cast<std::int32_t>(h >> 40);
    x[i] = static_cast<float>(m - 8388608) * 1.1920928955078125e-07f;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

const char* ref_backend() {
  return kernels::backend_name(kernels::active_backend());
}

int ref_force_backend(int scalar0_avx2_1) {
  return guarded([&] {
    kernels::force_backend(scalar0_avx2_1 ? kernels::Backend::avx2
                                          : kernels::Backend::scalar);
  });
}

void ref_partition_range(std::size_t len, int n, int k, std::size_t* lo,
                         std::size_t* sz) {
  auto [a, b] = partition_range(len, n, k);
  *lo = a;
  *sz = b;
}

// Codec::encode (codec.hpp:32).  wire must hold payload_size(n) bytes.
int ref_encode(int codec, const float* x, std::size_t n, std::uint8_t* wire) {
  return guarded([&] {
    Payload p = make_codec(codec).encode(std::span<const float>(x, n));
    std::memcpy(wire, p.data(), p.size());
  });
}

int ref_decode(int codec, const std::uint8_t* wire, std::size_t wire_len,
               std::size_t n, float* out) {
  return guarded([&] {
    make_codec(codec).decode(std::span<const std::uint8_t>(wire, wire_len),
                             std::span<float>(out, n));
  });
}

// compensate_encode (codec.hpp:52-54)
int ref_compensate_encode(int codec, const float* x, float* delta,
                          std::size_t n, std::uint8_t* wire, float* decoded) {
  return guarded([&] {
    std::vector<float> dec;
    Payload p = compensate_encode(make_codec(codec),
                                  std::span<const float>(x, n),
                                  std::span<float>(delta, n), nullptr, &dec);
    std::memcpy(wire, p.data(), p.size());
    if (decoded && n) std::memcpy(decoded, dec.data(), 4 * n);
  });
}

// kernels.hpp raw loops (for the reference's own quantize KATs)
void ref_quantize_u8(const float* x, std::uint8_t* out, float min,
                     float inv_step, std::size_t n) {
  kernels::quantize_u8(x, out, min, inv_step, n);
}
void ref_minmax(const float* x, std::size_t n, float* lo, float* hi) {
  auto [a, b] = kernels::minmax(x, n);
  *lo = a;
  *hi = b;
}

// c_fp_s over g worker threads; xs[r] updated in place.
int ref_c_fp_s(int g, std::size_t len, float* const* xs, std::uint64_t* bytes_sent,
               std::uint64_t* msgs_sent) {
  return guarded([&] {
    SimCluster cluster(g, fast_profile());
    run_workers(cluster, g, [&](Endpoint& ep, int r) {
      c_fp_s(ep, 0.0, std::span<float>(xs[r], len));
    });
    for (int r = 0; r < g; ++r) {
      if (bytes_sent) bytes_sent[r] = cluster.endpoint(r).bytes_sent();
      if (msgs_sent) msgs_sent[r] = cluster.endpoint(r).messages_sent();
    }
  });
}

// c_lp_s; deltas/eps NULL = stateless, else per-rank ErrorState in/out.
int ref_c_lp_s(int g, std::size_t len, float* const* xs, int codec,
               float* const* deltas, float* const* eps, int rounds,
               std::uint64_t* bytes_sent) {
  return guarded([&] {
    SimCluster cluster(g, fast_profile());
    const Codec c = make_codec(codec);
    run_workers(cluster, g, [&](Endpoint& ep, int r) {
      const std::size_t own = owned_partition_len(len, g, r);
      if (deltas) {
        ErrorState es(len, own);
        std::memcpy(es.delta.data(), deltas[r], 4 * len);
        if (own) std::memcpy(es.epsilon.data(), eps[r], 4 * own);
        for (int t = 0; t < rounds; ++t)
          c_lp_s(ep, 0.0, std::span<float>(xs[r], len), c, &es);
        std::memcpy(deltas[r], es.delta.data(), 4 * len);
        if (own) std::memcpy(eps[r], es.epsilon.data(), 4 * own);
      } else {
        for (int t = 0; t < rounds; ++t)
          c_lp_s(ep, 0.0, std::span<float>(xs[r], len), c, nullptr);
      }
    });
    if (bytes_sent)
      for (int r = 0; r < g; ++r) bytes_sent[r] = cluster.endpoint(r).bytes_sent();
  });
}

// hierarchical_c (collectives.cpp:290-385) on a SimCluster whose ranks sit
// on nodes[r] (sim_transport.hpp node assignment), no error feedback.
int ref_hierarchical_c(int g, std::size_t len, float* const* xs, const int* nodes, int codec) {
  return guarded([&] {
    SimCluster cluster(g, fast_profile(), std::vector<int>(nodes, nodes + g));
    const Codec c = make_codec(codec);
    run_workers(cluster, g, [&](Endpoint& ep, int r) {
      hierarchical_c(ep, 0.0, std::span<float>(xs[r], len), c, nullptr);
    });
  });
}

int ref_d_fp_s(int g, std::size_t len, float* const* xs, int topo_kind,
               std::uint64_t seed, std::uint64_t round, int mode) {
  return guarded([&] {
    SimCluster cluster(g, fast_profile());
    const Topology topo = make_topo(topo_kind, g, seed);
    run_workers(cluster, g, [&](Endpoint& ep, int r) {
      d_fp_s(ep, 0.0, std::span<float>(xs[r], len), topo, round,
             mode ? ReduceMode::average : ReduceMode::sum);
    });
  });
}

int ref_d_lp_s(int g, std::size_t len, float* const* xs, int topo_kind,
               std::uint64_t seed, std::uint64_t round, int codec, int mode) {
  return guarded([&] {
    SimCluster cluster(g, fast_profile());
    const Topology topo = make_topo(topo_kind, g, seed);
    const Codec c = make_codec(codec);
    run_workers(cluster, g, [&](Endpoint& ep, int r) {
      d_lp_s(ep, 0.0, std::span<float>(xs[r], len), topo, round, c,
             mode ? ReduceMode::average : ReduceMode::sum);
    });
  });
}

// Topology::neighbors (collectives.cpp:181-213); returns the count or -1.
int ref_neighbors(int topo_kind, int n, std::uint64_t seed, int rank,
                  std::uint64_t round, int* out) {
  int count = -1;
  guarded([&] {
    auto v = make_topo(topo_kind, n, seed).neighbors(rank, round);
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    count = static_cast<int>(v.size());
  });
  return count;
}

// The reference tests' input generators (test_codec.cpp:53-60,
// test_collectives.cpp:41-47), for fixtures.
void ref_random_uniform(std::uint32_t seed, std::size_t n, float lo, float hi,
                        float* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<float> d(lo, hi);
  for (std::size_t i = 0; i < n; ++i) out[i] = d(rng);
}
void ref_random_normal(std::uint32_t seed, std::size_t n, float* out) {
  std::mt19937 rng(seed);
  std::normal_distribution<float> d(0.0f, 1.0f);
  for (std::size_t i = 0; i < n; ++i) out[i] = d(rng);
}

void ref_synth(float* x, std::size_t n, std::uint64_t seed) { synth(x, n, seed); }

// Timing harness for the CPU baseline: g worker threads on a
// SimCluster with fast_profile call the primitive once; wall time is taken
// from thread spawn to join and therefore includes the reference's own
// allocations and first touch.  Inputs are regenerated (untimed) before each
// repetition.  prim: 0 codec(encode+decode, g must be 1), 1 c_fp_s,
// 2 c_lp_s (uint8, no EC), 3 d_fp_s ring, 4 d_lp_s ring (uint8),
// 5 onebit codec (encode+decode, g must be 1), 6 c_lp_s (onebit, no EC),
// 7 d_lp_s ring (onebit).
int ref_time_primitive(int prim, int g, std::size_t len, int reps,
                       double* seconds) {
  return guarded([&] {
    std::vector<std::vector<float>> xs(static_cast<std::size_t>(g),
                                       std::vector<float>(len));
    const Codec u8 = make_codec(1);
    const Codec ob = make_codec(2);
    const Topology ring = make_topo(0, g, 0);
    for (int t = 0; t < reps; ++t) {
      {  // untimed: one generator thread per worker (full-size buckets, g up to 8)
        std::vector<std::thread> gen;
        for (int r = 0; r < g; ++r)
          gen.emplace_back([&, r] { synth(xs[static_cast<std::size_t>(r)].data(), len, 2026u + r); });
        for (auto& th : gen) th.join();
      }
      const auto t0 = std::chrono::steady_clock::now();
      if (prim == 0 || prim == 5) {  // standalone codec: uniform8 (0) or onebit (5)
        const Codec c = make_codec(prim == 0 ? 1 : 2);
        Payload p = c.encode(xs[0]);
        c.decode(p, std::span<float>(xs[0]));
      } else {
        SimCluster cluster(g, fast_profile());
        run_workers(cluster, g, [&](Endpoint& ep, int r) {
          std::span<float> x(xs[static_cast<std::size_t>(r)]);
          switch (prim) {
            case 1: c_fp_s(ep, 0.0, x); break;
            case 2: c_lp_s(ep, 0.0, x, u8, nullptr); break;
            case 3: d_fp_s(ep, 0.0, x, ring, 0, ReduceMode::average); break;
            case 4: d_lp_s(ep, 0.0, x, ring, 0, u8, ReduceMode::average); break;
            case 6: c_lp_s(ep, 0.0, x, ob, nullptr); break;
            case 7: d_lp_s(ep, 0.0, x, ring, 0, ob, ReduceMode::average); break;
            default: throw Error("unknown primitive");
          }
        });
      }
      seconds[t] = std::chrono::duration<double>(
                       std::chrono::steady_clock::now() - t0)
                       .count();
    }
  });
}

}  // extern "C"
