// rcomm_link.cpp -- the B200 primitives behind the reference's OWN API
// (include/rcomm_b200/rcomm_link.hpp).  Built instead of the reference's
// proj/src/collectives.cpp, against the reference's headers: every symbol
// collectives.cpp defines is defined here, so the reference's callers
// (algorithms.cpp, engine.cpp, runner.cpp, the tests) link against the
// sm_100a kernels of libb2comm.so unchanged.
//
// Host spans are staged through device buffers cached per (bucket, length)
// and per ErrorState; every call is a blocking rendezvous like the
// reference's (collectives.hpp:38-41), and the device status is checked
// BEFORE anything is written back, so a failing call (non-finite input:
// codec.cpp:24-27) leaves x and the error state untouched.
#include "rcomm_b200/rcomm_link.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

namespace rcomm {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

void b2_check(int status) {
  if (status != B2_OK) throw Error(std::string(b2_status_string(status)) + ": " + b2_last_error());
}

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

NvlEndpoint& nvl(Endpoint& ep) {
  auto* p = dynamic_cast<NvlEndpoint*>(&ep);
  if (!p) throw Error("the B200 collectives need an rcomm::NvlEndpoint (rcomm_b200/rcomm_link.hpp)");
  return *p;
}

void check_codec(const Codec& c, std::mt19937* rng) {
  if (c.kind == CodecKind::uniform8 && c.rounding == Rounding::stochastic && !rng)
    throw Error("uniform8 stochastic rounding needs a generator");  // codec.cpp:70
}
// Rounding::stochastic: one 64-bit seed per call from the caller's generator
// (the levels' distribution is the reference's; the draws are a counter hash
// on the device, not the mt19937 stream, codec.cpp:67-78)
bool stochastic(const Codec& c) { return c.kind == CodecKind::uniform8 && c.rounding == Rounding::stochastic; }
std::uint64_t draw_seed(std::mt19937* rng) { return (std::uint64_t((*rng)()) << 32) | std::uint64_t((*rng)()); }

std::size_t payload_bytes(const Codec& c, std::size_t n) {  // codec.cpp:31-38
  return b2_payload_size(static_cast<int>(c.kind), n);
}

}  // namespace

// ------------------------------------------------------------- staging
struct NvlEndpoint::Staging {
  int device;
  std::map<std::pair<std::uint32_t, std::size_t>, float*> x;                 // (bucket, len) -> device
  std::map<std::tuple<const void*, std::size_t, std::size_t>, float*> es;   // ErrorState -> delta|eps
  explicit Staging(int dev) : device(dev) {}
  ~Staging() {
    DeviceScope ds(device);
    for (auto& kv : x) cudaFree(kv.second);
    for (auto& kv : es) cudaFree(kv.second);
  }
  float* bucket(std::uint32_t b, std::size_t n) {
    auto& p = x[{b, n}];
    if (!p) cuda_check(cudaMalloc(&p, std::max<std::size_t>(n, 4) * sizeof(float)), "cudaMalloc bucket staging");
    return p;
  }
  float* state(const ErrorState* s) {
    auto& p = es[{s, s->delta.size(), s->epsilon.size()}];
    if (!p) {
      const std::size_t dl = (s->delta.size() + 3) / 4 * 4;  // epsilon 16-byte aligned after delta
      cuda_check(cudaMalloc(&p, std::max<std::size_t>(dl + s->epsilon.size(), 4) * sizeof(float)),
                 "cudaMalloc error-state staging");
    }
    return p;
  }
};

// Stage x (and the error state) in, run `launch`, check the device status,
// stage the results back out.
template <class F>
static void staged_call(NvlEndpoint& ep, std::uint32_t bucket, std::span<float> x, ErrorState* es, F&& launch) {
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  const std::size_t n = x.size();
  float* dx = ep.staging().bucket(bucket, n);
  float *dd = nullptr, *de = nullptr;
  if (n) cuda_check(cudaMemcpyAsync(dx, x.data(), 4 * n, cudaMemcpyHostToDevice, s), "stage bucket in");
  if (es) {
    dd = ep.staging().state(es);
    de = dd + (es->delta.size() + 3) / 4 * 4;
    if (!es->delta.empty())
      cuda_check(cudaMemcpyAsync(dd, es->delta.data(), 4 * es->delta.size(), cudaMemcpyHostToDevice, s), "delta in");
    if (!es->epsilon.empty())
      cuda_check(cudaMemcpyAsync(de, es->epsilon.data(), 4 * es->epsilon.size(), cudaMemcpyHostToDevice, s),
                 "epsilon in");
  }
  b2_check(launch(dx, dd, de, s));
  b2_check(b2_comm_sync(ep.handle(), s));  // the reference throws before x changes
  if (n) cuda_check(cudaMemcpyAsync(x.data(), dx, 4 * n, cudaMemcpyDeviceToHost, s), "stage bucket out");
  if (es) {
    if (!es->delta.empty())
      cuda_check(cudaMemcpyAsync(es->delta.data(), dd, 4 * es->delta.size(), cudaMemcpyDeviceToHost, s), "delta out");
    if (!es->epsilon.empty())
      cuda_check(cudaMemcpyAsync(es->epsilon.data(), de, 4 * es->epsilon.size(), cudaMemcpyDeviceToHost, s),
                 "epsilon out");
  }
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
}

// ------------------------------------------------------------- endpoint
int NvlEndpoint::gather_trampoline(void* user, const void* send, std::size_t bytes, void* recv) {
  try {
    static_cast<NvlEndpoint*>(user)->allgather_(send, bytes, recv);
    return 0;
  } catch (...) {
    return 1;
  }
}

NvlEndpoint::NvlEndpoint(int rank, int world, int device, AllGather allgather, std::vector<int> node_of)
    : rank_(rank), world_(world), device_(device), allgather_(std::move(allgather)), node_of_(std::move(node_of)) {
  if (node_of_.empty()) node_of_.assign(static_cast<std::size_t>(world_), 0);
  if (static_cast<int>(node_of_.size()) != world_) throw Error("NvlEndpoint: node_of size must equal the world size");
  DeviceScope ds(device_);
  cudaStream_t s;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_ = s;
  b2_check(b2_comm_create(world_, rank_, device_, allgather_ ? &NvlEndpoint::gather_trampoline : nullptr, this,
                          &comm_));
  staging_ = std::make_unique<Staging>(device_);
}

NvlEndpoint::~NvlEndpoint() {
  staging_.reset();
  if (comm_) b2_comm_destroy(comm_);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

int NvlEndpoint::node_of(int r) const {
  if (r < 0 || r >= world_) throw Error("unknown rank " + std::to_string(r));  // sim_transport.cpp:24-25
  return node_of_[static_cast<std::size_t>(r)];
}

double NvlEndpoint::send(double, int, std::uint32_t, std::span<const std::uint8_t>) {
  throw Error("NvlEndpoint: point-to-point send is not part of the B200 path (the primitives move data over NVLink)");
}
std::pair<double, Bytes> NvlEndpoint::recv(double, int, std::uint32_t) {
  throw Error("NvlEndpoint: point-to-point recv is not part of the B200 path (the primitives move data over NVLink)");
}

struct NvlThreadGroup::State {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::vector<std::uint8_t>> slots;
  int arrived = 0, departed = 0;
  std::uint64_t gen = 0;
};

NvlThreadGroup::NvlThreadGroup(int world) : s_(std::make_shared<State>()) {
  s_->world = world;
  s_->slots.resize(static_cast<std::size_t>(world));
}

NvlEndpoint::AllGather NvlThreadGroup::allgather(int rank) {
  auto s = s_;
  return [s, rank](const void* send, std::size_t bytes, void* recv) {
    std::unique_lock<std::mutex> lk(s->mu);
    const std::uint64_t g1 = s->gen;
    s->slots[static_cast<std::size_t>(rank)].assign(static_cast<const std::uint8_t*>(send),
                                                    static_cast<const std::uint8_t*>(send) + bytes);
    if (++s->arrived == s->world) {
      s->arrived = 0;
      ++s->gen;
      s->cv.notify_all();
    } else {
      s->cv.wait(lk, [&] { return s->gen != g1; });
    }
    for (int r = 0; r < s->world; ++r)
      std::memcpy(static_cast<std::uint8_t*>(recv) + static_cast<std::size_t>(r) * bytes,
                  s->slots[static_cast<std::size_t>(r)].data(), bytes);
    const std::uint64_t g2 = s->gen;  // nobody overwrites a slot before everyone copied it
    if (++s->departed == s->world) {
      s->departed = 0;
      ++s->gen;
      s->cv.notify_all();
    } else {
      s->cv.wait(lk, [&] { return s->gen != g2; });
    }
  };
}

// ------------------------------------------------- collectives.cpp symbols
std::pair<std::size_t, std::size_t> partition_range(std::size_t len, int n, int k) {  // collectives.cpp:167-175
  std::size_t lo, sz;
  b2_partition_range(len, n, k, &lo, &sz);
  return {lo, sz};
}

std::size_t owned_partition_len(std::size_t len, int world, int idx) {  // collectives.cpp:177-179
  return b2_owned_partition_len(len, world, idx);
}

std::vector<int> Topology::neighbors(int rank, std::uint64_t round) const {  // collectives.cpp:181-213
  if (rank < 0 || rank >= n) throw Error("topology: rank out of range");
  std::vector<int> out(static_cast<std::size_t>(std::max(n, 3)));
  const int m = b2_topology_neighbors(static_cast<int>(kind) == 0 ? B2_TOPO_RING
                                      : static_cast<int>(kind) == 1 ? B2_TOPO_RANDOM
                                                                    : B2_TOPO_FULL,
                                      n, seed, rank, round, out.data());
  if (m < 0) throw Error("topology: unknown kind");
  out.resize(static_cast<std::size_t>(m));
  return out;
}

double c_fp_s(Endpoint& ep_, double now, std::span<float> x, std::uint32_t bucket) {  // collectives.cpp:215-220
  NvlEndpoint& ep = nvl(ep_);
  const int g = ep.world_size(), me = ep.rank();
  if (g == 1) return now;  // scatter_reduce_fp: x untouched (collectives.cpp:49)
  staged_call(ep, bucket, x, nullptr, [&](float* dx, float*, float*, cudaStream_t s) {
    return b2_c_fp_s(ep.handle(), dx, x.size(), bucket, s);
  });
  const std::size_t own = owned_partition_len(x.size(), g, me);
  ep.account(4 * (x.size() - own) + 4 * own * std::size_t(g - 1), 2 * std::size_t(g - 1));
  return now;
}

double c_lp_s(Endpoint& ep_, double now, std::span<float> x, const Codec& codec, ErrorState* es,
              std::mt19937* rng, std::uint32_t bucket) {  // collectives.cpp:222-227, 91-163
  NvlEndpoint& ep = nvl(ep_);
  check_codec(codec, rng);
  const int g = ep.world_size(), me = ep.rank();
  const std::size_t len = x.size(), mylen = owned_partition_len(len, g, me);
  if (es) {  // collectives.cpp:102-107
    if (es->delta.size() != len) throw Error("c_lp_s: delta length does not match bucket length");
    if (es->epsilon.size() != mylen) throw Error("c_lp_s: epsilon length does not match owned partition");
  }
  const std::uint64_t seed = stochastic(codec) ? draw_seed(rng) : 0;
  staged_call(ep, bucket, x, es, [&](float* dx, float* dd, float* de, cudaStream_t s) {
    if (stochastic(codec))
      return b2_c_lp_s_stochastic(ep.handle(), dx, len, dd, es ? es->delta.size() : 0, es ? de : nullptr,
                                  es ? es->epsilon.size() : 0, seed, bucket, s);
    return b2_c_lp_s(ep.handle(), dx, len, static_cast<int>(codec.kind), dd, es ? es->delta.size() : 0,
                     es ? de : nullptr, es ? es->epsilon.size() : 0, bucket, s);
  });
  if (g > 1) {
    std::uint64_t sent = 0;
    for (int k = 0; k < g; ++k)
      if (k != me) sent += payload_bytes(codec, partition_range(len, g, k).second);
    sent += std::uint64_t(g - 1) * payload_bytes(codec, mylen);
    ep.account(sent, 2 * std::uint64_t(g - 1));
  }
  return now;
}

double d_fp_s(Endpoint& ep_, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              ReduceMode mode, std::uint32_t bucket) {  // collectives.cpp:229-258
  NvlEndpoint& ep = nvl(ep_);
  if (topo.n != ep.world_size()) throw Error("topology size mismatch");
  const auto nb = topo.neighbors(ep.rank(), round);
  staged_call(ep, bucket, x, nullptr, [&](float* dx, float*, float*, cudaStream_t s) {
    return b2_d_fp_s(ep.handle(), dx, x.size(), nb.data(), static_cast<int>(nb.size()),
                     mode == ReduceMode::average ? B2_REDUCE_AVERAGE : B2_REDUCE_SUM, bucket, s);
  });
  ep.account((nb.size() - 1) * 4 * x.size(), nb.size() - 1);
  return now;
}

double d_lp_s(Endpoint& ep_, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              const Codec& codec, ReduceMode mode, std::mt19937* rng, std::uint32_t bucket) {  // :260-288
  NvlEndpoint& ep = nvl(ep_);
  check_codec(codec, rng);
  if (topo.n != ep.world_size()) throw Error("topology size mismatch");
  const auto nb = topo.neighbors(ep.rank(), round);
  const std::uint64_t seed = stochastic(codec) ? draw_seed(rng) : 0;
  staged_call(ep, bucket, x, nullptr, [&](float* dx, float*, float*, cudaStream_t s) {
    const int md = mode == ReduceMode::average ? B2_REDUCE_AVERAGE : B2_REDUCE_SUM;
    if (stochastic(codec))
      return b2_d_lp_s_stochastic(ep.handle(), dx, x.size(), nb.data(), static_cast<int>(nb.size()), md, seed,
                                  bucket, s);
    return b2_d_lp_s(ep.handle(), dx, x.size(), nb.data(), static_cast<int>(nb.size()),
                     static_cast<int>(codec.kind), md, bucket, s);
  });
  ep.account((nb.size() - 1) * payload_bytes(codec, x.size()), nb.size() - 1);
  return now;
}

// collectives.cpp:290-385.  One node (every rank of an NVLink domain): the
// reference aggregates the members in fp64 in ascending rank order from +0.0
// and rounds once, with no compression -- for two or more ranks exactly
// C_FP_S's fold; for a single rank (float)(0.0 + (double)x), i.e. D_FP_S
// over the singleton neighbourhood (-0.0 becomes +0.0, as in the
// reference).  Nodes beyond one NVLink domain need an inter-node transport,
// which this path does not have.
double hierarchical_c(Endpoint& ep_, double now, std::span<float> x, const Codec& codec, ErrorState* es,
                      std::mt19937* rng, std::uint32_t bucket) {
  NvlEndpoint& ep = nvl(ep_);
  (void)es;
  (void)rng;
  (void)codec;
  const int n = ep.world_size();
  for (int r = 0; r < n; ++r)
    if (ep.node_of(r) != ep.node_of(0))
      throw Error("hierarchical_c: ranks on more than one node need an inter-node transport "
                  "(the B200 path spans one NVLink domain)");
  staged_call(ep, bucket, x, nullptr, [&](float* dx, float*, float*, cudaStream_t s) {
    return b2_hierarchical_c(ep.handle(), dx, x.size(), bucket, s);
  });
  return now;
}

}  // namespace rcomm
