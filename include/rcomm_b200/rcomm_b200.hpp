// rcomm_b200.hpp -- C++ host layer over libb2comm (include/b2comm.h) that
// keeps rcomm's public API shape, so code written against
//   /root/reference/proj/include/rcomm/{collectives,codec,tensor}.hpp
// compiles against this header with `rcomm::` -> `rcomm::b200::` and an
// `Endpoint&` -> `B200Endpoint&`.
//
//   reference                                  here
//   Error (tensor.hpp:12-14)                   b200::Error (same base, std::runtime_error)
//   Codec / CodecKind / Rounding (codec.hpp)   b200::Codec (uniform8 + identity on the GPU)
//   ErrorState (codec.hpp:40-47)               b200::ErrorState (device buffers)
//   compensate_encode (codec.hpp:52-54)        b200::compensate_encode
//   FlatTensor / BucketArena (tensor.hpp)      b200::FlatTensor / b200::BucketArena (device arena)
//   Topology / ReduceMode / partition_range    b200::Topology / ReduceMode / partition_range
//   c_fp_s / c_lp_s / d_fp_s / d_lp_s          same names, same argument order and meaning
//   Endpoint (transport.hpp:52-85)             b200::B200Endpoint (one GPU per worker)
//
// Buffers: a std::span<float> may point at DEVICE memory (zero-copy, the fast
// path) or at HOST memory (e.g. the reference tests' std::vector<float>): host
// spans are staged through the GPU and copied back, so blocking semantics and
// results are identical.  Primitives are blocking (the reference's
// rendezvous semantics) and return `now` unchanged (no virtual clock).
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "b2comm.h"

namespace rcomm::b200 {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
  int status = B2_ERR_INVALID;
  Error(int st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};

// Throw b200::Error for a non-OK libb2comm status.
void check(int status);

enum class CodecKind { identity = B2_CODEC_IDENTITY, uniform8 = B2_CODEC_UNIFORM8, onebit = B2_CODEC_ONEBIT };
enum class Rounding { nearest, stochastic };
enum class TopologyKind { ring = B2_TOPO_RING, random = B2_TOPO_RANDOM, full = B2_TOPO_FULL };
enum class ReduceMode { sum = B2_REDUCE_SUM, average = B2_REDUCE_AVERAGE };

using Payload = std::vector<std::uint8_t>;

// codec.hpp:25-36.  encode/decode work on host or device spans; the payload
// is the exact reference wire layout [min f32][max f32][u8 x N] on the host.
struct Codec {
  CodecKind kind = CodecKind::identity;
  Rounding rounding = Rounding::nearest;

  bool lossless() const { return kind == CodecKind::identity; }
  std::size_t payload_size(std::size_t n) const { return b2_payload_size(static_cast<int>(kind), n); }
  Payload encode(std::span<const float> x, std::mt19937* rng = nullptr) const;
  void decode(std::span<const std::uint8_t> payload, std::span<float> out) const;
  std::vector<float> decode(std::span<const std::uint8_t> payload, std::size_t n) const;
};

// Device-resident error-feedback state (codec.hpp:40-47).  delta/epsilon are
// device buffers; read them back with delta_host()/epsilon_host().
class ErrorState {
 public:
  ErrorState() = default;
  ErrorState(std::size_t bucket_len, std::size_t owned_len, int device = -1);
  ~ErrorState();
  ErrorState(const ErrorState&) = delete;
  ErrorState& operator=(const ErrorState&) = delete;
  ErrorState(ErrorState&& o) noexcept;
  ErrorState& operator=(ErrorState&& o) noexcept;

  float* delta() { return delta_; }
  float* epsilon() { return eps_; }
  std::size_t delta_len() const { return dlen_; }
  std::size_t epsilon_len() const { return elen_; }
  std::vector<float> delta_host() const;
  std::vector<float> epsilon_host() const;

 private:
  float* delta_ = nullptr;
  float* eps_ = nullptr;
  std::size_t dlen_ = 0, elen_ = 0;
};

// codec.hpp:52-54 (uniform8): encodes Q(x - delta), delta <- exact residual.
// x and delta are host or device spans of equal length.
Payload compensate_encode(const Codec& codec, std::span<const float> x, std::span<float> delta,
                          std::mt19937* rng = nullptr, std::vector<float>* decoded = nullptr);

std::pair<std::size_t, std::size_t> partition_range(std::size_t len, int n, int k);
std::size_t owned_partition_len(std::size_t len, int world, int idx);

struct Topology {  // collectives.hpp:18-25
  TopologyKind kind = TopologyKind::full;
  int n = 1;
  std::uint64_t seed = 0;
  std::vector<int> neighbors(int rank, std::uint64_t round) const;
};

namespace phase {  // collectives.hpp:29-38
constexpr std::uint32_t scatter = 0, gather = 1, inter = 2, bcast = 3;
constexpr std::uint32_t make_tag(std::uint32_t bucket, std::uint32_t ph) { return bucket * 16 + ph; }
}  // namespace phase

// Window-handle exchange among the workers (the only host-side
// communication): gather `bytes` from every rank into recv (rank-major).
using AllGather = std::function<void(const void* send, std::size_t bytes, void* recv)>;

// An in-process group of worker threads, one per GPU -- SimCluster's threading
// model (sim_transport.cpp:93-128) with real devices.
class ThreadGroup {
 public:
  explicit ThreadGroup(int world);
  ~ThreadGroup();
  int world() const;
  AllGather allgather(int rank);

 private:
  struct State;
  std::shared_ptr<State> s_;
};

// One worker's endpoint on one GPU (the role of rcomm::Endpoint).
class B200Endpoint {
 public:
  B200Endpoint(int rank, int world, int device, AllGather allgather = {});
  ~B200Endpoint();
  B200Endpoint(const B200Endpoint&) = delete;
  B200Endpoint& operator=(const B200Endpoint&) = delete;

  int rank() const { return rank_; }
  int node() const { return 0; }
  int world_size() const { return world_; }
  int node_of(int r) const;
  int device() const { return device_; }
  b2_comm_t handle() const { return comm_; }
  void* stream() const { return stream_; }

  std::uint64_t bytes_sent() const { return bytes_sent_; }
  std::uint64_t messages_sent() const { return messages_sent_; }
  void reset_counters() { bytes_sent_ = messages_sent_ = 0; }
  void account(std::uint64_t bytes, std::uint64_t msgs) {
    bytes_sent_ += bytes;
    messages_sent_ += msgs;
  }
  // Synchronize this endpoint's stream, throw on a latched device error.
  void sync();
  // Device staging buffer of a host bucket, cached per (bucket, length).
  float* staging(std::uint32_t bucket, std::size_t n);

 private:
  static int gather_trampoline(void* user, const void* send, std::size_t bytes, void* recv);
  int rank_, world_, device_;
  AllGather allgather_;
  b2_comm_t comm_ = nullptr;
  void* stream_ = nullptr;  // cudaStream_t owned by the endpoint
  std::uint64_t bytes_sent_ = 0, messages_sent_ = 0;
  std::map<std::pair<std::uint32_t, std::size_t>, void*> staging_;
};

// collectives.hpp:50-72 -- same names, argument order and meaning.
double c_fp_s(B200Endpoint& ep, double now, std::span<float> x, std::uint32_t bucket = 0);
double c_lp_s(B200Endpoint& ep, double now, std::span<float> x, const Codec& codec, ErrorState* es,
              std::mt19937* rng = nullptr, std::uint32_t bucket = 0);
double d_fp_s(B200Endpoint& ep, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              ReduceMode mode, std::uint32_t bucket = 0);
// collectives.hpp:80-82 over one NVLink node (every rank of the endpoint):
// the reference's member fold without compression, whatever the codec
double hierarchical_c(B200Endpoint& ep, double now, std::span<float> x, const Codec& codec, ErrorState* es,
                      std::mt19937* rng = nullptr, std::uint32_t bucket = 0);
double d_lp_s(B200Endpoint& ep, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              const Codec& codec, ReduceMode mode, std::mt19937* rng = nullptr, std::uint32_t bucket = 0);

// tensor.hpp:16-86 over device memory.  After flatten() every member is a
// view into the arena: writes through either handle alias (tensor.cpp:63-64).
class FlatTensor {
 public:
  FlatTensor() = default;
  FlatTensor(std::string name, std::vector<std::size_t> shape);  // zeros on the current device
  FlatTensor(std::string name, std::vector<std::size_t> shape, const std::vector<float>& values, int device = -1);

  const std::string& name() const { return name_; }
  const std::vector<std::size_t>& shape() const { return shape_; }
  std::size_t size() const { return len_; }
  float* data() { return storage_ ? storage_.get() + offset_ : nullptr; }  // device pointer
  const float* data() const { return storage_ ? storage_.get() + offset_ : nullptr; }
  std::span<float> span() { return {data(), len_}; }
  std::vector<float> to_host() const;
  bool is_view() const { return offset_ != 0 || capacity_ != len_; }

 private:
  friend class BucketArena;
  std::string name_;
  std::vector<std::size_t> shape_;
  std::shared_ptr<float> storage_;  // device allocation (cudaFree deleter)
  std::size_t offset_ = 0, len_ = 0, capacity_ = 0;
};

struct TensorView {
  std::string name;
  std::size_t offset;
  std::size_t length;
};

class BucketArena {
 public:
  const std::vector<TensorView>& members() const { return members_; }
  std::size_t size() const { return len_; }
  float* data() { return storage_.get(); }
  std::span<float> span() { return {storage_.get(), len_}; }
  FlatTensor as_flat(const std::string& name = "arena") const;
  static BucketArena flatten(std::span<FlatTensor*> tensors);
  static BucketArena flatten(std::vector<FlatTensor*> tensors) { return flatten(std::span<FlatTensor*>(tensors)); }

 private:
  std::shared_ptr<float> storage_;
  std::size_t len_ = 0;
  std::vector<TensorView> members_;
};

// ----------------------------------------------------------------- engine
// engine.hpp / engine.cpp:76-107: greedy reverse-order gradient bucketing
// (layer L-1 first; a bucket closes when the next layer would exceed the
// capacity; fusion off = one bucket per layer), and communication overlapping
// backward: at a bucket's trigger layer (its last member to finish backward)
// the bucket's collective is issued on a dedicated stream behind an event of
// the compute stream.
struct EngineBucket {
  std::size_t id = 0;
  std::vector<std::size_t> layers;  // backward order
  std::size_t trigger_layer = 0;
  std::size_t elements = 0;
};
std::vector<EngineBucket> plan_buckets(const std::vector<std::size_t>& layer_sizes,
                                       std::size_t capacity_bytes = std::size_t(8) << 20, bool fusion = true);

class OverlapEngine {
 public:
  enum class Primitive { c_lp_s, c_fp_s };
  OverlapEngine(B200Endpoint& ep, std::vector<std::size_t> layer_sizes,
                std::size_t capacity_bytes = std::size_t(8) << 20, bool fusion = true,
                Primitive prim = Primitive::c_lp_s, std::uint32_t bucket_base = 1u << 20);
  ~OverlapEngine();
  OverlapEngine(const OverlapEngine&) = delete;
  OverlapEngine& operator=(const OverlapEngine&) = delete;

  const std::vector<EngineBucket>& buckets() const { return buckets_; }
  float* grad(std::size_t layer);                // device view into the bucket arena
  std::span<float> arena(std::size_t bucket);    // device span of one bucket
  // layer's gradient is complete on compute_stream (cudaStream_t)
  void layer_done(std::size_t layer, void* compute_stream);
  // compute_stream waits for every bucket issued since the last finish().
  // Non-blocking: a device error of these buckets is thrown by synchronize(),
  // or by the next finish() once they have completed (one iteration late).
  void finish(void* compute_stream);
  // wait for every bucket issued so far; throw a latched device error
  void synchronize();

 private:
  B200Endpoint& ep_;
  Primitive prim_;
  std::uint32_t base_;
  std::vector<std::size_t> sizes_;
  std::vector<EngineBucket> buckets_;
  std::vector<std::size_t> bucket_of_, offset_;
  std::vector<float*> arenas_;
  void* comm_ = nullptr;  // cudaStream_t
  void* done_ = nullptr;  // cudaEvent_t: the last finish()'s buckets complete
  bool issued_ = false;
  std::size_t pending_ = 0;
};

}  // namespace rcomm::b200
