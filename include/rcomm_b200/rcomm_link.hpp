// rcomm_link.hpp -- link-time drop-in of the B200 primitives UNDER the
// reference's own API (/root/reference/proj/include/rcomm/collectives.hpp).
//
// A maintainer builds paper_2107_01499_b200/host/rcomm_link.cpp INSTEAD of
// proj/src/collectives.cpp, against the reference's headers, and links
// libb2comm.so.  Every call site of the reference -- aggregate_centralized
// (algorithms.cpp:39-47), DecentralizedSgd::run (algorithms.cpp:187-202),
// OneBitAdam (algorithms.cpp:117,147), replica_param_spread, the engine --
// then runs the sm_100a kernels unchanged, with the reference's own
// rcomm::Codec / rcomm::ErrorState / rcomm::Topology types, host spans and
// blocking semantics.  The only new type is the endpoint: an
// rcomm::NvlEndpoint is an rcomm::Endpoint (transport.hpp:52-85) bound to one
// GPU of the NVLink/NVSwitch domain; the primitives take it through the
// reference's `Endpoint&` parameter.  Point-to-point send/recv are not part
// of this path and throw.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "b2comm.h"
#include "rcomm/collectives.hpp"
#include "rcomm/transport.hpp"

namespace rcomm {

class NvlEndpoint : public Endpoint {
 public:
  // allgather(send, bytes, recv): gather `bytes` from every rank into recv
  // (world * bytes, rank-major); used once per window to exchange handles.
  using AllGather = std::function<void(const void* send, std::size_t bytes, void* recv)>;
  // node_of[r]: node of rank r (hierarchical_c); empty = one node.
  NvlEndpoint(int rank, int world, int device, AllGather allgather, std::vector<int> node_of = {});
  ~NvlEndpoint() override;
  NvlEndpoint(const NvlEndpoint&) = delete;
  NvlEndpoint& operator=(const NvlEndpoint&) = delete;

  int rank() const override { return rank_; }
  int node() const override { return node_of_[static_cast<std::size_t>(rank_)]; }
  int world_size() const override { return world_; }
  int node_of(int rank) const override;

  // not part of the B200 hot path: the primitives move data over NVLink
  double send(double now, int dst, std::uint32_t tag, std::span<const std::uint8_t> payload) override;
  std::pair<double, Bytes> recv(double now, int src, std::uint32_t tag) override;
  double compute(double now, double seconds) override { return now + seconds; }
  void report_done(double) override {}

  std::uint64_t bytes_sent() const override { return bytes_sent_; }
  std::uint64_t messages_sent() const override { return messages_sent_; }
  void reset_counters() override { bytes_sent_ = messages_sent_ = 0; }

  // B200 side
  b2_comm_t handle() const { return comm_; }
  int device() const { return device_; }
  void* stream() const { return stream_; }
  void account(std::uint64_t bytes, std::uint64_t msgs) {
    bytes_sent_ += bytes;
    messages_sent_ += msgs;
  }
  struct Staging;  // cached device copies of host buckets / error states
  Staging& staging() { return *staging_; }

 private:
  static int gather_trampoline(void* user, const void* send, std::size_t bytes, void* recv);
  int rank_, world_, device_;
  AllGather allgather_;
  std::vector<int> node_of_;
  b2_comm_t comm_ = nullptr;
  void* stream_ = nullptr;
  std::unique_ptr<Staging> staging_;
  std::uint64_t bytes_sent_ = 0, messages_sent_ = 0;
};

// In-process rendezvous for one NvlEndpoint per thread (SimCluster's
// threading model, sim_transport.cpp:93-128): share one instance.
class NvlThreadGroup {
 public:
  explicit NvlThreadGroup(int world);
  NvlEndpoint::AllGather allgather(int rank);

 private:
  struct State;
  std::shared_ptr<State> s_;
};

}  // namespace rcomm
