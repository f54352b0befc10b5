// rcomm_b200.cpp -- C++ host layer over the C ABI (see include/rcomm_b200/rcomm_b200.hpp).
//
// Everything that computes goes through libb2comm's sm_100a kernels; this
// file only validates arguments the way the reference does, stages host
// spans through device memory, and turns status codes into exceptions.
#include "rcomm_b200/rcomm_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <unordered_set>

namespace rcomm::b200 {

void check(int status) {
  if (status != B2_OK)
    throw Error(status, std::string(b2_status_string(status)) + ": " + b2_last_error());
}

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(B2_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct DevBuf {  // owned device allocation
  void* p = nullptr;
  explicit DevBuf(std::size_t bytes) {
    if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// A float span resolved to a 16-byte aligned device buffer; host spans (and
// misaligned device spans) are staged through a device buffer cached per
// (endpoint, bucket, length) and written back by finish() -- which the
// primitives call only after ep.sync() has checked the device status, so a
// failing call leaves x untouched (the reference throws from encode before x
// changes, codec.cpp:24-27).
struct Staged {
  std::span<float> user;
  float* dev = nullptr;
  bool staged = false;
  Staged(B200Endpoint& ep, std::uint32_t bucket, std::span<float> x, cudaStream_t s) : user(x) {
    if (is_device_ptr(x.data()) && (reinterpret_cast<std::uintptr_t>(x.data()) & 15) == 0) {
      dev = x.data();
      return;
    }
    staged = true;
    dev = ep.staging(bucket, x.size());
    if (!x.empty())
      cuda_check(cudaMemcpyAsync(dev, x.data(), x.size() * sizeof(float), cudaMemcpyDefault, s), "stage in");
  }
  void finish(cudaStream_t s) {
    if (staged && !user.empty()) {
      cuda_check(cudaMemcpyAsync(user.data(), dev, user.size() * sizeof(float), cudaMemcpyDefault, s), "stage out");
      cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    }
  }
};

std::vector<float> to_host(std::span<const float> x) {
  std::vector<float> h(x.size());
  if (!x.empty()) cuda_check(cudaMemcpy(h.data(), x.data(), x.size() * 4, cudaMemcpyDefault), "copy to host");
  return h;
}

void check_codec(const Codec& c, std::mt19937* rng, bool collective = true) {
  (void)collective;
  if (c.kind == CodecKind::uniform8 && c.rounding == Rounding::stochastic && !rng)
    throw Error(B2_ERR_INVALID, "uniform8 stochastic rounding needs a generator");  // codec.cpp:70
}
bool stochastic(const Codec& c) { return c.kind == CodecKind::uniform8 && c.rounding == Rounding::stochastic; }
// one 64-bit seed per call, advancing the caller's generator (codec.cpp:71-74)
std::uint64_t draw_seed(std::mt19937* rng) { return (std::uint64_t((*rng)()) << 32) | std::uint64_t((*rng)()); }

}  // namespace

// ------------------------------------------------------------------ codec
Payload Codec::encode(std::span<const float> x, std::mt19937* rng) const {
  check_codec(*this, rng, /*collective=*/false);
  const std::size_t n = x.size();
  if (kind == CodecKind::identity) {  // codec.cpp:41,47-50: the payload is x, after check_finite
    if (n == 0) return {};
    DevBuf xs(4 * n), zero(4 * n), y(4 * n), flag(sizeof(int));
    cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage in");
    cuda_check(cudaMemset(zero.p, 0, 4 * n), "memset");
    cuda_check(cudaMemset(flag.p, 0, sizeof(int)), "memset");
    check(b2_identity_compensate_encode(xs.as<float>(), zero.as<float>(), n, y.as<float>(), flag.as<int>(), nullptr));
    int bad = 0;
    cuda_check(cudaMemcpy(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost), "flag");
    if (bad) throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");
    Payload p(4 * n);
    cuda_check(cudaMemcpy(p.data(), y.p, 4 * n, cudaMemcpyDeviceToHost), "copy payload");
    return p;
  }
  if (kind == CodecKind::onebit) {  // codec.cpp:81-88
    const std::size_t ps = payload_size(n);
    DevBuf xs((n ? n : 1) * 4), wire((ps + 15) / 16 * 16);
    if (n) cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage in");
    check(b2_onebit_encode(xs.as<float>(), n, wire.as<std::uint8_t>(), nullptr));
    Payload p(ps);
    cuda_check(cudaMemcpy(p.data(), wire.p, ps, cudaMemcpyDeviceToHost), "copy payload");
    float scale;
    std::memcpy(&scale, p.data(), 4);
    if (std::isnan(scale)) throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");  // the kernel's mark
    return p;
  }
  DevBuf xs((n ? n : 1) * 4), codes(n + 64), hdr(B2_U8_HDR_BYTES), wire(8 + n);
  if (n) cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage in");
  if (rounding == Rounding::stochastic) {  // seed drawn from (and advancing) the caller's mt19937
    const std::uint64_t seed = (std::uint64_t((*rng)()) << 32) | std::uint64_t((*rng)());
    check(b2_u8_encode_stochastic(xs.as<float>(), n, codes.as<std::uint8_t>(), hdr.as<float>(), seed, nullptr));
  } else {
    check(b2_u8_encode(xs.as<float>(), n, codes.as<std::uint8_t>(), hdr.as<float>(), nullptr));
  }
  check(b2_u8_pack_wire(codes.as<std::uint8_t>(), hdr.as<float>(), n, wire.as<std::uint8_t>(), nullptr));
  Payload p(8 + n);
  cuda_check(cudaMemcpy(p.data(), wire.p, 8 + n, cudaMemcpyDeviceToHost), "copy payload");
  float lohi[2];
  std::memcpy(lohi, p.data(), 8);
  if (!std::isfinite(lohi[0]) || !std::isfinite(lohi[1]))
    throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");  // codec.cpp:24-27
  return p;
}

void Codec::decode(std::span<const std::uint8_t> payload, std::span<float> out) const {
  const std::size_t n = out.size();
  if (payload.size() != payload_size(n)) throw Error(B2_ERR_INVALID, "decode: malformed payload (length mismatch)");
  if (n == 0) return;
  if (kind == CodecKind::onebit) {  // codec.cpp:110-114
    DevBuf wire((payload.size() + 15) / 16 * 16), res(4 * n);
    cuda_check(cudaMemcpy(wire.p, payload.data(), payload.size(), cudaMemcpyDefault), "stage payload");
    check(b2_onebit_decode(wire.as<std::uint8_t>(), n, res.as<float>(), nullptr));
    cuda_check(cudaMemcpy(out.data(), res.p, 4 * n, cudaMemcpyDefault), "copy out");
    return;
  }
  if (kind == CodecKind::identity) {
    cuda_check(cudaMemcpy(out.data(), payload.data(), 4 * n, cudaMemcpyDefault), "decode copy");
    return;
  }
  DevBuf wire(8 + n), codes(n + 64), hdr(B2_U8_HDR_BYTES), res(4 * n);
  cuda_check(cudaMemcpy(wire.p, payload.data(), 8 + n, cudaMemcpyDefault), "stage payload");
  check(b2_u8_unpack_wire(wire.as<std::uint8_t>(), n, codes.as<std::uint8_t>(), hdr.as<float>(), nullptr));
  check(b2_u8_decode(codes.as<std::uint8_t>(), hdr.as<float>(), n, res.as<float>(), nullptr));
  cuda_check(cudaMemcpy(out.data(), res.p, 4 * n, cudaMemcpyDefault), "copy out");
}

std::vector<float> Codec::decode(std::span<const std::uint8_t> payload, std::size_t n) const {
  std::vector<float> out(n);
  decode(payload, std::span<float>(out));
  return out;
}

Payload compensate_encode(const Codec& codec, std::span<const float> x, std::span<float> delta, std::mt19937* rng,
                          std::vector<float>* decoded) {
  check_codec(codec, rng);
  const std::size_t n = x.size();
  if (delta.size() != n) throw Error(B2_ERR_INVALID, "compensate_encode: length mismatch");  // codec.cpp:129
  if (codec.kind == CodecKind::onebit) {  // y = x - delta, P = Q(y), delta = y - D(P) (codec.cpp:130-136)
    const std::size_t ps = codec.payload_size(n);
    DevBuf xs((n ? n : 1) * 4), ds((n ? n : 1) * 4), dec((n ? n : 4) * 4), wire((ps + 15) / 16 * 16);
    if (n) {
      cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage x");
      cuda_check(cudaMemcpy(ds.p, delta.data(), 4 * n, cudaMemcpyDefault), "stage delta");
    }
    check(b2_onebit_compensate_encode(xs.as<float>(), ds.as<float>(), n, wire.as<std::uint8_t>(), dec.as<float>(),
                                      nullptr));
    Payload p(ps);
    cuda_check(cudaMemcpy(p.data(), wire.p, ps, cudaMemcpyDeviceToHost), "copy payload");
    float scale;
    std::memcpy(&scale, p.data(), 4);
    if (std::isnan(scale)) throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");  // before delta changes
    if (n) cuda_check(cudaMemcpy(delta.data(), ds.p, 4 * n, cudaMemcpyDefault), "delta out");
    if (decoded) {
      decoded->resize(n);
      if (n) cuda_check(cudaMemcpy(decoded->data(), dec.p, 4 * n, cudaMemcpyDeviceToHost), "decoded out");
    }
    return p;
  }
  if (codec.kind == CodecKind::identity) {
    DevBuf xs((n ? n : 1) * 4), ds((n ? n : 1) * 4), y((n ? n : 1) * 4), flag(sizeof(int));
    if (n) {
      cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage x");
      cuda_check(cudaMemcpy(ds.p, delta.data(), 4 * n, cudaMemcpyDefault), "stage delta");
    }
    cuda_check(cudaMemset(flag.p, 0, sizeof(int)), "memset");
    check(b2_identity_compensate_encode(xs.as<float>(), ds.as<float>(), n, y.as<float>(), flag.as<int>(), nullptr));
    int bad = 0;
    cuda_check(cudaMemcpy(&bad, flag.p, sizeof(int), cudaMemcpyDeviceToHost), "flag");
    if (bad) throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");  // codec.cpp:24-27, delta untouched
    Payload p(4 * n);
    if (n) {
      cuda_check(cudaMemcpy(p.data(), y.p, 4 * n, cudaMemcpyDeviceToHost), "copy payload");
      cuda_check(cudaMemcpy(delta.data(), ds.p, 4 * n, cudaMemcpyDefault), "delta out");
    }
    if (decoded) {
      decoded->resize(n);
      if (n) std::memcpy(decoded->data(), p.data(), 4 * n);
    }
    return p;
  }
  DevBuf xs((n ? n : 1) * 4), ds((n ? n : 1) * 4), codes(n + 64), hdr(B2_U8_HDR_BYTES), dec((n ? n : 1) * 4),
      wire(8 + n);
  if (n) {
    cuda_check(cudaMemcpy(xs.p, x.data(), 4 * n, cudaMemcpyDefault), "stage x");
    cuda_check(cudaMemcpy(ds.p, delta.data(), 4 * n, cudaMemcpyDefault), "stage delta");
  }
  check(b2_u8_compensate_encode(xs.as<float>(), ds.as<float>(), n, codes.as<std::uint8_t>(), hdr.as<float>(),
                                dec.as<float>(), nullptr));
  check(b2_u8_pack_wire(codes.as<std::uint8_t>(), hdr.as<float>(), n, wire.as<std::uint8_t>(), nullptr));
  Payload p(8 + n);
  cuda_check(cudaMemcpy(p.data(), wire.p, 8 + n, cudaMemcpyDeviceToHost), "copy payload");
  float lohi[2];
  std::memcpy(lohi, p.data(), 8);
  if (!std::isfinite(lohi[0]) || !std::isfinite(lohi[1]))
    throw Error(B2_ERR_NONFINITE, "encode: non-finite input value");
  if (n) cuda_check(cudaMemcpy(delta.data(), ds.p, 4 * n, cudaMemcpyDefault), "delta out");
  if (decoded) {
    decoded->resize(n);
    if (n) cuda_check(cudaMemcpy(decoded->data(), dec.p, 4 * n, cudaMemcpyDeviceToHost), "decoded out");
  }
  return p;
}

ErrorState::ErrorState(std::size_t bucket_len, std::size_t owned_len, int device) : dlen_(bucket_len), elen_(owned_len) {
  DeviceScope ds(device);
  cuda_check(cudaMalloc(&delta_, std::max<std::size_t>(dlen_, 4) * 4), "cudaMalloc delta");
  cuda_check(cudaMalloc(&eps_, std::max<std::size_t>(elen_, 4) * 4), "cudaMalloc epsilon");
  cuda_check(cudaMemset(delta_, 0, std::max<std::size_t>(dlen_, 4) * 4), "memset");
  cuda_check(cudaMemset(eps_, 0, std::max<std::size_t>(elen_, 4) * 4), "memset");
}
ErrorState::~ErrorState() {
  if (delta_) cudaFree(delta_);
  if (eps_) cudaFree(eps_);
}
ErrorState::ErrorState(ErrorState&& o) noexcept { *this = std::move(o); }
ErrorState& ErrorState::operator=(ErrorState&& o) noexcept {
  std::swap(delta_, o.delta_);
  std::swap(eps_, o.eps_);
  std::swap(dlen_, o.dlen_);
  std::swap(elen_, o.elen_);
  return *this;
}
std::vector<float> ErrorState::delta_host() const { return to_host({delta_, dlen_}); }
std::vector<float> ErrorState::epsilon_host() const { return to_host({eps_, elen_}); }

// ------------------------------------------------------------- topology
std::pair<std::size_t, std::size_t> partition_range(std::size_t len, int n, int k) {
  std::size_t lo, sz;
  b2_partition_range(len, n, k, &lo, &sz);
  return {lo, sz};
}
std::size_t owned_partition_len(std::size_t len, int world, int idx) { return b2_owned_partition_len(len, world, idx); }

std::vector<int> Topology::neighbors(int rank, std::uint64_t round) const {
  std::vector<int> out(static_cast<std::size_t>(std::max(n, 3)));
  const int m = b2_topology_neighbors(static_cast<int>(kind), n, seed, rank, round, out.data());
  if (m < 0) throw Error(B2_ERR_INVALID, b2_last_error());
  out.resize(static_cast<std::size_t>(m));
  return out;
}

// ---------------------------------------------------------- thread group
struct ThreadGroup::State {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::vector<std::uint8_t>> slots;
  int arrived = 0, departed = 0;
  std::uint64_t gen = 0;
};

ThreadGroup::ThreadGroup(int world) : s_(std::make_shared<State>()) {
  s_->world = world;
  s_->slots.resize(static_cast<std::size_t>(world));
}
ThreadGroup::~ThreadGroup() = default;
int ThreadGroup::world() const { return s_->world; }

AllGather ThreadGroup::allgather(int rank) {
  auto s = s_;
  return [s, rank](const void* send, std::size_t bytes, void* recv) {
    std::unique_lock<std::mutex> lk(s->mu);
    const std::uint64_t my_gen = s->gen;
    s->slots[static_cast<std::size_t>(rank)].assign(static_cast<const std::uint8_t*>(send),
                                                    static_cast<const std::uint8_t*>(send) + bytes);
    if (++s->arrived == s->world) {
      s->arrived = 0;
      ++s->gen;
      s->cv.notify_all();
    } else {
      s->cv.wait(lk, [&] { return s->gen != my_gen; });
    }
    for (int r = 0; r < s->world; ++r)
      std::memcpy(static_cast<std::uint8_t*>(recv) + static_cast<std::size_t>(r) * bytes,
                  s->slots[static_cast<std::size_t>(r)].data(), bytes);
    // second rendezvous: nobody overwrites a slot before everyone copied it
    const std::uint64_t g2 = s->gen;
    if (++s->departed == s->world) {
      s->departed = 0;
      ++s->gen;
      s->cv.notify_all();
    } else {
      s->cv.wait(lk, [&] { return s->gen != g2; });
    }
  };
}

// ---------------------------------------------------------------- endpoint
int B200Endpoint::gather_trampoline(void* user, const void* send, std::size_t bytes, void* recv) {
  try {
    static_cast<B200Endpoint*>(user)->allgather_(send, bytes, recv);
    return 0;
  } catch (...) {
    return 1;
  }
}

B200Endpoint::B200Endpoint(int rank, int world, int device, AllGather allgather)
    : rank_(rank), world_(world), device_(device), allgather_(std::move(allgather)) {
  DeviceScope ds(device_);
  cudaStream_t s;
  cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_ = s;
  check(b2_comm_create(world_, rank_, device_, allgather_ ? &B200Endpoint::gather_trampoline : nullptr, this, &comm_));
}

float* B200Endpoint::staging(std::uint32_t bucket, std::size_t n) {
  auto& p = staging_[{bucket, n}];
  if (!p) {
    DeviceScope ds(device_);
    float* q = nullptr;
    cuda_check(cudaMalloc(&q, std::max<std::size_t>(n, 4) * sizeof(float)), "cudaMalloc staging");
    p = q;
  }
  return static_cast<float*>(p);
}

B200Endpoint::~B200Endpoint() {
  {
    DeviceScope ds(device_);
    for (auto& kv : staging_) cudaFree(kv.second);
  }
  if (comm_) b2_comm_destroy(comm_);
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

int B200Endpoint::node_of(int r) const {
  if (r < 0 || r >= world_) throw Error(B2_ERR_INVALID, "unknown rank " + std::to_string(r));
  return 0;
}

void B200Endpoint::sync() { check(b2_comm_sync(comm_, stream_)); }

// --------------------------------------------------------------- primitives
double c_fp_s(B200Endpoint& ep, double now, std::span<float> x, std::uint32_t bucket) {
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  Staged b(ep, bucket, x, s);
  check(b2_c_fp_s(ep.handle(), b.dev, x.size(), bucket, s));
  ep.sync();  // throws on a latched device error before anything is written back
  b.finish(s);
  const int g = ep.world_size(), me = ep.rank();
  if (g > 1) {
    const std::size_t own = owned_partition_len(x.size(), g, me);
    ep.account(4 * (x.size() - own) + 4 * own * (g - 1), 2 * (g - 1));  // 2(n-1) messages, test_collectives.cpp:95
  }
  return now;
}

double c_lp_s(B200Endpoint& ep, double now, std::span<float> x, const Codec& codec, ErrorState* es,
              std::mt19937* rng, std::uint32_t bucket) {
  check_codec(codec, rng);
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  Staged b(ep, bucket, x, s);
  if (stochastic(codec))
    check(b2_c_lp_s_stochastic(ep.handle(), b.dev, x.size(), es ? es->delta() : nullptr, es ? es->delta_len() : 0,
                               es ? es->epsilon() : nullptr, es ? es->epsilon_len() : 0, draw_seed(rng), bucket, s));
  else
    check(b2_c_lp_s(ep.handle(), b.dev, x.size(), static_cast<int>(codec.kind), es ? es->delta() : nullptr,
                    es ? es->delta_len() : 0, es ? es->epsilon() : nullptr, es ? es->epsilon_len() : 0, bucket, s));
  ep.sync();  // throws on a latched device error before anything is written back
  b.finish(s);
  const int g = ep.world_size(), me = ep.rank();
  if (g > 1) {
    std::uint64_t sent = 0;
    for (int k = 0; k < g; ++k)
      if (k != me) sent += codec.payload_size(partition_range(x.size(), g, k).second);
    sent += (g - 1) * codec.payload_size(owned_partition_len(x.size(), g, me));
    ep.account(sent, 2 * (g - 1));
  }
  return now;
}

double hierarchical_c(B200Endpoint& ep, double now, std::span<float> x, const Codec& codec, ErrorState* es,
                      std::mt19937* rng, std::uint32_t bucket) {  // collectives.cpp:290-385, one NVLink node
  (void)codec;
  (void)es;
  (void)rng;
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  Staged b(ep, bucket, x, s);
  check(b2_hierarchical_c(ep.handle(), b.dev, x.size(), bucket, s));
  ep.sync();
  b.finish(s);
  return now;
}

namespace {
std::vector<int> nbrs_of(B200Endpoint& ep, const Topology& topo, std::uint64_t round) {
  if (topo.n != ep.world_size()) throw Error(B2_ERR_INVALID, "topology size mismatch");  // collectives.cpp:232
  return topo.neighbors(ep.rank(), round);
}
}  // namespace

double d_fp_s(B200Endpoint& ep, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              ReduceMode mode, std::uint32_t bucket) {
  const auto nb = nbrs_of(ep, topo, round);
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  Staged b(ep, bucket, x, s);
  check(b2_d_fp_s(ep.handle(), b.dev, x.size(), nb.data(), static_cast<int>(nb.size()), static_cast<int>(mode),
                  bucket, s));
  ep.sync();  // throws on a latched device error before anything is written back
  b.finish(s);
  ep.account((nb.size() - 1) * 4 * x.size(), nb.size() - 1);
  return now;
}

double d_lp_s(B200Endpoint& ep, double now, std::span<float> x, const Topology& topo, std::uint64_t round,
              const Codec& codec, ReduceMode mode, std::mt19937* rng, std::uint32_t bucket) {
  check_codec(codec, rng);
  const auto nb = nbrs_of(ep, topo, round);
  DeviceScope ds(ep.device());
  auto s = static_cast<cudaStream_t>(ep.stream());
  Staged b(ep, bucket, x, s);
  if (stochastic(codec))
    check(b2_d_lp_s_stochastic(ep.handle(), b.dev, x.size(), nb.data(), static_cast<int>(nb.size()),
                               static_cast<int>(mode), draw_seed(rng), bucket, s));
  else
    check(b2_d_lp_s(ep.handle(), b.dev, x.size(), nb.data(), static_cast<int>(nb.size()),
                    static_cast<int>(codec.kind), static_cast<int>(mode), bucket, s));
  ep.sync();  // throws on a latched device error before anything is written back
  b.finish(s);
  ep.account((nb.size() - 1) * codec.payload_size(x.size()), nb.size() - 1);
  return now;
}

// ------------------------------------------------------------------ tensors
namespace {
std::size_t shape_product(const std::vector<std::size_t>& shape) {  // tensor.cpp:9-17
  std::size_t p = 1;
  for (std::size_t d : shape) {
    if (d == 0) throw Error(B2_ERR_INVALID, "tensor shape has a zero dimension");
    p *= d;
  }
  return shape.empty() ? 0 : p;
}
std::shared_ptr<float> device_alloc(std::size_t n, int device) {
  DeviceScope ds(device);
  float* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<std::size_t>(n, 4) * sizeof(float)), "cudaMalloc tensor");
  return std::shared_ptr<float>(p, [](float* q) { cudaFree(q); });
}
}  // namespace

FlatTensor::FlatTensor(std::string name, std::vector<std::size_t> shape)
    : name_(std::move(name)), shape_(std::move(shape)) {
  if (name_.empty()) throw Error(B2_ERR_INVALID, "tensor name must be non-empty");
  len_ = capacity_ = shape_product(shape_);
  storage_ = device_alloc(len_, -1);
  cuda_check(cudaMemset(storage_.get(), 0, std::max<std::size_t>(len_, 4) * 4), "memset");
}

FlatTensor::FlatTensor(std::string name, std::vector<std::size_t> shape, const std::vector<float>& values,
                       int device)
    : name_(std::move(name)), shape_(std::move(shape)) {
  if (name_.empty()) throw Error(B2_ERR_INVALID, "tensor name must be non-empty");
  len_ = capacity_ = shape_product(shape_);
  if (values.size() != len_) throw Error(B2_ERR_INVALID, "tensor '" + name_ + "': shape/data length mismatch");
  storage_ = device_alloc(len_, device);
  if (len_) cuda_check(cudaMemcpy(storage_.get(), values.data(), 4 * len_, cudaMemcpyHostToDevice), "upload");
}

std::vector<float> FlatTensor::to_host() const { return b200::to_host({data(), len_}); }

FlatTensor BucketArena::as_flat(const std::string& name) const {
  FlatTensor t;
  t.name_ = name;
  t.shape_ = {len_};
  t.storage_ = storage_;
  t.offset_ = 0;
  t.len_ = t.capacity_ = len_;
  return t;
}

BucketArena BucketArena::flatten(std::span<FlatTensor*> tensors) {  // tensor.cpp:46-68
  if (tensors.empty()) throw Error(B2_ERR_INVALID, "flatten: empty tensor list");
  std::unordered_set<std::string> seen;
  std::size_t total = 0;
  for (FlatTensor* t : tensors) {
    if (t->size() == 0) throw Error(B2_ERR_INVALID, "flatten: zero-length tensor '" + t->name() + "'");
    if (!seen.insert(t->name()).second) throw Error(B2_ERR_INVALID, "flatten: duplicate tensor name '" + t->name() + "'");
    total += t->size();
  }
  int device = 0;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, tensors[0]->data()) == cudaSuccess) device = a.device;
  BucketArena arena;
  arena.storage_ = device_alloc(total, device);
  arena.len_ = total;
  std::vector<const float*> srcs;
  std::vector<std::size_t> lens;
  for (FlatTensor* t : tensors) {
    srcs.push_back(t->data());
    lens.push_back(t->size());
  }
  DeviceScope ds(device);
  check(b2_bucket_flatten(srcs.data(), lens.data(), static_cast<int>(srcs.size()), arena.storage_.get(), nullptr));
  cuda_check(cudaDeviceSynchronize(), "flatten sync");
  std::size_t off = 0;
  for (FlatTensor* t : tensors) {
    arena.members_.push_back({t->name(), off, t->size()});
    t->storage_ = arena.storage_;  // repoint: writes alias both ways (tensor.cpp:63-64)
    t->offset_ = off;
    t->capacity_ = total;
    off += t->size();
  }
  return arena;
}

}  // namespace rcomm::b200

// ------------------------------------------------------------------- engine
namespace rcomm::b200 {

std::vector<EngineBucket> plan_buckets(const std::vector<std::size_t>& layer_sizes, std::size_t capacity_bytes,
                                       bool fusion) {
  if (layer_sizes.empty()) throw Error(B2_ERR_INVALID, "engine: model has no parameter tensors");  // engine.cpp:40
  const std::size_t cap = fusion ? capacity_bytes : 0;
  std::vector<EngineBucket> out;
  std::size_t used = 0;
  const std::size_t L = layer_sizes.size();
  for (std::size_t i = 0; i < L; ++i) {  // engine.cpp:80-95
    const std::size_t l = L - 1 - i;
    const std::size_t bytes = 4 * layer_sizes[l];
    if (out.empty() || used + bytes > cap) {
      EngineBucket b;
      b.id = out.size();
      out.push_back(std::move(b));
      used = 0;
    }
    out.back().layers.push_back(l);
    out.back().trigger_layer = l;
    out.back().elements += layer_sizes[l];
    used += bytes;
  }
  return out;
}

OverlapEngine::OverlapEngine(B200Endpoint& ep, std::vector<std::size_t> layer_sizes, std::size_t capacity_bytes,
                             bool fusion, Primitive prim, std::uint32_t bucket_base)
    : ep_(ep), prim_(prim), base_(bucket_base), sizes_(std::move(layer_sizes)) {
  buckets_ = plan_buckets(sizes_, capacity_bytes, fusion);
  DeviceScope ds(ep_.device());
  bucket_of_.assign(sizes_.size(), 0);
  offset_.assign(sizes_.size(), 0);
  for (const auto& b : buckets_) {
    float* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<std::size_t>(b.elements, 4) * sizeof(float)), "cudaMalloc bucket arena");
    cuda_check(cudaMemset(p, 0, b.elements * sizeof(float)), "cudaMemset bucket arena");
    arenas_.push_back(p);
    std::size_t off = 0;
    for (std::size_t l : b.layers) {
      bucket_of_[l] = b.id;
      offset_[l] = off;
      off += sizes_[l];
    }
  }
  int lo = 0, hi = 0;  // highest priority: freed SMs go to the communication CTAs first
  cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
  cudaStream_t s;
  cuda_check(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi), "cudaStreamCreate comm");
  comm_ = s;
  cudaEvent_t ev;
  cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  done_ = ev;
}

OverlapEngine::~OverlapEngine() {
  DeviceScope ds(ep_.device());
  if (comm_) {
    cudaStreamSynchronize(static_cast<cudaStream_t>(comm_));
    cudaStreamDestroy(static_cast<cudaStream_t>(comm_));
  }
  if (done_) cudaEventDestroy(static_cast<cudaEvent_t>(done_));
  for (float* p : arenas_) cudaFree(p);
}

float* OverlapEngine::grad(std::size_t layer) { return arenas_.at(bucket_of_.at(layer)) + offset_[layer]; }

std::span<float> OverlapEngine::arena(std::size_t bucket) {
  return {arenas_.at(bucket), buckets_.at(bucket).elements};
}

void OverlapEngine::layer_done(std::size_t layer, void* compute_stream) {
  const EngineBucket& b = buckets_.at(bucket_of_.at(layer));
  if (layer != b.trigger_layer) return;
  DeviceScope ds(ep_.device());
  cudaEvent_t ev;
  cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventRecord(ev, static_cast<cudaStream_t>(compute_stream)), "cudaEventRecord");
  auto cs = static_cast<cudaStream_t>(comm_);
  cuda_check(cudaStreamWaitEvent(cs, ev, 0), "cudaStreamWaitEvent");
  cudaEventDestroy(ev);  // released once the wait is satisfied
  const std::uint32_t bucket = base_ + static_cast<std::uint32_t>(b.id);
  if (prim_ == Primitive::c_lp_s)
    check(b2_c_lp_s(ep_.handle(), arenas_[b.id], b.elements, B2_CODEC_UNIFORM8, nullptr, 0, nullptr, 0, bucket, cs));
  else
    check(b2_c_fp_s(ep_.handle(), arenas_[b.id], b.elements, bucket, cs));
  ++pending_;
}

void OverlapEngine::finish(void* compute_stream) {
  if (pending_ != buckets_.size())
    throw Error(B2_ERR_INVALID, "engine: " + std::to_string(pending_) + " of " + std::to_string(buckets_.size()) +
                                    " buckets issued this iteration");
  DeviceScope ds(ep_.device());
  auto done = static_cast<cudaEvent_t>(done_);
  // the previous iteration's buckets, once complete, report their errors
  if (issued_ && cudaEventQuery(done) == cudaSuccess) check(b2_comm_poll(ep_.handle()));
  cudaGetLastError();  // cudaErrorNotReady from the query is not an error
  cuda_check(cudaEventRecord(done, static_cast<cudaStream_t>(comm_)), "cudaEventRecord");
  cuda_check(cudaStreamWaitEvent(static_cast<cudaStream_t>(compute_stream), done, 0), "cudaStreamWaitEvent");
  issued_ = true;
  pending_ = 0;
}

void OverlapEngine::synchronize() {
  DeviceScope ds(ep_.device());
  cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(comm_)), "cudaStreamSynchronize comm");
  check(b2_comm_poll(ep_.handle()));
}

}  // namespace rcomm::b200
