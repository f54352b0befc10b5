// comm.cu -- communicator, peer windows and the C-ABI entry points of the
// primitives (include/b2comm.h).
//
// The reference's Endpoint moves opaque byte messages between workers
// (transport.hpp:52-85; sim_transport.cpp:29-69, where send() copies the
// payload into the peer's mailbox).  Here the "mailbox" is a window of
// device memory that every peer maps: one cudaMalloc per (bucket, family,
// size) whose CUDA IPC handle (or raw pointer, for ranks living in the same
// process) is exchanged once through the caller's allgather.  Kernels then
// store into / load from peer windows directly over NVLink/NVSwitch; the
// (src, tag) FIFO matching of the reference becomes epoch-tagged counters in
// each window's header (collectives.cuh: WinHdr).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <numeric>
#include <random>
#include <tuple>
#include <vector>

#include "b2_host.h"
#include "collectives.cuh"

namespace b2 {
int launch_central(const CentralArgs& a, int codec, bool ec, cudaStream_t s, int sms);
int launch_decent(const DecentArgs& a, int codec, cudaStream_t s, int sms);
int launch_decent_small(const DecentArgs& a, int codec, cudaStream_t s, int sms);
int launch_central_stag(const CentralArgs& a, bool ec, cudaStream_t s, int sms);
int launch_central_small(const CentralArgs& a, int codec, bool ec, cudaStream_t s, int sms);
int max_persistent_grid();
int launch_onebit_central(const OnebitArgs& a, bool ec, cudaStream_t s, int sms);
int launch_onebit_decent(const OnebitDecentArgs& a, cudaStream_t s, int sms);
size_t onebit_slot_bytes(size_t maxchunk);
}  // namespace b2

using namespace b2;

namespace {

enum Family { kCentral = 0, kDecentral = 1, kOnebit = 2, kOnebitD = 3 };

struct Window {
  size_t bytes = 0;
  uint8_t* local = nullptr;
  uint8_t* peer[kMaxRanks] = {};
  bool ipc_opened[kMaxRanks] = {};
  size_t off_gate = 0, gate_stride = 0, off_recv1 = 0, slot_stride = 0, off_out2 = 0, off_dbuf[2] = {0, 0};
  size_t off_sgate = 0, sgate_stride = 0, off_qgate = 0, off_land = 0;  // central_stag.cu
  size_t off_cgate = 0, off_cgate2 = 0;  // small_central.cu: [g][kSmallMaxGridD] each, or 0
  unsigned long long epoch = 0;
  unsigned long long small_calls = 0;    // small_central.cu launches (its counters' target)
  unsigned long long exp_reads[2] = {0, 0};
  unsigned long long sends_from[kMaxRanks] = {};  // D_*: calls (|N| > 1) in which rank j sent to me
  float2* partials = nullptr;
  unsigned* cta_done = nullptr;
  unsigned long long* sched = nullptr;  // [kSchedPasses] tile counters + end counter
  Fail* fail = nullptr;                 // device: status word + every rank's poison word
};

struct Blob {  // what each rank publishes about one window
  int ok;   // 0: this rank's allocation failed -- every rank fails the window together
  int pid;
  int device;
  int grid;  // persistent grid size: per-CTA arrival counts must agree across ranks
  unsigned long long ptr;
  unsigned long long bytes;
  cudaIpcMemHandle_t handle;
};

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct b2_comm {
  int world = 1, rank = 0, device = 0;
  b2_allgather_fn allgather = nullptr;
  void* user = nullptr;
  std::map<std::tuple<uint32_t, int, size_t, int>, Window*> wins;
  int* status_h = nullptr;  // mapped pinned host word
  int* status_d = nullptr;
  unsigned long long timeout_ns = 600000ull * 1000000ull;  // 10 min; tests and benches set their own
  bool poisoned = false;  // a rendezvous timed out: every further launch is refused
  int sm_budget = 0;      // SMs per primitive launch (0: all); identical on every rank
  unsigned long long launches = 0;
  unsigned long long* trace = nullptr;  // device [max grid * kTraceSlots], when enabled
  int trace_grid = 0;
  cudaStream_t aux = nullptr;      // non-blocking: poison reads while kernels run
  unsigned long long* poison_h = nullptr;  // pinned landing word of those reads
  std::mutex mu;
};

namespace {

struct DeviceGuard {  // make the communicator's GPU current for this call
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void free_window(b2_comm* c, Window* w) {
  for (int j = 0; j < kMaxRanks; ++j)
    if (w->ipc_opened[j]) cudaIpcCloseMemHandle(w->peer[j]);
  if (w->local) cudaFree(w->local);
  if (w->partials) cudaFree(w->partials);
  if (w->cta_done) cudaFree(w->cta_done);
  if (w->sched) cudaFree(w->sched);
  if (w->fail) cudaFree(w->fail);
  delete w;
  (void)c;
}

// Collective: every rank calls with identical (bucket, family, n, elem).
int get_window(b2_comm* c, uint32_t bucket, int family, size_t n, int elem, Window** out) {
  const auto key = std::make_tuple(bucket, family, n, elem);
  auto it = c->wins.find(key);
  if (it != c->wins.end()) {
    *out = it->second;
    return B2_OK;
  }
  const int g = c->world;
  Window* w = new Window();
  size_t off = 256;  // WinHdr
  if (family == kCentral) {
    const size_t maxchunk = (n + g - 1) / g;
    const size_t nreg = maxchunk / (16 * kGateUnits) + 2;
    // uint8 phase-1 region counters of my chunk (PassDesc::gate)
    w->off_gate = off;
    off += round_up(sizeof(unsigned long long) * nreg, 256);
    // staggered path: per-source region counters, out2 publication counters
    w->sgate_stride = nreg;
    w->off_sgate = off;
    off += round_up(sizeof(unsigned long long) * nreg * size_t(g), 256);
    w->off_qgate = off;
    off += round_up(sizeof(unsigned long long) * nreg, 256);
    if (n <= kSmallCentralWin && g > 1) {  // small_central.cu: per-CTA counters
      w->off_cgate = off;
      off += round_up(sizeof(unsigned long long) * kSmallMaxGridD * size_t(g), 256);
      w->off_cgate2 = off;
      off += round_up(sizeof(unsigned long long) * kSmallMaxGridD * size_t(g), 256);
    }
    // chunk k sits at slot offset e - (lo_k & ~15): up to 15 elements of head room
    w->slot_stride = round_up(size_t(elem) * (maxchunk + 16), 256);
    w->off_recv1 = off;
    off += size_t(g) * w->slot_stride;
    w->off_out2 = off;
    off += w->slot_stride;
    if (elem == 1 && g > 1) {  // uint8: landing slots of the staggered path
      w->off_land = off;
      off += size_t(g) * w->slot_stride;
    }
  } else if (family == kOnebit) {
    // slot j = rank j's onebit payload of my chunk; out2 = my phase-2 payload
    w->slot_stride = onebit_slot_bytes((n + g - 1) / g);
    w->off_recv1 = off;
    off += size_t(g) * w->slot_stride;
    w->off_out2 = off;
    off += w->slot_stride;
  } else if (family == kOnebitD) {
    // my bucket's onebit payload, double-buffered by call parity
    const size_t b = onebit_slot_bytes(n);
    w->off_dbuf[0] = off;
    off += b;
    w->off_dbuf[1] = off;
    off += b;
  } else {
    // arrival counters: for every source rank one per region of the bucket
    // (+ one for the unaligned tail), cumulative over the calls in which that
    // rank was my neighbour (the relation is symmetric, so I know how many)
    const size_t nreg = n / (16 * kGateUnits) + 1;
    // counters per source: the ring kernel's regions + tail, or the small
    // kernel's one per CTA (small_coll.cu)
    w->gate_stride = std::max(nreg + 1, kSmallMaxGridD + 1);
    w->off_gate = off;
    off += round_up(sizeof(unsigned long long) * w->gate_stride * size_t(g), 256);
    const size_t b = round_up(size_t(elem) * (n + 8), 256);
    w->off_dbuf[0] = off;
    off += b;
    w->off_dbuf[1] = off;
    off += b;
  }
  w->bytes = off;
  auto fail = [&](int rc) {
    free_window(c, w);
    return rc;
  };
  const bool ok =
      cudaMalloc(&w->local, w->bytes) == cudaSuccess &&
      cudaMemset(w->local, 0, (family == kDecentral || family == kOnebitD) ? w->off_dbuf[0] : w->off_recv1) ==
          cudaSuccess &&
      cudaMalloc(&w->partials, sizeof(float2) * (kMaxRanks + 1) *
                                   std::max<size_t>(max_persistent_grid(), kSmallMaxGridD)) == cudaSuccess &&
      cudaMalloc(&w->cta_done, sizeof(unsigned) * (kMaxRanks + 4)) == cudaSuccess &&
      cudaMemset(w->cta_done, 0, sizeof(unsigned) * (kMaxRanks + 4)) == cudaSuccess &&
      cudaMalloc(&w->sched, sizeof(unsigned long long) * (kSchedPasses + 1)) == cudaSuccess &&
      cudaMemset(w->sched, 0, sizeof(unsigned long long) * (kSchedPasses + 1)) == cudaSuccess &&
      cudaMalloc(&w->fail, sizeof(Fail)) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  std::string why;
  if (!ok) why = cudaGetErrorString(cudaGetLastError());
  w->peer[c->rank] = w->local;
  if (g > 1) {
    // every rank takes part in the exchange even when its allocation failed,
    // so that all ranks fail together instead of the others blocking here
    Blob mine{};
    mine.ok = ok ? 1 : 0;
    mine.pid = static_cast<int>(getpid());
    mine.device = c->device;
    mine.grid = c->sm_budget > 0 && c->sm_budget < sm_count() ? c->sm_budget : sm_count();
    mine.ptr = reinterpret_cast<unsigned long long>(w->local);
    mine.bytes = w->bytes;
    if (ok && cudaIpcGetMemHandle(&mine.handle, w->local) != cudaSuccess) {
      mine.ok = 0;
      why = cudaGetErrorString(cudaGetLastError());
    }
    std::vector<Blob> all(g);
    if (!c->allgather || c->allgather(c->user, &mine, sizeof(Blob), all.data()) != 0) {
      set_error("bootstrap allgather failed for bucket %u", bucket);
      return fail(B2_ERR_BOOTSTRAP);
    }
    for (int j = 0; j < g; ++j)
      if (!all[j].ok) {
        set_error("window allocation of %zu bytes failed on rank %d%s%s", w->bytes, j, j == c->rank ? ": " : "",
                  j == c->rank ? why.c_str() : "");
        return fail(B2_ERR_CUDA);
      }
    for (int j = 0; j < g; ++j) {
      if (all[j].bytes != w->bytes) {
        set_error("rank %d window size %llu != %zu: mismatched collective arguments", j,
                  all[j].bytes, w->bytes);
        return fail(B2_ERR_INVALID);
      }
      if (all[j].grid != mine.grid) {
        set_error("rank %d launches on %d SMs, rank %d on %d: the SM count and b2_comm_set_sm_budget must agree", j,
                  all[j].grid, c->rank, mine.grid);
        return fail(B2_ERR_INVALID);
      }
      if (j == c->rank) continue;
      if (all[j].pid == mine.pid) {  // same process: plain peer access
        if (all[j].device != c->device) {
          cudaError_t e = cudaDeviceEnablePeerAccess(all[j].device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            set_error("peer access %d->%d: %s", c->device, all[j].device, cudaGetErrorString(e));
            return fail(B2_ERR_CUDA);
          }
          cudaGetLastError();
        }
        w->peer[j] = reinterpret_cast<uint8_t*>(all[j].ptr);
      } else {
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, all[j].handle, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          set_error("cudaIpcOpenMemHandle(rank %d): %s", j, cudaGetErrorString(e));
          return fail(B2_ERR_CUDA);
        }
        w->peer[j] = static_cast<uint8_t*>(p);
        w->ipc_opened[j] = true;
      }
    }
  } else if (!ok) {
    set_error("window allocation of %zu bytes failed: %s", w->bytes, why.c_str());
    return fail(B2_ERR_CUDA);
  }
  Fail f{};
  f.host = c->status_d;
  f.n = g;
  for (int j = 0; j < g; ++j)
    f.peer[j] = reinterpret_cast<unsigned long long*>(w->peer[j] + offsetof(WinHdr, poison));
  f.mine = f.peer[c->rank];
  if (cudaMemcpy(w->fail, &f, sizeof(Fail), cudaMemcpyHostToDevice) != cudaSuccess) {
    set_error("window init failed: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(B2_ERR_CUDA);
  }
  c->wins[key] = w;
  *out = w;
  return B2_OK;
}

// A communicator whose device latched a rendezvous timeout is poisoned: the
// windows' epochs no longer agree across ranks, so every further launch is
// refused until the communicator is destroyed and re-created.
int refuse_if_poisoned(b2_comm* c) {
  if (!c->poisoned && (__atomic_load_n(c->status_h, __ATOMIC_ACQUIRE) & kStatusTimeout)) c->poisoned = true;
  if (c->poisoned) {
    set_error("communicator poisoned by an earlier rendezvous timeout: destroy and re-create it");
    return B2_ERR_TIMEOUT;
  }
  return B2_OK;
}

int check_comm(b2_comm* c, const float* x, size_t n) {
  B2_REQUIRE(c, "null communicator");
  B2_REQUIRE(n == 0 || x, "null bucket pointer");
  B2_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, "bucket must be 16-byte aligned");
  return B2_OK;
}

}  // namespace

extern "C" {

int b2_version(void) { return B2COMM_VERSION; }

const char* b2_status_string(int s) {
  switch (s) {
    case B2_OK: return "ok";
    case B2_ERR_INVALID: return "invalid argument";
    case B2_ERR_CUDA: return "cuda error";
    case B2_ERR_NONFINITE: return "encode: non-finite input value";
    case B2_ERR_TIMEOUT: return "rendezvous timeout";
    case B2_ERR_UNSUPPORTED: return "unsupported";
    case B2_ERR_BOOTSTRAP: return "bootstrap failure";
  }
  return "unknown";
}

void b2_partition_range(size_t len, int n, int k, size_t* lo, size_t* sz) {
  const size_t base = len / size_t(n), extra = len % size_t(n), uk = size_t(k);
  *lo = uk * base + std::min(uk, extra);
  *sz = base + (uk < extra ? 1 : 0);
}

size_t b2_owned_partition_len(size_t len, int world, int idx) {
  size_t lo, sz;
  b2_partition_range(len, world, idx, &lo, &sz);
  return sz;
}

size_t b2_payload_size(int codec, size_t n) {  // codec.cpp:31-38
  switch (codec) {
    case B2_CODEC_IDENTITY: return 4 * n;
    case B2_CODEC_UNIFORM8: return 8 + n;
    case B2_CODEC_ONEBIT: return 4 + (n + 7) / 8;
  }
  return 0;
}

// Topology::neighbors, collectives.cpp:181-213 -- the random matching uses
// the same mt19937_64 seed mix and std::shuffle, so every rank (and the
// reference) agrees on it.
int b2_topology_neighbors(int kind, int n, uint64_t seed, int rank, uint64_t round, int* out) {
  if (rank < 0 || rank >= n || !out) {
    set_error("topology: rank out of range");
    return -1;
  }
  std::vector<int> nb;
  if (kind == B2_TOPO_FULL) {
    nb.resize(size_t(n));
    std::iota(nb.begin(), nb.end(), 0);
  } else if (kind == B2_TOPO_RING) {
    nb = {(rank + n - 1) % n, rank, (rank + 1) % n};
    std::sort(nb.begin(), nb.end());
    nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
  } else if (kind == B2_TOPO_RANDOM) {
    std::mt19937_64 rng(seed ^ (0x9e3779b97f4a7c15ULL * (round + 1)));
    std::vector<int> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    int peer = rank;
    for (int i = 0; i + 1 < n; i += 2) {
      if (perm[i] == rank) peer = perm[i + 1];
      if (perm[i + 1] == rank) peer = perm[i];
    }
    nb = {rank};
    if (peer != rank) nb.push_back(peer);
    std::sort(nb.begin(), nb.end());
  } else {
    set_error("topology: unknown kind");
    return -1;
  }
  std::copy(nb.begin(), nb.end(), out);
  return static_cast<int>(nb.size());
}

int b2_comm_create(int world, int rank, int device, b2_allgather_fn allgather, void* user,
                   b2_comm_t* out) {
  B2_REQUIRE(out, "null output handle");
  B2_REQUIRE(world >= 1 && world <= B2_MAX_RANKS, "world size %d outside [1, %d]", world,
             B2_MAX_RANKS);
  B2_REQUIRE(rank >= 0 && rank < world, "rank %d outside [0, %d)", rank, world);
  B2_REQUIRE(world == 1 || allgather, "world > 1 needs an allgather bootstrap");
  DeviceGuard dg(device);
  int coop = 0;
  B2_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  B2_REQUIRE(coop, "device %d does not support cooperative launch", device);
  b2_comm* c = new b2_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->allgather = allgather;
  c->user = user;
  if (cudaHostAlloc(&c->status_h, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&c->status_d, c->status_h, 0) != cudaSuccess) {
    set_error("status word allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
    delete c;
    return B2_ERR_CUDA;
  }
  *c->status_h = 0;
  *out = c;
  return B2_OK;
}

int b2_comm_destroy(b2_comm_t c) {
  if (!c) return B2_OK;
  DeviceGuard dg(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->wins) free_window(c, kv.second);
  if (c->trace) cudaFree(c->trace);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->poison_h) cudaFreeHost(c->poison_h);
  if (c->status_h) cudaFreeHost(c->status_h);
  delete c;
  return B2_OK;
}

int b2_comm_enable_trace(b2_comm_t c, int on) {
  B2_REQUIRE(c, "null communicator");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if (on && !c->trace) {
    c->trace_grid = std::max(max_persistent_grid(), int(kSmallMaxGridD));  // small_coll.cu grids reach 1024
    B2_CUDA_TRY(cudaMalloc(&c->trace, sizeof(unsigned long long) * kTraceSlots * c->trace_grid));
    B2_CUDA_TRY(cudaMemset(c->trace, 0, sizeof(unsigned long long) * kTraceSlots * c->trace_grid));
  } else if (!on && c->trace) {
    cudaFree(c->trace);
    c->trace = nullptr;
  }
  return B2_OK;
}

int b2_comm_read_trace(b2_comm_t c, uint64_t* out, int max_ctas, int* n_slots) {
  B2_REQUIRE(c && out && n_slots, "null argument");
  B2_REQUIRE(c->trace, "tracing is not enabled");
  DeviceGuard dg(c->device);
  const int n = std::min(max_ctas, c->trace_grid);
  B2_CUDA_TRY(cudaMemcpy(out, c->trace, sizeof(uint64_t) * kTraceSlots * n, cudaMemcpyDeviceToHost));
  *n_slots = kTraceSlots;
  return B2_OK;
}

int b2_comm_set_sm_budget(b2_comm_t c, int sms) {
  B2_REQUIRE(c, "null communicator");
  B2_REQUIRE(sms >= 0, "SM budget %d is negative", sms);
  DeviceGuard dg(c->device);
  std::lock_guard<std::mutex> lk(c->mu);
  c->sm_budget = sms >= sm_count() ? 0 : sms;
  return B2_OK;
}

// A peer that timed out writes the poison word of every rank's window
// (b2_device.cuh latch); a rank whose own calls never waited for the late
// rank (a D_* rank outside its neighbourhood) has not run a kernel that saw
// it, so the windows' poison words are read here too (a copy on a
// non-blocking stream: it does not wait for kernels still spinning).
int b2_comm_poisoned(b2_comm_t c) {
  if (!c) return 0;
  std::lock_guard<std::mutex> lk(c->mu);
  if (__atomic_load_n(c->status_h, __ATOMIC_ACQUIRE) & kStatusTimeout) c->poisoned = true;
  if (!c->poisoned && !c->wins.empty()) {
    DeviceGuard dg(c->device);
    if (!c->aux && cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess) c->aux = nullptr;
    if (!c->poison_h && cudaHostAlloc(reinterpret_cast<void**>(&c->poison_h), sizeof(unsigned long long),
                                      cudaHostAllocDefault) != cudaSuccess)
      c->poison_h = nullptr;
    if (c->aux && c->poison_h) {
      for (auto& kv : c->wins) {
        *c->poison_h = 0;
        if (cudaMemcpyAsync(c->poison_h, kv.second->local + offsetof(WinHdr, poison), sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, c->aux) != cudaSuccess ||
            cudaStreamSynchronize(c->aux) != cudaSuccess)
          break;
        if (*c->poison_h) {
          c->poisoned = true;
          break;
        }
      }
    }
  }
  return c->poisoned ? 1 : 0;
}

// Collective (every rank, same bucket): free the bucket's windows once no
// rank's kernels can still touch them -- each rank drains its device, then a
// barrier through the bootstrap allgather, then IPC mappings are closed and
// the memory freed.
int b2_comm_release_bucket(b2_comm_t c, uint32_t bucket) {
  B2_REQUIRE(c, "null communicator");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  B2_CUDA_TRY(cudaDeviceSynchronize());
  if (c->world > 1) {
    std::vector<int> all(c->world);
    int mine = 1;
    if (!c->allgather || c->allgather(c->user, &mine, sizeof(int), all.data()) != 0) {
      set_error("bootstrap allgather failed while releasing bucket %u", bucket);
      return B2_ERR_BOOTSTRAP;
    }
  }
  for (auto it = c->wins.begin(); it != c->wins.end();) {
    if (std::get<0>(it->first) == bucket) {
      free_window(c, it->second);
      it = c->wins.erase(it);
    } else {
      ++it;
    }
  }
  return B2_OK;
}

size_t b2_comm_window_bytes(b2_comm_t c) {
  if (!c) return 0;
  std::lock_guard<std::mutex> lk(c->mu);
  size_t b = 0;
  for (auto& kv : c->wins) b += kv.second->bytes;
  return b;
}

int b2_comm_rank(b2_comm_t c) { return c ? c->rank : -1; }
int b2_comm_world(b2_comm_t c) { return c ? c->world : -1; }
uint64_t b2_comm_launches(b2_comm_t c) { return c ? c->launches : 0; }

int b2_comm_set_timeout_ms(b2_comm_t c, uint64_t ms) {
  B2_REQUIRE(c, "null communicator");
  c->timeout_ns = static_cast<unsigned long long>(ms) * 1000000ull;
  return B2_OK;
}

int b2_comm_poll(b2_comm_t c) {
  B2_REQUIRE(c, "null communicator");
  const int s = __atomic_exchange_n(c->status_h, 0, __ATOMIC_SEQ_CST);
  if ((s & kStatusTimeout) || c->poisoned) {  // sticky: see refuse_if_poisoned
    c->poisoned = true;
    set_error("rendezvous timeout: a peer did not arrive (the communicator is poisoned)");
    return B2_ERR_TIMEOUT;
  }
  if (s & kStatusNonFinite) {
    set_error("encode: non-finite input value");
    return B2_ERR_NONFINITE;
  }
  return B2_OK;
}

int b2_comm_sync(b2_comm_t c, void* stream) {
  B2_REQUIRE(c, "null communicator");
  DeviceGuard dg(c->device);
  B2_CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return b2_comm_poll(c);
}

// The world size that takes the staggered C_LP_S (default 2; B2_STAG=0
// disables it, B2_STAG=<g> selects another world size for A/B measurements)
static int stag_world() {
  static const int v = [] {
    const char* e = getenv("B2_STAG");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}

// B2_STATIC_SCHED=1: static round-robin tile assignment (A/B measurements)
static bool static_sched() {
  static const bool v = [] {
    const char* e = getenv("B2_STATIC_SCHED");
    return e && e[0] == '1';
  }();
  return v;
}

static int central(b2_comm_t c, float* x, size_t n, int codec, int check_finite, float* delta,
                   size_t delta_len, float* eps, size_t eps_len, uint32_t bucket, void* stream, int sr_on = 0,
                   uint64_t sr_seed = 0) {
  int rc = check_comm(c, x, n);
  if (rc) return rc;
  B2_REQUIRE((delta == nullptr) == (eps == nullptr), "delta and eps must both be set or both null");
  const size_t own = b2_owned_partition_len(n, c->world, c->rank);
  if (delta) {  // collectives.cpp:102-107
    B2_REQUIRE(delta_len == n, "c_lp_s: delta length does not match bucket length");
    B2_REQUIRE(eps_len == own, "c_lp_s: epsilon length does not match owned partition");
    B2_REQUIRE((reinterpret_cast<uintptr_t>(delta) & 15) == 0, "delta must be 16-byte aligned");
  }
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if ((rc = refuse_if_poisoned(c))) return rc;
  Window* w = nullptr;
  rc = get_window(c, bucket, kCentral, n, codec == B2_CODEC_UNIFORM8 ? 1 : 4, &w);
  if (rc) return rc;
  CentralArgs a{};
  a.x = x;
  a.n = n;
  a.g = c->world;
  a.me = c->rank;
  a.check_finite = check_finite;
  a.delta = delta;
  a.eps = eps;
  for (int j = 0; j < c->world; ++j) a.win[j] = w->peer[j];
  a.off_gate = w->off_gate;
  a.off_recv1 = w->off_recv1;
  a.slot_stride = w->slot_stride;
  a.off_out2 = w->off_out2;
  a.off_sgate = w->off_sgate;
  a.sgate_stride = w->sgate_stride;
  a.off_qgate = w->off_qgate;
  a.off_land = w->off_land;
  a.partials = w->partials;
  a.cta_done = w->cta_done;
  a.gridbar = w->cta_done + kMaxRanks + 2;
  a.sched = static_sched() ? nullptr : w->sched;
  a.sched_end = reinterpret_cast<unsigned*>(w->sched + kSchedPasses);
  a.status = w->fail;
  a.timeout_ns = c->timeout_ns;
  a.trace = c->trace;
  a.sr_on = sr_on;
  a.sr_seed = sr_seed;
  // small buckets: the register-resident kernel (small_central.cu), with its
  // own call counter and counter arrays
  rc = B2_ERR_UNSUPPORTED;
  if (w->off_cgate) {
    CentralArgs sa = a;
    sa.epoch = w->small_calls + 1;
    sa.off_sgate = w->off_cgate;
    sa.off_sgate2 = w->off_cgate2;
    sa.sgate_stride = kSmallMaxGridD;
    rc = launch_central_small(sa, codec == B2_CODEC_UNIFORM8 ? kU8 : kIdentity, delta != nullptr,
                              static_cast<cudaStream_t>(stream), c->sm_budget);
    if (rc == B2_OK) {
      ++w->small_calls;
      ++c->launches;
      return rc;
    }
    if (rc != B2_ERR_UNSUPPORTED) return rc;
  }
  a.epoch = ++w->epoch;
  // uint8 at g == 2 with 16-aligned equal chunks: the staggered schedule
  // (central_stag.cu; measured faster at g = 2 only); every
  // rank decides identically from (n, g)
  if (codec == B2_CODEC_UNIFORM8 && c->world == stag_world() && n % (16 * size_t(c->world)) == 0 &&
      (!eps || (reinterpret_cast<uintptr_t>(eps) & 15) == 0))
    rc = launch_central_stag(a, delta != nullptr, static_cast<cudaStream_t>(stream), c->sm_budget);
  else
    rc = launch_central(a, codec == B2_CODEC_UNIFORM8 ? kU8 : kIdentity, delta != nullptr,
                        static_cast<cudaStream_t>(stream), c->sm_budget);
  if (rc == B2_OK) ++c->launches;
  return rc;
}

// c_lp_s with Codec{onebit} (the 1-bit Adam aggregation, algorithms.cpp:141-148)
static int onebit_central(b2_comm_t c, float* x, size_t n, float* delta, size_t delta_len, float* eps,
                          size_t eps_len, uint32_t bucket, void* stream) {
  int rc = check_comm(c, x, n);
  if (rc) return rc;
  B2_REQUIRE((delta == nullptr) == (eps == nullptr), "delta and eps must both be set or both null");
  const size_t own = b2_owned_partition_len(n, c->world, c->rank);
  if (delta) {  // collectives.cpp:102-107
    B2_REQUIRE(delta_len == n, "c_lp_s: delta length does not match bucket length");
    B2_REQUIRE(eps_len == own, "c_lp_s: epsilon length does not match owned partition");
    B2_REQUIRE((reinterpret_cast<uintptr_t>(delta) & 15) == 0 && (reinterpret_cast<uintptr_t>(eps) & 15) == 0,
               "delta and epsilon must be 16-byte aligned");
  }
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if ((rc = refuse_if_poisoned(c))) return rc;
  Window* w = nullptr;
  rc = get_window(c, bucket, kOnebit, n, 1, &w);
  if (rc) return rc;
  OnebitArgs a{};
  a.x = x;
  a.n = n;
  a.g = c->world;
  a.me = c->rank;
  a.epoch = ++w->epoch;
  a.delta = delta;
  a.eps = eps;
  for (int j = 0; j < c->world; ++j) a.win[j] = w->peer[j];
  a.off_recv1 = w->off_recv1;
  a.slot_stride = w->slot_stride;
  a.off_out2 = w->off_out2;
  a.partials = reinterpret_cast<double*>(w->partials);
  a.status = w->fail;
  a.timeout_ns = c->timeout_ns;
  rc = launch_onebit_central(a, delta != nullptr, static_cast<cudaStream_t>(stream), c->sm_budget);
  if (rc == B2_OK) ++c->launches;
  return rc;
}

int b2_c_fp_s(b2_comm_t c, float* x, size_t n, uint32_t bucket, void* stream) {
  int rc = check_comm(c, x, n);
  if (rc) return rc;
  if (c->world == 1) return B2_OK;  // collectives.cpp:49: x untouched
  return central(c, x, n, B2_CODEC_IDENTITY, 0, nullptr, 0, nullptr, 0, bucket, stream);
}

int b2_c_lp_s(b2_comm_t c, float* x, size_t n, int codec, float* delta, size_t delta_len,
              float* eps, size_t eps_len, uint32_t bucket, void* stream) {
  if (codec == B2_CODEC_ONEBIT) return onebit_central(c, x, n, delta, delta_len, eps, eps_len, bucket, stream);
  B2_REQUIRE(codec == B2_CODEC_UNIFORM8 || codec == B2_CODEC_IDENTITY, "unknown codec %d", codec);
  return central(c, x, n, codec, 1, delta, delta_len, eps, eps_len, bucket, stream);
}

static int decentral(b2_comm_t c, float* x, size_t n, const int* nbrs, int n_nbrs, int codec,
                     int check_finite, int mode, uint32_t bucket, void* stream, int sr_on = 0,
                     uint64_t sr_seed = 0) {
  int rc = check_comm(c, x, n);
  if (rc) return rc;
  B2_REQUIRE(nbrs && n_nbrs >= 1 && n_nbrs <= c->world, "neighbour list of size %d invalid", n_nbrs);
  B2_REQUIRE(mode == B2_REDUCE_SUM || mode == B2_REDUCE_AVERAGE, "unknown reduce mode %d", mode);
  bool has_self = false;
  for (int i = 0; i < n_nbrs; ++i) {
    B2_REQUIRE(nbrs[i] >= 0 && nbrs[i] < c->world, "neighbour %d out of range", nbrs[i]);
    B2_REQUIRE(i == 0 || nbrs[i] > nbrs[i - 1], "neighbour list must be sorted and unique");
    has_self |= nbrs[i] == c->rank;
  }
  B2_REQUIRE(has_self, "neighbour list must include the calling rank");
  std::lock_guard<std::mutex> lk(c->mu);
  DeviceGuard dg(c->device);
  if ((rc = refuse_if_poisoned(c))) return rc;
  Window* w = nullptr;
  if (codec == B2_CODEC_ONEBIT) {  // d_lp_s with Codec{onebit}: pull design, onebit_coll.cu
    rc = get_window(c, bucket, kOnebitD, n, 1, &w);
    if (rc) return rc;
    OnebitDecentArgs a{};
    a.x = x;
    a.n = n;
    a.me = c->rank;
    a.nnb = n_nbrs;
    for (int i = 0; i < n_nbrs; ++i) a.nbrs[i] = nbrs[i];
    a.epoch = ++w->epoch;
    a.parity = static_cast<int>(a.epoch & 1);
    a.expected_reads = w->exp_reads[a.parity];
    a.inv = mode == B2_REDUCE_AVERAGE ? 1.0 / static_cast<double>(n_nbrs) : 1.0;
    for (int j = 0; j < c->world; ++j) a.win[j] = w->peer[j];
    a.off_dbuf = w->off_dbuf[a.parity];
    a.partials = reinterpret_cast<double*>(w->partials);
    a.status = w->fail;
    a.timeout_ns = c->timeout_ns;
    rc = launch_onebit_decent(a, static_cast<cudaStream_t>(stream), c->sm_budget);
    if (rc == B2_OK) {
      w->exp_reads[a.parity] += static_cast<unsigned long long>(n_nbrs - 1);  // symmetric: my readers
      ++c->launches;
    }
    return rc;
  }
  rc = get_window(c, bucket, kDecentral, n, codec == B2_CODEC_UNIFORM8 ? 1 : 4, &w);
  if (rc) return rc;
  DecentArgs a{};
  a.x = x;
  a.n = n;
  a.me = c->rank;
  a.nnb = n_nbrs;
  for (int i = 0; i < n_nbrs; ++i) a.nbrs[i] = nbrs[i];
  a.check_finite = check_finite;
  a.epoch = ++w->epoch;
  a.parity = static_cast<int>(a.epoch & 1);
  a.expected_reads = w->exp_reads[a.parity];
  a.inv = mode == B2_REDUCE_AVERAGE ? 1.0 / static_cast<double>(n_nbrs) : 1.0;
  for (int j = 0; j < c->world; ++j) a.win[j] = w->peer[j];
  a.off_dbuf = w->off_dbuf[a.parity];
  a.off_gate = w->off_gate;
  a.gate_stride = w->gate_stride;
  for (int i = 0; i < n_nbrs; ++i)
    a.sends[i] = w->sends_from[nbrs[i]] + (n_nbrs > 1 ? 1 : 0);
  a.partials = w->partials;
  a.cta_done = w->cta_done;
  a.gridbar = w->cta_done + kMaxRanks + 2;
  a.sched = static_sched() ? nullptr : w->sched;
  a.sched_end = reinterpret_cast<unsigned*>(w->sched + kSchedPasses);
  a.status = w->fail;
  a.timeout_ns = c->timeout_ns;
  a.trace = c->trace;
  a.sr_on = sr_on;
  a.sr_seed = sr_seed;
  rc = launch_decent_small(a, codec == B2_CODEC_UNIFORM8 ? kU8 : kIdentity, static_cast<cudaStream_t>(stream),
                           c->sm_budget);
  if (rc == B2_ERR_UNSUPPORTED)
    rc = launch_decent(a, codec == B2_CODEC_UNIFORM8 ? kU8 : kIdentity, static_cast<cudaStream_t>(stream),
                       c->sm_budget);
  if (rc == B2_OK) {
    w->exp_reads[a.parity] += static_cast<unsigned long long>(n_nbrs - 1);
    if (n_nbrs > 1)
      for (int i = 0; i < n_nbrs; ++i) w->sends_from[nbrs[i]] = a.sends[i];
    ++c->launches;
  }
  return rc;
}

int b2_c_lp_s_stochastic(b2_comm_t c, float* x, size_t n, float* delta, size_t delta_len, float* eps,
                         size_t eps_len, uint64_t seed, uint32_t bucket, void* stream) {
  return central(c, x, n, B2_CODEC_UNIFORM8, 1, delta, delta_len, eps, eps_len, bucket, stream, 1, seed);
}

int b2_d_lp_s_stochastic(b2_comm_t c, float* x, size_t n, const int* nbrs, int n_nbrs, int mode, uint64_t seed,
                         uint32_t bucket, void* stream) {
  return decentral(c, x, n, nbrs, n_nbrs, B2_CODEC_UNIFORM8, 1, mode, bucket, stream, 1, seed);
}

int b2_hierarchical_c(b2_comm_t c, float* x, size_t n, uint32_t bucket, void* stream) {
  int rc = check_comm(c, x, n);
  if (rc) return rc;
  if (c->world > 1) return central(c, x, n, B2_CODEC_IDENTITY, 0, nullptr, 0, nullptr, 0, bucket, stream);
  const int self = c->rank;  // one rank: (float)(0.0 + (double)x), D_FP_S over {self}
  return decentral(c, x, n, &self, 1, B2_CODEC_IDENTITY, 0, B2_REDUCE_SUM, bucket, stream);
}

int b2_d_fp_s(b2_comm_t c, float* x, size_t n, const int* nbrs, int n_nbrs, int mode,
              uint32_t bucket, void* stream) {
  return decentral(c, x, n, nbrs, n_nbrs, B2_CODEC_IDENTITY, 0, mode, bucket, stream);
}

int b2_d_lp_s(b2_comm_t c, float* x, size_t n, const int* nbrs, int n_nbrs, int codec, int mode,
              uint32_t bucket, void* stream) {
  B2_REQUIRE(codec == B2_CODEC_UNIFORM8 || codec == B2_CODEC_IDENTITY || codec == B2_CODEC_ONEBIT,
             "unknown codec %d", codec);
  return decentral(c, x, n, nbrs, n_nbrs, codec, 1, mode, bucket, stream);
}

}  // extern "C"
