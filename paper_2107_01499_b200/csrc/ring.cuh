// ring.cuh -- warp-specialized TMA streaming for the persistent collective
// kernels: one producer warp issues cp.async.bulk copies (global -- local
// HBM or a peer GPU's window over NVLink -- into shared memory) into a ring
// of kStages x kStageBytes stages guarded by mbarriers; kConsumerWarps
// consumer warps compute from shared memory.  Memory-level parallelism is the
// ring size (192 KB per SM in flight), independent of register count.
//
// A "pass" streams an element range [s, s+n) of up to kMaxRanks equally
// shaped sources; its 16-element-aligned body is cut into tiles of
// tile_units * 16 elements handed to CTAs round-robin.  The (< 16 element)
// unaligned head and tail are processed by the consumers of the last CTA
// with plain loads.  Producer and consumers walk identical tile sequences,
// so the ring cursor (stage, phase) stays in lock step across passes.
#pragma once

#include <cstdint>

#include "b2_device.cuh"

namespace b2 {

// Warp roles: warp 0 = producer (TMA loads), warp 1 = storer (TMA bulk
// stores of staged payloads to peers + their completion/signalling), warps
// 2.. = consumers.  20 warps = 5 per SM sub-partition at 96 registers.
constexpr int kConsumerWarps = 18;
constexpr int kConsumers = 32 * kConsumerWarps;          // 576 consumer threads
constexpr int kFirstConsumer = 64;                        // threadIdx of consumer 0
constexpr int kRingThreads = kConsumers + kFirstConsumer; // 640
constexpr int kStages = 5;
constexpr int kStageBytes = 32768;
constexpr int kSlots = 5;                                 // staging ring for pushed payloads
constexpr int kSlotBytes = 8192;                          // codes of one 32 KB fp32 tile
constexpr int kRingSmem = 256 + kStages * kStageBytes + kSlots * kSlotBytes;  // 200 KB + barriers
constexpr int kConsumerBar = 1;                           // named barrier id

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global (local HBM or peer-mapped NVLink address) -> shared, completes tx on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Order this thread's generic-proxy global writes before later async-proxy
// (TMA) reads of the same bytes, on this or another GPU.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// shared -> global (local HBM or a peer's window) bulk store, tracked by the
// issuing thread's bulk async-group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the smem source of every committed bulk store but the N most recent has been read
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// every committed bulk store has completed (its writes are performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kConsumerBar), "n"(kConsumers) : "memory");
}

struct PassDesc {
  size_t s = 0, n = 0;                  // element range
  int nsrc = 1, eb = 4;                 // sources, bytes per element
  const uint8_t* base[kMaxRanks] = {};  // address of element e of source i = base[i] + eb * e
  const unsigned long long* wait_flag = nullptr;  // producer: wait *flag >= target before loading
  unsigned long long wait_target = 0;
  bool reverse = false;  // walk this CTA's tiles backwards: re-reads the tail of a
                         // range that was streamed forwards just before from L2
  __host__ __device__ int tile_units() const { return kStageBytes / (nsrc * 16 * eb); }
  __host__ __device__ size_t u0() const { return (s + 15) >> 4; }
  __host__ __device__ size_t u1() const { return (s + n) >> 4; }
  __host__ __device__ size_t nunits() const { return u1() > u0() ? u1() - u0() : 0; }
  __host__ __device__ size_t body_begin() const { return nunits() ? 16 * u0() : s + n; }
  __host__ __device__ size_t body_end() const { return nunits() ? 16 * u1() : s + n; }
};

struct Ring {
  uint64_t* full;
  uint64_t* empty;
  uint64_t* staged;  // consumers -> storer: slot filled
  uint64_t* sfree;   // storer -> consumers: slot read by the bulk store
  uint8_t* buf;
  uint8_t* slots;
  int stage = 0;
  unsigned phase = 0;
  int slot = 0;       // staging cursor (consumers and storer walk it in lock step)
  unsigned sphase = 0;
  bool producer;
  bool storer;
  int ct;  // consumer thread index 0..kConsumers-1 (producer / storer: -1)
  int* status;
  unsigned long long timeout_ns;

  __device__ void init(uint8_t* smem, int* st, unsigned long long to) {
    full = reinterpret_cast<uint64_t*>(smem);
    empty = full + kStages;
    staged = empty + kStages;
    sfree = staged + kSlots;
    buf = smem + 256;
    slots = buf + size_t(kStages) * kStageBytes;
    producer = threadIdx.x < 32;
    storer = threadIdx.x >= 32 && threadIdx.x < kFirstConsumer;
    ct = threadIdx.x >= kFirstConsumer ? int(threadIdx.x) - kFirstConsumer : -1;
    status = st;
    timeout_ns = to;
    if (threadIdx.x == 0) {
      for (int i = 0; i < kStages; ++i) {
        mbar_init(full + i, 1);
        mbar_init(empty + i, kConsumerWarps);
      }
      for (int i = 0; i < kSlots; ++i) {
        mbar_init(staged + i, kConsumerWarps);
        mbar_init(sfree + i, 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  __device__ __forceinline__ void advance_slot() {
    if (++slot == kSlots) {
      slot = 0;
      sphase ^= 1u;
    }
  }
  // consumers: wait until the current staging slot may be overwritten
  __device__ __forceinline__ uint8_t* slot_acquire() {
    mbar_wait(sfree + slot, sphase ^ 1u);
    return slots + size_t(slot) * kSlotBytes;
  }
  // consumers: the slot is filled (every consumer thread calls this)
  __device__ __forceinline__ void slot_commit() {
    fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(staged + slot);
    advance_slot();
  }
  // storer lane 0: push the next filled slot to dst.  Up to kPushInFlight
  // bulk stores stay in flight; a slot is released to the consumers once its
  // store has finished reading shared memory (FIFO order).
  static constexpr int kPushInFlight = kSlots - 1;
  int pending = 0;    // storer: slots pushed but not yet released
  int rel = 0;        // storer: oldest unreleased slot
  __device__ __forceinline__ void slot_push(void* dst, unsigned bytes) {
    mbar_wait(staged + slot, sphase);
    bulk_s2g(dst, slots + size_t(slot) * kSlotBytes, bytes);
    advance_slot();
    if (++pending > kPushInFlight) {
      bulk_wait_read<kPushInFlight>();
      mbar_arrive(sfree + rel);
      rel = rel + 1 == kSlots ? 0 : rel + 1;
      --pending;
    }
  }
  __device__ __forceinline__ void advance() {
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
  // storer lane 0: every push performed (writes visible); release all slots
  __device__ __forceinline__ void push_drain() {
    bulk_wait_all();
    while (pending > 0) {
      mbar_arrive(sfree + rel);
      rel = rel + 1 == kSlots ? 0 : rel + 1;
      --pending;
    }
  }

  // Stream one pass.  consume(stage_ptr, first_element, units, tile_units)
  // runs on every consumer thread for every tile this CTA owns.
  template <class F>
  __device__ void run(const PassDesc& p, F&& consume) {
    const int T = p.tile_units();
    const size_t ntiles = (p.nunits() + T - 1) / T;
    const size_t m = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    bool waited = p.wait_flag == nullptr;
    for (size_t i = 0; i < m; ++i) tile(p, tile_index(p, i, m), consume, waited);
  }
  __device__ __forceinline__ size_t tile_index(const PassDesc& p, size_t i, size_t m) const {
    return blockIdx.x + (p.reverse ? m - 1 - i : i) * gridDim.x;
  }

  // Stream two passes with their tiles interleaved (a0 b0 a1 b1 ...), so e.g.
  // an NVLink-bound push pass overlaps an HBM-bound min/max pass.
  template <class FA, class FB>
  __device__ void run2(const PassDesc& pa, FA&& fa, const PassDesc& pb, FB&& fb) {
    const int Ta = pa.tile_units(), Tb = pb.tile_units();
    const size_t na = (pa.nunits() + Ta - 1) / Ta, nb = (pb.nunits() + Tb - 1) / Tb;
    const size_t ma = na > blockIdx.x ? (na - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const size_t mb = nb > blockIdx.x ? (nb - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const size_t m = ma > mb ? ma : mb;
    bool wa = pa.wait_flag == nullptr, wb = pb.wait_flag == nullptr;
    for (size_t i = 0; i < m; ++i) {
      if (i < ma) tile(pa, tile_index(pa, i, ma), fa, wa);
      if (i < mb) tile(pb, tile_index(pb, i, mb), fb, wb);
    }
  }

  // Stream np passes with their tiles interleaved round-robin (pass 0 tile 0,
  // pass 1 tile 0, ..., pass 0 tile 1, ...): e.g. pull every owner's payload
  // at once, which keeps NVLink fan-in balanced whatever the rank skew.
  template <class F>
  __device__ void run_multi(const PassDesc* ps, int np, F&& consume) {
    run_multi(ps, np, consume, [](int) {});
  }
  // ready(i) runs on the producer lane right after pass i's wait flag is
  // satisfied and before its first tile is handed over, so anything it writes
  // to shared memory (e.g. the pass's codec header) is visible to the
  // consumers of every tile of pass i (mbarrier release/acquire).
  template <class F, class R>
  __device__ void run_multi(const PassDesc* ps, int np, F&& consume, R&& ready) {
    size_t mm[kMaxRanks];
    bool w[kMaxRanks];
    size_t m = 0;
    for (int i = 0; i < np; ++i) {
      const int T = ps[i].tile_units();
      const size_t nt = (ps[i].nunits() + T - 1) / T;
      mm[i] = nt > blockIdx.x ? (nt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
      m = mm[i] > m ? mm[i] : m;
      w[i] = false;
    }
    for (size_t t = 0; t < m; ++t)
      for (int i = 0; i < np; ++i)
        if (t < mm[i]) {
          if (producer && threadIdx.x == 0 && !w[i]) {
            if (ps[i].wait_flag) {
              wait_geq(ps[i].wait_flag, ps[i].wait_target, timeout_ns, status);
              fence_proxy_async();
            }
            ready(i);
          }
          w[i] = true;
          tile(ps[i], tile_index(ps[i], t, mm[i]),
               [&](const uint8_t* st, size_t e0, size_t units, int T) { consume(i, st, e0, units, T); }, w[i]);
        }
  }

  // One tile of a pass (producer lane 0 issues, consumers consume).  The
  // producer honours the pass's wait flag before its first tile (`waited`).
  template <class F>
  __device__ __forceinline__ void tile(const PassDesc& p, size_t t, F&& consume, bool& waited) {
    const size_t u0 = p.u0(), nun = p.nunits();
    const int T = p.tile_units();
    const size_t units = (nun - t * T) < size_t(T) ? (nun - t * T) : size_t(T);
    if (storer) return;
    if (producer) {
      if ((threadIdx.x & 31) != 0) return;
      if (!waited) {
        wait_geq(p.wait_flag, p.wait_target, timeout_ns, status);
        fence_proxy_async();
        waited = true;
      }
      mbar_wait(empty + stage, phase ^ 1u);
      const unsigned bytes = unsigned(units * 16 * p.eb);
      mbar_expect_tx(full + stage, bytes * p.nsrc);
      uint8_t* dst = buf + size_t(stage) * kStageBytes;
      const size_t off = size_t(p.eb) * 16 * (u0 + t * T);
      for (int i = 0; i < p.nsrc; ++i)
        bulk_g2s(dst + size_t(i) * T * 16 * p.eb, p.base[i] + off, bytes, full + stage);
      advance();
      return;
    }
    mbar_wait(full + stage, phase);
    consume(buf + size_t(stage) * kStageBytes, 16 * (u0 + t * T), units, T);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(empty + stage);
    advance();
  }

  // Unaligned head/tail elements of a pass (consumer warp 0 of the last CTA).
  template <class F>
  __device__ void edges(const PassDesc& p, F&& fn) const {
    if (ct < 0 || blockIdx.x != gridDim.x - 1 || ct >= 32) return;
    const size_t b0 = p.body_begin(), b1 = p.body_end(), e1 = p.s + p.n;
    for (size_t e = p.s + ct; e < b0; e += 32) fn(e);
    for (size_t e = b1 + ct; e < e1; e += 32) fn(e);
  }
};

// (lo, hi) over the consumer threads of the CTA; result valid in all consumers.
__device__ __forceinline__ float2 consumer_minmax(float lo, float hi, float2* smem /*[32]*/) {
  lo = warp_min_nan(lo);
  hi = warp_max_nan(hi);
  const int w = (threadIdx.x >> 5) - kFirstConsumer / 32, l = threadIdx.x & 31;
  consumer_sync();
  if (l == 0) smem[w] = make_float2(lo, hi);
  consumer_sync();
  const float2 v = l < kConsumerWarps ? smem[l] : smem[0];
  lo = warp_min_nan(v.x);
  hi = warp_max_nan(v.y);
  return make_float2(lo, hi);
}

// Grid-wide barrier among the CONSUMER threads of every CTA (the producer
// warps keep prefetching across it).  ws[0] = arrival count, ws[1] = generation.
__device__ __forceinline__ void consumer_grid_sync(unsigned* ws) {
  __threadfence();
  consumer_sync();
  if (threadIdx.x == kFirstConsumer) {
    volatile unsigned* gen = ws + 1;
    const unsigned g0 = *gen;
    if (atomicAdd(ws, 1u) == gridDim.x - 1) {
      atomicExch(ws, 0u);
      __threadfence();
      atomicAdd(ws + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  consumer_sync();
}

// Fence this CTA's (consumer) writes and report whether this CTA arrived
// last at ctr (ctr is then reset for the next call).  SYS = true for writes
// that went to a PEER's memory (phase-1 pushes): they must be performed at
// system scope before the owner is signalled.  Writes to local memory that
// peers later read through this GPU's L2 need only gpu scope; the flag itself
// is released at system scope by the caller.  The proxy fence makes the data
// visible to TMA (async-proxy) readers.
template <bool SYS>
__device__ __forceinline__ bool consumer_arrive(unsigned* ctr, int* flag_smem,
                                                unsigned long long* tr = nullptr) {
  fence_proxy_async();  // every writer: generic -> async-proxy (TMA readers)
  consumer_sync();      // all consumer writes happen-before consumer 0's fence
  if (threadIdx.x == kFirstConsumer) {
    if (tr) tr[0] = globaltimer();
    // one cumulative fence per CTA (the cooperative-groups grid-sync pattern)
    if (SYS)
      __threadfence_system();
    else
      __threadfence();
    if (tr) tr[1] = globaltimer();
    const unsigned old = atomicAdd(ctr, 1u);
    const int last = old == gridDim.x - 1;
    if (last) {
      atomicExch(ctr, 0u);
      __threadfence_system();
    }
    if (tr) tr[2] = globaltimer();
    *flag_smem = last;
  }
  consumer_sync();
  return *flag_smem != 0;
}

}  // namespace b2
