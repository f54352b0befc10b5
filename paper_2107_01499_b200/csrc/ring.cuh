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
constexpr int kRingSmem = 512 + kStages * kStageBytes + kSlots * kSlotBytes;  // 200 KB + control
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
  void** slot_dst;     // smem [kSlots]: push destination of a staged slot
  unsigned* slot_len;  // smem [kSlots]: its byte count (0 = end-of-chunk marker)
  int stage = 0;
  unsigned phase = 0;
  int slot = 0;       // staging cursor (consumers and storer walk it in lock step)
  unsigned sphase = 0;
  bool producer;
  bool storer;
  int ct;  // consumer thread index 0..kConsumers-1 (producer / storer: -1)
  unsigned long long* info;            // smem [kStages]: (pass << 40 | tile) of a stage, ~0 = END
  unsigned long long* sched = nullptr;  // global per-pass tile counters (dynamic mode) or null
  int npass = 0;                        // passes streamed so far (identical in every role)
  int* status;
  unsigned long long timeout_ns;

  __device__ void init(uint8_t* smem, int* st, unsigned long long to, unsigned long long* sched_ctrs = nullptr) {
    sched = sched_ctrs;
    full = reinterpret_cast<uint64_t*>(smem);
    empty = full + kStages;
    staged = empty + kStages;
    sfree = staged + kSlots;
    info = reinterpret_cast<unsigned long long*>(sfree + kSlots);
    slot_dst = reinterpret_cast<void**>(info + kStages);
    slot_len = reinterpret_cast<unsigned*>(slot_dst + kSlots);
    buf = smem + 512;
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
  // consumers: the slot is filled (every consumer thread calls this).
  // Consumer 0 records where the storer must push it (bytes == 0: a marker).
  __device__ __forceinline__ void slot_commit(void* dst, unsigned bytes) {
    if (ct == 0) {
      slot_dst[slot] = dst;
      slot_len[slot] = bytes;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(staged + slot);
    advance_slot();
  }
  // storer lane 0: push the next filled slot.  Up to kPushInFlight bulk
  // stores stay in flight; a slot is released to the consumers once its store
  // has finished reading shared memory (FIFO order).  Returns false (and
  // consumes the slot) on a marker.
  static constexpr int kPushInFlight = kSlots - 1;
  int pending = 0;    // storer: slots pushed but not yet released
  int rel = 0;        // storer: oldest unreleased slot
  __device__ __forceinline__ bool slot_push() {
    mbar_wait(staged + slot, sphase);
    const unsigned bytes = slot_len[slot];
    if (bytes == 0) {  // marker: release it in FIFO order too
      advance_slot();
      ++pending;
      return false;
    }
    bulk_s2g(slot_dst[slot], slots + size_t(slot) * kSlotBytes, bytes);
    advance_slot();
    if (++pending > kPushInFlight) {
      bulk_wait_read<kPushInFlight>();
      mbar_arrive(sfree + rel);
      rel = rel + 1 == kSlots ? 0 : rel + 1;
      --pending;
    }
    return true;
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

  // ---------------------------------------------------------------- passes
  // Stream one pass.  consume(stage_ptr, first_element, units, tile_units)
  // runs on every consumer thread for every tile handed to this CTA.
  template <class F>
  __device__ void run(const PassDesc& p, F&& consume) {
    stream(&p, 1, [&](int, const uint8_t* st, size_t e0, size_t units, int T) { consume(st, e0, units, T); },
           [](int) {});
  }

  // Two passes with their tiles interleaved (a b a b ...), so e.g. an
  // NVLink-bound push pass overlaps an HBM-bound min/max pass.
  template <class FA, class FB>
  __device__ void run2(const PassDesc& pa, FA&& fa, const PassDesc& pb, FB&& fb) {
    const PassDesc ps[2] = {pa, pb};
    stream(ps, 2,
           [&](int i, const uint8_t* st, size_t e0, size_t units, int T) {
             if (i == 0)
               fa(st, e0, units, T);
             else
               fb(st, e0, units, T);
           },
           [](int) {});
  }

  // np passes interleaved round-robin: e.g. pull every owner's payload at
  // once (balanced NVLink fan-in whatever the rank skew).  ready(i) runs on
  // the producer lane after pass i's wait flag is satisfied and before its
  // first tile is handed over, so what it writes to shared memory (e.g. the
  // pass's codec header) is visible to the consumers of all of pass i's tiles.
  template <class F>
  __device__ void run_multi(const PassDesc* ps, int np, F&& consume) {
    stream(ps, np, consume, [](int) {});
  }
  template <class F, class R>
  __device__ void run_multi(const PassDesc* ps, int np, F&& consume, R&& ready) {
    stream(ps, np, consume, ready);
  }

  // The scheduler.  Static mode (sched == nullptr): CTA b takes tiles b, b+G,
  // ... of every pass.  Dynamic mode: the producer lane grabs tiles from one
  // global counter per pass (atomicAdd), so fast SMs take more tiles and every
  // CTA finishes a pass at about the same time -- static assignment left a
  // 10-20 us spread per pass, and every grid barrier waits for the slowest
  // CTA.  Reverse passes hand tiles out from the END (the producer maps the
  // counter c to ntiles-1-c), which is what makes a reverse re-read hit L2.
  // The stage's tile (or the END marker) travels to the consumers in shared
  // memory (info[]), published by the mbarrier arrive.
  template <class F, class R>
  __device__ void stream(const PassDesc* ps, int np, F&& consume, R&& ready) {
    const int pid0 = npass;
    npass += np;
    if (storer) return;
    if (producer) {
      if ((threadIdx.x & 31) != 0) return;
      bool live[kMaxRanks], got[kMaxRanks];
      size_t nt[kMaxRanks], k[kMaxRanks];
      int nlive = 0;
      for (int i = 0; i < np; ++i) {
        const int T = ps[i].tile_units();
        nt[i] = (ps[i].nunits() + T - 1) / T;
        k[i] = 0;
        got[i] = false;
        live[i] = nt[i] > (sched ? 0 : blockIdx.x);
        nlive += live[i];
      }
      int nready = 0;
      while (nlive) {
        for (int i = 0; i < np; ++i) {
          if (!live[i]) continue;
          if (!got[i]) {
            // A pass whose data is not published yet is skipped while another
            // pass has tiles to hand out; with nothing else to do, block.
            if (ps[i].wait_flag && ld_acquire_sys(ps[i].wait_flag) < ps[i].wait_target) {
              if (nready > 0) continue;
              wait_geq(ps[i].wait_flag, ps[i].wait_target, timeout_ns, status);
            }
            if (ps[i].wait_flag) fence_proxy_async();
            ready(i);
            got[i] = true;
            ++nready;
          }
          size_t t;
          if (sched) {
            const unsigned long long c = atomicAdd(sched + pid0 + i, 1ull);
            if (c >= nt[i]) {
              live[i] = false;
              --nlive;
              --nready;
              continue;
            }
            t = ps[i].reverse ? nt[i] - 1 - c : c;
          } else {
            const size_t m = (nt[i] - blockIdx.x + gridDim.x - 1) / gridDim.x;
            const size_t j = k[i]++;
            t = blockIdx.x + (ps[i].reverse ? m - 1 - j : j) * gridDim.x;
            if (k[i] == m) {
              live[i] = false;
              --nlive;
              --nready;
            }
          }
          issue(ps[i], i, t);
        }
      }
      mbar_wait(empty + stage, phase ^ 1u);  // END marker
      info[stage] = ~0ull;
      mbar_arrive(full + stage);
      advance();
      return;
    }
    while (true) {
      mbar_wait(full + stage, phase);
      const unsigned long long inf = info[stage];
      if (inf == ~0ull) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + stage);
        advance();
        break;
      }
      const int i = int(inf >> 40);
      const size_t t = size_t(inf & ((1ull << 40) - 1));
      const PassDesc& p = ps[i];
      const int T = p.tile_units();
      const size_t nun = p.nunits();
      const size_t units = (nun - t * T) < size_t(T) ? (nun - t * T) : size_t(T);
      consume(i, buf + size_t(stage) * kStageBytes, 16 * (p.u0() + t * T), units, T);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(empty + stage);
      advance();
    }
  }

  // producer lane: load tile t of pass p (index i) into the next stage
  __device__ __forceinline__ void issue(const PassDesc& p, int i, size_t t) {
    const size_t nun = p.nunits();
    const int T = p.tile_units();
    const size_t units = (nun - t * T) < size_t(T) ? (nun - t * T) : size_t(T);
    mbar_wait(empty + stage, phase ^ 1u);
    info[stage] = (static_cast<unsigned long long>(i) << 40) | t;
    const unsigned bytes = unsigned(units * 16 * p.eb);
    mbar_expect_tx(full + stage, bytes * p.nsrc);
    uint8_t* dst = buf + size_t(stage) * kStageBytes;
    const size_t off = size_t(p.eb) * 16 * (p.u0() + t * T);
    for (int s = 0; s < p.nsrc; ++s) bulk_g2s(dst + size_t(s) * T * 16 * p.eb, p.base[s] + off, bytes, full + stage);
    advance();
  }

  // Kernel epilogue (all threads): the last CTA resets the dynamic tile
  // counters for the next launch on this workspace.
  __device__ void finish(unsigned* end_ctr) {
    __syncthreads();
    if (sched && threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(end_ctr, 1u) == gridDim.x - 1) {
        for (int i = 0; i < npass; ++i) sched[i] = 0ull;
        *end_ctr = 0u;
        __threadfence();
      }
    }
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
