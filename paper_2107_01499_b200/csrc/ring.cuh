// ring.cuh -- warp-specialized TMA streaming for the persistent collective
// kernels: a producer warp issues cp.async.bulk copies (global -- local HBM
// or a peer GPU's window over NVLink -- into shared memory) into a ring of
// kStages x kStageBytes stages guarded by mbarriers; kConsumerWarps consumer
// warps compute from shared memory.  Memory-level parallelism is the ring
// (160 KB per SM in flight), independent of register count.
//
// A "pass" streams an element range [s, s+n) of up to kMaxRanks equally
// shaped sources; its 16-element-aligned body is cut into tiles of
// tile_units * 16 elements.  Tiles are handed out "guided" (a static share
// per CTA, the tail by a global atomic counter per pass), optionally gated on
// arrival counters (PassDesc::gate); the producer tells the consumers which
// tile a stage holds through shared memory (TileInfo), so several passes can
// be interleaved tile by tile.  The (< 16 element) unaligned head and tail
// are processed by the consumers of the last CTA with plain loads.  Split
// mode runs two such pipelines side by side (split_begin); push credits hand
// the consumers' stores to a signaller warp that publishes them (slot_commit).
#pragma once

#include <cstdint>

#include "b2_device.cuh"

namespace b2 {

// Warp roles: warp 0 = producer (TMA loads), warp 1 = signaller ("storer":
// confirms the consumers' stores and signals their readers, see slot_commit),
// warps 2..18 = consumers, warp 19 = second producer (split mode only, see
// split_begin).  20 warps = 5 per SM sub-partition at 96 registers.
constexpr int kConsumerWarps = 17;
constexpr int kConsumers = 32 * kConsumerWarps;          // 544 consumer threads
constexpr int kFirstConsumer = 64;                        // threadIdx of consumer 0
constexpr int kProducer2 = kFirstConsumer + kConsumers;  // threadIdx of the second producer (608)
constexpr int kRingThreads = kProducer2 + 32;             // 640
// Split mode: pipe A = stages [0, kSplitStagesA) with consumer warps
// [0, kSplitWarpsA), pipe B = the remaining stages and warps.
constexpr int kSplitStagesA = 3;
constexpr int kSplitWarpsA = 10;
#ifndef B2_RING_STAGES  // overridable for the ring microbenchmark (tests/cpp/ring_bench.cu)
#define B2_RING_STAGES 5
#endif
#ifndef B2_RING_STAGE_BYTES
#define B2_RING_STAGE_BYTES 32768
#endif
constexpr int kStages = B2_RING_STAGES;
constexpr int kStageBytes = B2_RING_STAGE_BYTES;
constexpr int kSlots = 64;                      // push credits: consumers -> signaller
constexpr int kCtrlBytes = 4096;                // mbarriers + stage/slot metadata + producer state
constexpr int kRingSmem = kCtrlBytes + kStages * kStageBytes;  // 162 KB by default
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
#ifdef B2_MBAR_POLL
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
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
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kConsumerBar), "n"(kConsumers) : "memory");
}

// Tile gating: a pass may be gated per region of kGateUnits (b2_device.cuh) 16-byte units
// (from the pass start): tile t may only be loaded once gate[region] >=
// gate_mult * (units of that region).  Writers add the units they delivered,
// so the count does not depend on anybody's tile size.

struct PassDesc {  // trivially constructible (lives in shared memory); build with make()
  size_t s, n;                     // element range
  int nsrc, eb;                    // sources, bytes per element
  const uint8_t* base[kMaxRanks];  // address of element e of source i = base[i] + eb * e (i < nsrc)
  const unsigned long long* wait_flag;  // producer: wait *flag >= target before loading
  unsigned long long wait_target;
  const unsigned long long* gate;  // per-region arrival counters, or null
  unsigned long long gate_mult;
  // gate_nsrc > 0: one cumulative counter per SOURCE instead of one for all:
  // region r is ready once gate[gate_src[s] * gate_stride + r] >=
  // gate_tgt[s] * units(r) for every s < gate_nsrc.  (D_* with a changing
  // topology: a rank that is not my neighbour in this call may run calls
  // ahead and add to my counters; only my current neighbours' counters are
  // checked, each against the number of calls in which it sent to me.)
  int gate_nsrc;
  int gate_src[kMaxRanks];
  unsigned long long gate_tgt[kMaxRanks];
  size_t gate_stride;
  bool reverse;  // walk the tiles backwards: re-reads the tail of a range
                 // that was streamed forwards just before from L2
  static __host__ __device__ PassDesc make() {
    PassDesc p{};
    p.nsrc = 1;
    p.eb = 4;
    return p;
  }
  // a power of two (so tiles of every pass over one range nest in gate regions)
  __host__ __device__ int tile_units() const {
    const int m = kStageBytes / (nsrc * 16 * eb);
    int t = 1;
    while (2 * t <= m) t *= 2;
    return t;
  }
  __host__ __device__ size_t u0() const { return (s + 15) >> 4; }
  __host__ __device__ size_t u1() const { return (s + n) >> 4; }
  __host__ __device__ size_t nunits() const { return u1() > u0() ? u1() - u0() : 0; }
  __host__ __device__ size_t body_begin() const { return nunits() ? 16 * u0() : s + n; }
  __host__ __device__ size_t body_end() const { return nunits() ? 16 * u1() : s + n; }
  __host__ __device__ size_t region_of(size_t t) const { return t * size_t(tile_units()) / kGateUnits; }
  // all sources of region r have landed (acquire: the caller's TMA loads follow)
  __device__ __forceinline__ bool gate_ready(size_t r, bool acquire) const {
    if (gate_nsrc == 0) {
      const unsigned long long v = acquire ? ld_acquire_sys(gate + r)
                                           : *reinterpret_cast<const volatile unsigned long long*>(gate + r);
      return v >= gate_target(r);
    }
    const unsigned long long u = gate_target(r) / (gate_mult ? gate_mult : 1);  // units of region r
    for (int s = 0; s < gate_nsrc; ++s) {
      const unsigned long long* q = gate + size_t(gate_src[s]) * gate_stride + r;
      const unsigned long long v = acquire ? ld_acquire_sys(q) : *reinterpret_cast<const volatile unsigned long long*>(q);
      if (v < gate_tgt[s] * u) return false;
    }
    return true;
  }
  __host__ __device__ unsigned long long gate_target(size_t r) const {
    const size_t left = nunits() - r * kGateUnits;
    return gate_mult * (left < size_t(kGateUnits) ? left : size_t(kGateUnits));
  }
};

// What the producer tells the consumers about a stage (pass == kEndPass: END).
struct TileInfo {
  unsigned long long e0;  // first element of the tile
  unsigned units;         // 16-byte units in the tile
  unsigned short pass;    // index of the pass in the stream() call
  unsigned short T;       // tile_units() of the pass (source stride in the stage)
};
constexpr unsigned short kEndPass = 0xFFFF;

// Producer-lane bookkeeping of one pass of a stream() call, in shared memory
// (per-tile work of the single producer lane is the ring's critical path:
// everything that does not change per tile is computed once per pass).
struct ProdPass {
  unsigned long long nt;    // tiles
  unsigned long long k;     // statically assigned tiles taken so far
  unsigned long long ms;    // statically assigned tiles of this CTA
  unsigned long long dyn0;  // first dynamically scheduled logical tile
  unsigned long long nun;   // 16-byte units
  unsigned long long u0;    // first unit
  unsigned long long rdy;   // gated passes: 1 + a region known to have landed (0: none)
  unsigned long long first, last;  // traced: globaltimer of the first / last tile issued
  unsigned T;               // tile units
  unsigned tbytes;          // bytes of one source of a full tile (T * 16 * eb)
};
constexpr int kMaxPasses = kMaxRanks + 1;
static_assert(2 * kMaxPasses * sizeof(ProdPass) <= 4096 - 2560, "producer state exceeds the control block");

// One mbarrier-guarded ring of stage buffers (a view of the shared stages).
struct Pipe {
  uint64_t* full;
  uint64_t* empty;
  int first;  // first stage buffer of this pipe
  int nst;    // stage buffers
  int stage = 0;
  unsigned phase = 0;
  unsigned long long nissued = 0;  // producer: tiles (+ END markers) issued
  __device__ __forceinline__ void advance() {
    ++nissued;
    if (++stage == nst) {
      stage = 0;
      phase ^= 1u;
    }
  }
  // producer: wait until every issued stage has been released by the consumers
  __device__ __forceinline__ void drain() {
    for (int j = 0; j < nst; ++j) {
      if (nissued < unsigned(j + 1)) break;
      const unsigned long long k = nissued - 1 - j;  // issue number
      mbar_wait(empty + int(k % nst), unsigned(k / nst) & 1u);
    }
  }
};

struct Ring {
  uint64_t* staged;  // consumers -> signaller: the pushes of a credit are issued
  uint64_t* sfree;   // signaller -> consumers: the credit is free again
  uint8_t* buf;
  unsigned* slot_len;  // smem [kSlots]: 0 = end marker
  unsigned long long** slot_sig;  // smem [kSlots]: counter to bump once the pushes have landed, or null
  unsigned* slot_sigv;            // smem [kSlots]: by how much
  // Pipe state stays in registers: named fields, no arrays / pointers into
  // the Ring (either would put the whole per-thread Ring in local memory)
  Pipe cp;        // the pipe this thread's role works on now
  Pipe p0;        // the all-stage pipe, parked while in split mode
  Pipe pA, pB;    // the split pipes, parked between split phases
  bool split_init = false;
  int slot = 0;       // staging cursor (consumers and storer walk it in lock step)
  unsigned sphase = 0;
  bool producer;      // warp 0 (lane 0 works)
  bool producer2;     // warp 20 (lane 0 works, split mode only)
  bool storer;
  bool split = false;
  int ct;   // consumer thread index 0..kConsumers-1 (other roles: -1)
  int gct;  // consumer index within its group (split mode) or ct
  int gn;   // consumers in that group (split mode) or kConsumers
  TileInfo* info;                       // smem [kStages]: the tile a stage buffer holds
  ProdPass* pst;                        // smem [kMaxPasses]: producer state of the current stream
  ProdPass* pst2;                       // smem [kMaxPasses]: second producer's
  volatile int* drained;                // smem: split-mode hand-over flags
  unsigned long long* sched = nullptr;  // global per-pass tile counters (dynamic mode) or null
  int npass = 0;                        // passes streamed so far (identical in every role)
  unsigned long long wt[4] = {0, 0, 0, 0};  // traced waits (ns): slot/gate, empty/retire, full
  bool timed = false;                   // accumulate wt[] (tracing only)
  Fail* status;
  unsigned long long timeout_ns;

  __device__ void init(uint8_t* smem, Fail* st, unsigned long long to, unsigned long long* sched_ctrs = nullptr) {
    sched = sched_ctrs;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    // pipe barriers: [full, empty] x (kStages + kSplitStagesA + (kStages - kSplitStagesA)) = 4 kStages
    staged = bars + 4 * kStages;
    sfree = staged + kSlots;
    info = reinterpret_cast<TileInfo*>(sfree + kSlots);
    slot_sig = reinterpret_cast<unsigned long long**>(info + kStages);
    slot_len = reinterpret_cast<unsigned*>(slot_sig + kSlots);
    slot_sigv = slot_len + kSlots;
    drained = reinterpret_cast<volatile int*>(slot_sigv + kSlots);
    pst = reinterpret_cast<ProdPass*>(smem + 2560);
    pst2 = pst + kMaxPasses;
    buf = smem + kCtrlBytes;
    cp = pipe_desc(0);
    producer = threadIdx.x < 32;
    storer = threadIdx.x >= 32 && threadIdx.x < kFirstConsumer;
    producer2 = threadIdx.x >= kProducer2;
    ct = threadIdx.x >= kFirstConsumer && threadIdx.x < kProducer2 ? int(threadIdx.x) - kFirstConsumer : -1;
    gct = ct;
    gn = kConsumers;
    status = st;
    timeout_ns = to;
    if (threadIdx.x == 0) {
      for (int k = 0; k < 3; ++k) {
        const Pipe q = pipe_desc(k);
        const unsigned warps = k == 0 ? kConsumerWarps : k == 1 ? kSplitWarpsA : kConsumerWarps - kSplitWarpsA;
        for (int i = 0; i < q.nst; ++i) {
          mbar_init(q.full + i, 1);
          mbar_init(q.empty + i, warps);
        }
      }
      for (int i = 0; i < kSlots; ++i) {
        mbar_init(staged + i, kSplitWarpsA);  // credits are committed by split group A
        mbar_init(sfree + i, 1);
      }
      drained[0] = drained[1] = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  // pipe k's barriers and stage buffers (0: all stages; 1, 2: split A, B)
  __device__ __forceinline__ Pipe pipe_desc(int k) const {
    uint64_t* bars = reinterpret_cast<uint64_t*>(buf - kCtrlBytes);
    Pipe q;
    if (k == 0) {
      q.full = bars;
      q.first = 0;
      q.nst = kStages;
    } else if (k == 1) {
      q.full = bars + 2 * kStages;
      q.first = 0;
      q.nst = kSplitStagesA;
    } else {
      q.full = bars + 2 * kStages + 2 * kSplitStagesA;
      q.first = kSplitStagesA;
      q.nst = kStages - kSplitStagesA;
    }
    q.empty = q.full + q.nst;
    return q;
  }
  __device__ __forceinline__ unsigned long long tnow() const { return timed ? globaltimer() : 0ull; }
  __device__ __forceinline__ void advance_slot() {
    if (++slot == kSlots) {
      slot = 0;
      sphase ^= 1u;
    }
  }
  // consumers of split group A (split mode) / B
  __device__ __forceinline__ bool group_a() const { return ct >= 0 && ct < 32 * kSplitWarpsA; }
  __device__ __forceinline__ bool group_b() const { return ct >= 32 * kSplitWarpsA; }

  // ------------------------------------------------ split mode
  // Two independent pipelines in one CTA: pipe A (producer warp 0, consumer
  // warps [0, kSplitWarpsA)) and pipe B (producer warp 19, the other consumer
  // warps), each on its own stage buffers, so tiles that arrive slowly (TMA
  // pulls over a saturated NVLink) never hold up the consumers of fast local
  // tiles -- one in-order ring has head-of-line blocking.  Every thread calls
  // split_begin / split_end at the same point; in between, stream_split()
  // runs pass list A on pipe A and list B on pipe B.
  __device__ void split_begin() {
    split = true;
    p0 = cp;
    if (!split_init) {  // the two pipes' barrier phases persist across split phases
      pA = pipe_desc(1);
      pB = pipe_desc(2);
      split_init = true;
    }
    if (producer) {
      if ((threadIdx.x & 31) == 0) {
        cp.drain();  // every stage buffer is free
        drained[0] = 1;
      }
      cp = pA;
    } else if (producer2) {
      if ((threadIdx.x & 31) == 0)
        while (drained[0] == 0) __nanosleep(32);
      cp = pB;
    } else if (ct >= 0) {
      const bool a = group_a();
      cp = a ? pA : pB;
      gct = a ? ct : ct - 32 * kSplitWarpsA;
      gn = a ? 32 * kSplitWarpsA : kConsumers - 32 * kSplitWarpsA;
    }
  }
  __device__ void split_end() {
    split = false;
    if (producer2) {
      if ((threadIdx.x & 31) == 0) {
        cp.drain();
        drained[1] = 1;
      }
    } else if (producer) {
      if ((threadIdx.x & 31) == 0) {
        cp.drain();
        while (drained[1] == 0) __nanosleep(32);
        drained[0] = drained[1] = 0;
      }
    }
    if (producer || group_a())
      pA = cp;
    else if (producer2 || group_b())
      pB = cp;
    cp = p0;
    gct = ct;
    gn = kConsumers;
  }
  // ------------------------------------------------ push credits
  // Consumers store pushed payloads straight to the destination (STG over
  // NVLink: measured faster than TMA bulk stores to peers) and hand the
  // signaller warp (the "storer" role) one credit per tile: the counter to
  // bump once those stores are visible at system scope.  The signaller takes
  // every credit staged so far, issues ONE fence.acq_rel.sys for the batch
  // (cumulative over the consumers' stores, ordered before it by the
  // mbarrier release/acquire) and bumps the counters with relaxed reds -- so
  // the consumers never block on NVLink completion, and a reader learns about
  // each tile a fence latency after its last store.
  __device__ __forceinline__ void slot_acquire() {  // every consumer thread
    const unsigned long long t0 = tnow();
    mbar_wait(sfree + slot, sphase ^ 1u);
    if (timed) wt[0] += globaltimer() - t0;
  }
  // every consumer thread, after its stores of the tile (sig == nullptr and
  // !marker: nothing to signal; marker: the signaller stops after this credit)
  __device__ __forceinline__ void slot_commit(unsigned long long* sig, unsigned sigv, bool marker = false) {
    if (ct == 0) {
      slot_sig[slot] = sig;
      slot_sigv[slot] = sigv;
      slot_len[slot] = marker ? 0u : 1u;
    }
    fence_proxy_async();  // the stores will be read by TMA (async proxy)
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(staged + slot);
    advance_slot();
  }
  // signaller lane 0: serve credits until the marker; returns after it.
  // emit(sig, value) performs one credit's signal after the batch fence
  // (default: a relaxed system-scope red on sig).
  __device__ __forceinline__ void signal_loop() {
    signal_loop([](unsigned long long* sig, unsigned v) { red_relaxed_sys_add(sig, v); });
  }
  template <class E>
  __device__ __forceinline__ void signal_loop(E&& emit) {
    bool done = false;
    while (!done) {
      mbar_wait(staged + slot, sphase);
      int n = 1;  // every credit staged by now joins the batch (a marker ends it)
      {
        int sl = slot;
        unsigned ph = sphase;
        while (n < kSlots && slot_len[sl] != 0) {
          const int nx = sl + 1 == kSlots ? 0 : sl + 1;
          const unsigned nph = sl + 1 == kSlots ? ph ^ 1u : ph;
          if (!mbar_test(staged + nx, nph)) break;
          sl = nx;
          ph = nph;
          ++n;
        }
      }
      const unsigned long long t0 = tnow();
      fence_acq_rel_sys();
      if (timed) wt[1] += globaltimer() - t0;
      for (int j = 0; j < n; ++j) {
        if (slot_len[slot] == 0) done = true;
        if (slot_sig[slot]) emit(slot_sig[slot], slot_sigv[slot]);
        mbar_arrive(sfree + slot);
        advance_slot();
      }
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

  // The scheduler.  Tile c of a pass (logical order) is physical tile
  // t = reverse ? ntiles-1-c : c; reverse passes therefore start at the END,
  // which is what makes a reverse re-read of a just-streamed range hit L2.
  // Static mode (sched == nullptr): CTA b takes logical tiles b, b+G, ...
  // Guided mode: the first kStaticEighths/8 of every pass is assigned
  // statically the same way, the rest is handed out by one global atomic
  // counter per pass, so fast SMs take more of the tail and every CTA
  // finishes a pass at about the same time (static assignment left a 10-20 us
  // spread per pass at 4 GPUs, and every grid barrier waits for the slowest
  // CTA) while the atomic's latency is paid on a quarter of the tiles only.
  // The stage's tile (or the END marker) travels to the consumers in shared
  // memory (info[]), published by the mbarrier arrive.
  static constexpr int kStaticEighths = 6;
  template <class F, class R>
  __device__ void stream(const PassDesc* ps, int np, F&& consume, R&& ready) {
    const int pid0 = npass;
    npass += np;
    stream_at(ps, np, pid0, consume, ready);
  }
  // Split mode: pass list A streams on pipe A, list B on pipe B, at once.
  template <class FA, class RA, class FB, class RB>
  __device__ void stream_split(const PassDesc* pa, int npa, FA&& ca, RA&& ra, const PassDesc* pb, int npb, FB&& cb,
                               RB&& rb) {
    const int pid0 = npass;
    npass += npa + npb;
    if (producer || group_a())
      stream_at(pa, npa, pid0, ca, ra);
    else if (producer2 || group_b())
      stream_at(pb, npb, pid0 + npa, cb, rb);
  }
  template <class F, class R>
  __device__ void stream_at(const PassDesc* ps, int np, int pid0, F&& consume, R&& ready) {
    if (storer || (producer2 && !split)) return;
    Pipe& P = cp;
    if (producer || producer2) {
      if ((threadIdx.x & 31) != 0) return;
      ProdPass* const pst = producer2 ? pst2 : this->pst;
      const unsigned long long G = gridDim.x, b = blockIdx.x;
      unsigned live = 0, got = 0, rev = 0, gated = 0;  // bit i: pass i
      for (int i = 0; i < np; ++i) {
        pst[i].first = pst[i].last = 0;
        const PassDesc& p = ps[i];
        ProdPass& q = pst[i];
        const int T = p.tile_units();
        q.T = unsigned(T);
        q.tbytes = unsigned(T * 16 * p.eb);
        q.u0 = p.u0();
        q.nun = p.nunits();
        q.nt = (q.nun + T - 1) / T;
        const unsigned long long mall = q.nt > b ? (q.nt - b + G - 1) / G : 0;
        const unsigned long long S = sched ? q.nt * kStaticEighths / 8 / G : mall;
        q.ms = S < mall ? S : mall;
        q.dyn0 = S * G;
        q.k = 0;
        q.rdy = 0;
        if (q.ms > 0 || (sched && q.dyn0 < q.nt)) live |= 1u << i;
        if (p.reverse) rev |= 1u << i;
        if (p.gate) gated |= 1u << i;
      }
      // logical index of pass i's next tile for this CTA (take: claim it);
      // ~0 = the pass has nothing left for this CTA
      auto next = [&](int i, bool take) -> unsigned long long {
        ProdPass& q = pst[i];
        const unsigned long long k = q.k;
        if (k < q.ms) {
          if (take) q.k = k + 1;
          return b + k * G;
        }
        if (!sched) return ~0ull;
        const unsigned long long c =
            q.dyn0 + (take ? atomicAdd(sched + pid0 + i, 1ull)
                           : *reinterpret_cast<volatile unsigned long long*>(sched + pid0 + i));
        return c < q.nt ? c : ~0ull;
      };
      bool force = false;  // a whole round skipped everything: block on the next gate
      while (live) {
        bool issued = false;
        for (int i = 0; i < np; ++i) {
          const unsigned bit = 1u << i;
          if (!(live & bit)) continue;
          if (!(got & bit)) {
            // A pass whose data is not published yet is skipped while another
            // pass has tiles to hand out; with nothing else to do, block.
            const PassDesc& p = ps[i];
            if (p.wait_flag && ld_acquire_sys(p.wait_flag) < p.wait_target) {
              if ((live & got) && !force) continue;
              const unsigned long long t0 = tnow();
              wait_geq(p.wait_flag, p.wait_target, timeout_ns, status);
              if (timed) wt[0] += globaltimer() - t0;
            }
            if (p.wait_flag) fence_proxy_async();
            ready(i);
            got |= bit;
          }
          if ((gated & bit) && (live & got & ~bit) && !force) {
            // peek at the next tile: if its region has not landed yet and
            // another pass has work, serve that one first (relaxed load; the
            // acquire happens once per region below)
            const unsigned long long c = next(i, false);
            if (c != ~0ull) {
              const PassDesc& p = ps[i];
              const size_t rg = p.region_of((rev & bit) ? pst[i].nt - 1 - c : c);
              if (pst[i].rdy != rg + 1 && !p.gate_ready(rg, false)) continue;
            }
          }
          const unsigned long long c = next(i, true);
          if (c == ~0ull) {
            live &= ~bit;
            continue;
          }
          if (timed) {
            const unsigned long long now = globaltimer();
            if (!pst[i].first) pst[i].first = now;
            pst[i].last = now;
          }
          const unsigned long long t = (rev & bit) ? pst[i].nt - 1 - c : c;
          if (gated & bit) {
            const PassDesc& p = ps[i];
            const size_t rg = p.region_of(t);
            if (pst[i].rdy != rg + 1) {
              const unsigned long long t0 = tnow();
              if (p.gate_nsrc == 0) {
                wait_geq(p.gate + rg, p.gate_target(rg), timeout_ns, status);
              } else {
                const unsigned long long u = p.gate_target(rg) / (p.gate_mult ? p.gate_mult : 1);
                for (int q = 0; q < p.gate_nsrc; ++q)
                  wait_geq(p.gate + size_t(p.gate_src[q]) * p.gate_stride + rg, p.gate_tgt[q] * u, timeout_ns,
                           status);
              }
              if (timed) wt[0] += globaltimer() - t0;
              fence_proxy_async();
              pst[i].rdy = rg + 1;
            }
          }
          issue(P, ps[i], pst[i], i, t);
          issued = true;
          force = false;
        }
        if (!issued && live) force = true;
      }
      mbar_wait(P.empty + P.stage, P.phase ^ 1u);  // END marker
      info[P.first + P.stage].pass = kEndPass;
      mbar_arrive(P.full + P.stage);
      P.advance();
      return;
    }
    // consumers: everything they need travels in info[]; the pass table is
    // only read by the producer lane
    while (true) {
      const unsigned long long t0 = tnow();
      mbar_wait(P.full + P.stage, P.phase);
      if (timed) wt[2] += globaltimer() - t0;
      const TileInfo ti = info[P.first + P.stage];
      if (ti.pass == kEndPass) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(P.empty + P.stage);
        P.advance();
        break;
      }
      consume(int(ti.pass), buf + size_t(P.first + P.stage) * kStageBytes, size_t(ti.e0), size_t(ti.units),
              int(ti.T));
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(P.empty + P.stage);
      P.advance();
    }
  }

  // producer lane: load tile t of pass p (index i) into the next stage
  __device__ __forceinline__ void issue(Pipe& P, const PassDesc& p, const ProdPass& q, int i, unsigned long long t) {
    const unsigned long long left = q.nun - t * q.T;
    const unsigned units = left < q.T ? unsigned(left) : q.T;
    const unsigned long long u = q.u0 + t * q.T;
    const int nsrc = p.nsrc, eb = p.eb;
    const unsigned long long t0 = tnow();
    mbar_wait(P.empty + P.stage, P.phase ^ 1u);
    if (timed) wt[1] += globaltimer() - t0;
    info[P.first + P.stage] = TileInfo{16ull * u, units, static_cast<unsigned short>(i), static_cast<unsigned short>(q.T)};
    const unsigned bytes = units * 16u * unsigned(eb);
    mbar_expect_tx(P.full + P.stage, bytes * unsigned(nsrc));
    uint8_t* dst = buf + size_t(P.first + P.stage) * kStageBytes;
    const unsigned long long off = 16ull * unsigned(eb) * u;
    for (int s = 0; s < nsrc; ++s) bulk_g2s(dst + size_t(s) * q.tbytes, p.base[s] + off, bytes, P.full + P.stage);
    P.advance();
  }

  // Kernel epilogue (all threads): the last CTA resets the dynamic tile
  // counters for the next launch on this workspace.
  __device__ void finish(unsigned* end_ctr) {
    __syncthreads();
    if (threadIdx.x == 0) fail_epilogue(status);
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
