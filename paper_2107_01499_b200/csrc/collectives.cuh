// collectives.cuh -- argument blocks and window layout shared by the
// collective kernels (collectives.cu) and the communicator (comm.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include "b2_device.cuh"

namespace b2 {

// Every rank's window for one (bucket, family, size) has the same layout.
// The first 256 bytes are control words; data regions follow, 256-aligned.
struct WinHdr {
  unsigned long long arrive1;   // central: #ranks whose phase-1 chunk for me landed (cumulative)
  unsigned long long ready2;    // central: epoch of my published phase-2 output
  unsigned long long dready[2]; // decentral: epoch of my published buffer, per parity
  unsigned long long dreads[2]; // decentral: #neighbour reads of my buffer completed (cumulative)
  unsigned long long arrive_e;  // central uint8: #ranks whose unaligned head/tail codes for me landed
  unsigned long long poison;    // nonzero: a rank timed out on this window (b2_device.cuh Fail); never cleared
  float2 hdr1[kMaxRanks];       // central uint8: (min,max) of my chunk as encoded by rank j
  float2 hdr2;                  // central uint8: (min,max) of my phase-2 payload
  float2 dhdr[2];               // decentral uint8: (min,max) of my bucket, per parity
};
static_assert(sizeof(WinHdr) <= 256, "window header exceeds 256 bytes");

enum Codec : int { kIdentity = 0, kU8 = 1 };

// Per-CTA phase timestamps (%globaltimer, ns) written by consumer thread 0
// when tracing is enabled -- the multi-GPU replacement for ncu, which cannot
// replay kernels that rendezvous with other GPUs.
constexpr int kTraceSlots = 32;
enum TracePoint : int {
  kTrStart = 0,
  kTrP1FirstA = 1,   // phase 1: first chunk's (min,max) final
  kTrP1FirstB = 2,   // phase 1: first chunk pushed
  kTrP1Done = 3,     // phase 1: all chunks pushed (g==1: pass B done)
  kTrP2Ready = 4,    // phase 2: all contributions arrived
  kTrP2A = 5,        // phase 2: second (min,max) final
  kTrP2Done = 6,     // phase 2: payload published
  kTrP3First = 7,    // phase 3: first owner's payload ready
  kTrEnd = 8,
  kTrP2Pass = 9,     // phase 2: second pass done, before the publication fence
  kTrP1Step = 10,    // 10..17: phase-1 step i (chunk me+1+i) pushed, before its fence
  kTrP1Fenced = 18,  // 18..25: phase-1 step i fenced and signalled
  kTrWait = 26,      // 26..31: accumulated ns (not stamps) -- Ring::wt[] of the traced stream
};

// Centralized ScatterReduce (C_FP_S, C_LP_S).
struct CentralArgs {
  float* x;
  size_t n;
  int g, me;
  int check_finite;             // identity c_lp_s: encode validates (codec.cpp:41)
  unsigned long long epoch;     // 1-based call counter of this window
  float* delta;                 // ErrorState::delta (n) or null
  float* eps;                   // ErrorState::epsilon (owned len) or null
  uint8_t* win[kMaxRanks];      // every rank's window base (peer-mapped; win[me] local)
  size_t off_gate, off_recv1, slot_stride, off_out2;
  // staggered C_LP_S (central_stag.cu): per-source arrival counters of my
  // chunk [g][sgate_stride], my out2 publication counters, landing slots
  size_t off_sgate, sgate_stride, off_qgate, off_land;
  size_t off_sgate2;            // small_central.cu: per-source out2 publication counters [g][sgate_stride]
  float2* partials;             // local workspace [(kMaxRanks + 1) * grid]
  unsigned* cta_done;           // local workspace [kMaxRanks + 2]
  unsigned* gridbar;            // local workspace [2]: consumer grid barrier
  unsigned long long* sched;    // local workspace [kSchedPasses]: dynamic tile counters, or null
  unsigned* sched_end;          // local workspace: CTAs finished (counter reset)
  Fail* status;                 // failure context of this window (b2_device.cuh)
  unsigned long long timeout_ns;
  unsigned long long* trace;    // [grid * kTraceSlots] globaltimer stamps, or null
  int sr_on;                    // stochastic rounding (uint8), b2_c_lp_s_stochastic
  unsigned long long sr_seed;   // per-call seed drawn from the caller's generator
};

// Dynamic tile counters per window: one per pass of a launch (C_*: at most
// 3g+2 passes, D_*: 3), reset by the last CTA of every launch.
constexpr int kSchedPasses = 64;

// C_LP_S with the onebit codec (onebit_coll.cu).  Own window family: slot j
// of recv1 = rank j's payload of my chunk, out2 = my phase-2 payload; every
// payload is [scale f32 | 12 B pad][sign words] so the words are 16-aligned.
struct OnebitArgs {
  float* x;
  size_t n;
  int g, me;
  unsigned long long epoch;     // 1-based call counter of this window
  float* delta;                 // ErrorState::delta (n) or null
  float* eps;                   // ErrorState::epsilon (owned len) or null
  uint8_t* win[kMaxRanks];
  size_t off_recv1, slot_stride, off_out2;
  double* partials;             // local workspace [(g + 1) * grid] fp64 |y| partial sums
  Fail* status;
  unsigned long long timeout_ns;
};

// D_LP_S with the onebit codec (onebit_coll.cu).  Pull design: every rank
// encodes its bucket into its own window (dbuf[parity]) and publishes
// dready[parity] = epoch; neighbours read it over NVLink and count their
// reads in dreads[parity], which the owner waits on before it overwrites
// that parity two calls later.
struct OnebitDecentArgs {
  float* x;
  size_t n;
  int me, nnb;
  int nbrs[kMaxRanks];          // sorted, self-inclusive
  int parity;
  unsigned long long epoch;
  unsigned long long expected_reads;  // dreads[parity] must reach this before we overwrite
  double inv;                   // 1/|N| (average) or 1.0 (sum), collectives.cpp:282-284
  uint8_t* win[kMaxRanks];
  size_t off_dbuf;              // offset of dbuf[parity]
  double* partials;             // local workspace [grid]
  Fail* status;
  unsigned long long timeout_ns;
};

// Per-source decode constants of the small-bucket D_* kernel (small_coll.cu).
struct SrcDecS {
  float lo, step, c23;
  int fast;
};
// Buckets up to this many elements try the register-resident D_* kernel
// (small_coll.cu) before the TMA ring; its per-CTA counters need
// gate_stride > kSmallMaxGridD.
constexpr size_t kSmallDecentMax = 16000000;
constexpr size_t kSmallMaxGridD = 1024;
// C_* buckets up to this many elements try the register-resident kernel
// (small_central.cu); windows that may take it carry its two per-CTA counter
// arrays [g][kSmallMaxGridD].  kSmallCentralWin bounds the windows that
// reserve them (B2_SMALL_C_MAX cannot raise the cut-over above it).
constexpr size_t kSmallCentralMax = 4000000;
constexpr size_t kSmallCentralWin = 16000000;

// Decentralized neighbourhood reduce (D_FP_S, D_LP_S).
struct DecentArgs {
  float* x;
  size_t n;
  int me, nnb;
  int nbrs[kMaxRanks];          // sorted, self-inclusive
  int check_finite;
  int parity;
  unsigned long long epoch;
  unsigned long long expected_reads;  // dreads[parity] must reach this before we overwrite
  double inv;                   // 1/|N| (average) or 1.0 (sum), collectives.cpp:252-254
  uint8_t* win[kMaxRanks];
  size_t off_dbuf;              // offset of dbuf[parity]
  size_t off_gate;              // arrival counters [source rank][region + tail], cumulative units (tail: calls)
  size_t gate_stride;           // counters per source
  unsigned long long sends[kMaxRanks];  // per neighbour i: calls so far in which nbrs[i] sent to me (incl. this one)
  float2* partials;
  unsigned* cta_done;
  unsigned* gridbar;
  unsigned long long* sched;
  unsigned* sched_end;
  Fail* status;
  unsigned long long timeout_ns;
  unsigned long long* trace;
  int sr_on;                    // stochastic rounding (uint8), b2_d_lp_s_stochastic
  unsigned long long sr_seed;
};

}  // namespace b2
