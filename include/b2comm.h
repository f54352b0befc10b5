/*
 * b2comm.h -- C ABI of the B200-native rcomm hot path (libb2comm.so).
 *
 * Drop-in boundary for rcomm's communication primitives
 * (/root/reference/proj/include/rcomm/collectives.hpp:50-87), the uniform8
 * ("MinMaxUInt8") codec (codec.hpp:13-54) and bucket flattening
 * (tensor.hpp:56-86).  Every entry point takes plain pointers and sizes; all
 * float/byte buffers are DEVICE pointers on the communicator's GPU unless
 * stated otherwise; `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Semantics are the reference's, bit for bit:
 * uniform8 codes and chunk min/max are bit-exact, fp64 reductions fold ranks
 * in ascending order from +0.0 and round once, no FMA anywhere.
 *
 * Error model: every function returns a b2_status.  Argument errors are
 * detected at the call and reported with a message retrievable through
 * b2_last_error() (thread-local).  Data-dependent errors that the reference
 * raises synchronously (non-finite encode input, codec.cpp:24-27) are found on
 * the device; they are latched in the communicator's status word and returned
 * by b2_comm_sync() (or b2_comm_poll()).  Where the reference would throw
 * rcomm::Error, the C++ wrapper (include/rcomm_b200/) rethrows.
 *
 * Threading / ordering: one host thread (or process) per GPU calls the same
 * primitive with the same bucket id, like one rcomm worker per Endpoint.
 * Completion is stream-ordered; calls on one bucket must be stream-ordered on
 * each rank (the reference's "one collective per tag at a time",
 * SPEC.md:300).  Peer buffers are library-owned windows exchanged once per
 * (bucket, primitive family, size) through the caller-supplied allgather;
 * if any rank fails to allocate one, every rank returns the error (no rank is
 * left blocking in the exchange).
 */
#ifndef B2COMM_H
#define B2COMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define B2COMM_VERSION 1
#define B2_MAX_RANKS 8
/* hdr buffers for the standalone codec hold [min f32][max f32][2 x u32 scratch] */
#define B2_U8_HDR_BYTES 16

typedef enum {
  B2_OK = 0,
  B2_ERR_INVALID = 1,     /* bad argument (size mismatch, null, alignment)   */
  B2_ERR_CUDA = 2,        /* CUDA runtime failure                            */
  B2_ERR_NONFINITE = 3,   /* encode saw NaN/Inf  (codec.cpp:26)              */
  B2_ERR_TIMEOUT = 4,     /* a peer never arrived (rendezvous timeout)       */
  B2_ERR_UNSUPPORTED = 5, /* an unsupported combination                        */
  B2_ERR_BOOTSTRAP = 6    /* the allgather callback failed                   */
} b2_status;

typedef enum { B2_CODEC_IDENTITY = 0, B2_CODEC_UNIFORM8 = 1, B2_CODEC_ONEBIT = 2 } b2_codec_kind;
typedef enum { B2_REDUCE_SUM = 0, B2_REDUCE_AVERAGE = 1 } b2_reduce_mode;
typedef enum { B2_TOPO_RING = 0, B2_TOPO_RANDOM = 1, B2_TOPO_FULL = 2 } b2_topology_kind;

typedef struct b2_comm* b2_comm_t;

/* Bootstrap hook: gather `bytes` from every rank into recv (world * bytes,
 * rank-major).  Called collectively (all ranks, same order) the first time a
 * (bucket, family, size) window is used.  Return 0 on success. */
typedef int (*b2_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);

/* ------------------------------------------------------------------ misc */
int b2_version(void);
const char* b2_last_error(void);
const char* b2_status_string(int status);

/* partition_range (collectives.hpp:42-43 / collectives.cpp:167-175) */
void b2_partition_range(size_t len, int n, int k, size_t* lo, size_t* sz);
/* owned_partition_len (collectives.hpp:87) */
size_t b2_owned_partition_len(size_t len, int world, int idx);
/* Codec::payload_size (codec.hpp:30, codec.cpp:31-38) */
size_t b2_payload_size(int codec, size_t n);
/* Topology::neighbors (collectives.hpp:18-25, collectives.cpp:181-213): sorted,
 * self-inclusive; writes up to n ints into out, returns the count (or -1). */
int b2_topology_neighbors(int kind, int n, uint64_t seed, int rank, uint64_t round, int* out);

/* ------------------------------------------- uniform8 codec (one GPU)
 * Codec::encode / decode (codec.hpp:32-35; codec.cpp:40-80, 93-109) split into
 * SoA device buffers: codes[n] (byte k = level of x[k]) and hdr (>= 16 bytes:
 * hdr[0] = min, hdr[1] = max as f32).  A non-finite input leaves a non-finite
 * value in hdr[0] or hdr[1] (NaN propagates) -- the host wrapper turns that
 * into the reference's Error.  n == 0 writes hdr = (0, 0). */
int b2_u8_encode(const float* x, size_t n, uint8_t* codes, float* hdr, void* stream);
int b2_u8_decode(const uint8_t* codes, const float* hdr, size_t n, float* out, void* stream);
/* Codec{uniform8, Rounding::stochastic}.encode (codec.cpp:67-78): as
 * b2_u8_encode, levels rounded up with probability q - floor(q); the uniform
 * draws come from a counter hash of (seed, element), not mt19937, so only
 * unbiasedness is shared with the reference (test_codec.cpp:175-192).  The
 * collectives take it through b2_c_lp_s_stochastic / b2_d_lp_s_stochastic. */
int b2_u8_encode_stochastic(const float* x, size_t n, uint8_t* codes, float* hdr, uint64_t seed,
                            void* stream);
/* compensate_encode (codec.hpp:49-54, codec.cpp:125-137) with uniform8:
 * y = x - delta; codes,hdr = Q(y); delta = y - D(Q(y)); decoded (nullable) = D(Q(y)) */
int b2_u8_compensate_encode(const float* x, float* delta, size_t n, uint8_t* codes,
                            float* hdr, float* decoded, void* stream);
/* compensate_encode with the identity codec: y = x - delta -> y (the payload
 * floats), delta = y - y; *nonfinite (device int) |= 1 if any y is non-finite
 * (the reference's encode throws, codec.cpp:24-27).  x, delta, y device. */
int b2_identity_compensate_encode(const float* x, float* delta, size_t n, float* y, int* nonfinite,
                                  void* stream);
/* compensate_encode with the onebit codec: decoded := y = x - delta,
 * wire = Q(y) (as b2_onebit_encode), decoded := D(Q(y)), delta = y - D(Q(y)).
 * decoded (n floats, 16-byte aligned) is required: it holds y meanwhile. */
int b2_onebit_compensate_encode(const float* x, float* delta, size_t n, uint8_t* wire, float* decoded,
                                void* stream);
/* Exact reference wire bytes [min f32 LE][max f32 LE][u8 x n] (codec.hpp:21-24)
 * into a device buffer of 8 + n bytes, and back. */
int b2_u8_pack_wire(const uint8_t* codes, const float* hdr, size_t n, uint8_t* wire, void* stream);

/* Codec onebit (codec.cpp:81-88, 110-114): wire = [scale f32][ceil(n/8)
 * bytes], scale = (float)(sum |x| in fp64) / (float)n, bit k (LE) = x[k] is
 * not negative (signbit).  The fp64 sum is deterministic but not in the
 * reference's order: scale is identical whenever that sum is exact and within
 * one float rounding otherwise.  A non-finite input gives a NaN scale (the
 * reference throws).  x, out, wire 16-byte aligned; wire holds 4 + ceil(n/8)
 * bytes rounded up to 4.  (Replaces Codec{onebit}.encode / decode; the
 * primitives below take B2_CODEC_ONEBIT too.) */
int b2_onebit_encode(const float* x, size_t n, uint8_t* wire, void* stream);
int b2_onebit_decode(const uint8_t* wire, size_t n, float* out, void* stream);
int b2_u8_unpack_wire(const uint8_t* wire, size_t n, uint8_t* codes, float* hdr, void* stream);

/* ----------------------------------------------------- bucket arena
 * BucketArena::flatten (tensor.hpp:76-81, tensor.cpp:46-68): concatenate
 * count device tensors (srcs[i], lens[i] floats; pointer/len arrays on the
 * HOST) into arena in registration order with no gaps, in one launch per 64
 * members.  Validation (non-empty list, no zero-length member) mirrors the
 * reference; name uniqueness is checked by the host wrappers.  unflatten
 * copies the arena back out (the reference aliases instead; the wrappers
 * return views and use this only when members must stay separate). */
int b2_bucket_flatten(const float* const* srcs, const size_t* lens, int count, float* arena, void* stream);
int b2_bucket_unflatten(const float* arena, float* const* dsts, const size_t* lens, int count, void* stream);

/* Synthetic gradient: x[i] = splitmix64-hash(seed, offset+i)
 * mapped to [-1, 1) with 24-bit resolution; identical to oracle's orc_synth. */
int b2_fill_synthetic(float* x, size_t n, uint64_t seed, uint64_t offset, void* stream);

/* ---------------------------------------------------- communicator
 * One per (process or thread, GPU).  world <= B2_MAX_RANKS, all ranks on one
 * NVLink/NVSwitch node.  allgather is used only to exchange window handles. */
int b2_comm_create(int world, int rank, int device, b2_allgather_fn allgather, void* user, b2_comm_t* out);
int b2_comm_destroy(b2_comm_t comm);
int b2_comm_rank(b2_comm_t comm);
int b2_comm_world(b2_comm_t comm);
/* Synchronize `stream` and return (and clear) the latched device status. */
int b2_comm_sync(b2_comm_t comm, void* stream);
/* Return (and clear) the latched status without synchronizing. */
int b2_comm_poll(b2_comm_t comm);
/* Rendezvous timeout for device-side waits, in milliseconds (default 600000).
 * A wait that times out latches B2_ERR_TIMEOUT and POISONS the window on every
 * rank (a word in each rank's window header) before this rank publishes
 * anything else; a late rank that consumes anything published after that
 * sees the poison at its kernel end and fails too.  From then on the
 * communicator is poisoned: b2_comm_sync/poll keep returning B2_ERR_TIMEOUT
 * and every primitive is refused with B2_ERR_TIMEOUT until the communicator
 * is destroyed and re-created (there is no way to re-agree the epochs). */
int b2_comm_set_timeout_ms(b2_comm_t comm, uint64_t ms);
/* SM budget of every primitive launch: `sms` persistent CTAs (one per SM)
 * instead of one per SM of the device, leaving the other SMs to compute that
 * runs concurrently (communication overlapping backward, engine.cpp:113-153).
 * 0 = all SMs (default).  Every rank must set the same budget (checked when a
 * window is first exchanged). */
int b2_comm_set_sm_budget(b2_comm_t comm, int sms);
/* 1 when the communicator is poisoned by a rendezvous timeout (see above):
 * its own latched status, or a poison word a peer wrote into one of its
 * windows (read with a small copy on a private non-blocking stream, so it
 * does not wait for kernels still running). */
int b2_comm_poisoned(b2_comm_t comm);
/* Collective (every rank, same bucket id): free every window of `bucket`
 * (all primitive families and sizes).  Drains this GPU, then synchronises the
 * ranks through the bootstrap allgather before unmapping, so no peer kernel
 * can still be reading.  Windows are otherwise kept for the communicator's
 * lifetime (one per (bucket, family, size)). */
int b2_comm_release_bucket(b2_comm_t comm, uint32_t bucket);
/* Device bytes held in peer windows by this communicator. */
size_t b2_comm_window_bytes(b2_comm_t comm);
/* Number of kernel launches this communicator has issued (evidence counter). */
uint64_t b2_comm_launches(b2_comm_t comm);
/* Phase tracing (the multi-GPU stand-in for ncu, which cannot replay kernels
 * that rendezvous across GPUs): when enabled every primitive launch records
 * %globaltimer stamps (ns) per CTA at its phase boundaries; read_trace copies
 * the last launch's stamps, max_ctas x n_slots uint64 (0 = not reached). */
int b2_comm_enable_trace(b2_comm_t comm, int on);
int b2_comm_read_trace(b2_comm_t comm, uint64_t* out, int max_ctas, int* n_slots);

/* --------------------------------------------------- the primitives
 * x: this rank's bucket (device, n floats, 16-byte aligned), updated in place.
 *
 * c_fp_s  (collectives.hpp:51-52; scatter_reduce_fp collectives.cpp:42-87):
 *   every rank ends with (float) sum_j (double) x_j, ranks folded ascending;
 *   world == 1 leaves x untouched.
 * c_lp_s  (collectives.hpp:59-61; scatter_reduce_lp collectives.cpp:91-163):
 *   codec B2_CODEC_UNIFORM8 (ByteGrad), B2_CODEC_ONEBIT (the 1-bit Adam
 *   aggregation, algorithms.cpp:141-148) or B2_CODEC_IDENTITY.  delta/eps both
 *   NULL = stateless; else ErrorState (codec.hpp:40-47): delta has n floats,
 *   eps has owned_partition_len(n, world, rank) floats, both updated.
 *   stochastic rounding: b2_c_lp_s_stochastic below.
 * d_fp_s  (collectives.hpp:64-66; collectives.cpp:229-258)
 * d_lp_s  (collectives.hpp:69-72; collectives.cpp:260-288):
 *   nbrs = Topology::neighbors(rank, round) (sorted, self-inclusive, HOST
 *   array); the neighbour relation must be symmetric, as every rcomm
 *   Topology is.  mode = B2_REDUCE_SUM / B2_REDUCE_AVERAGE.  Any codec.
 * *_stochastic: the uniform8 codec with Rounding::stochastic
 *   (codec.cpp:67-78) in every encode of the primitive (C_LP_S: both
 *   phases): level = floor(q) + (u < q - floor(q)), u from a counter hash of
 *   (seed, rank, phase, element).  `seed` is drawn per call from the caller's
 *   generator by the host wrappers; the draws are not the reference's
 *   mt19937 stream, so only unbiasedness is shared with it. */
int b2_c_fp_s(b2_comm_t comm, float* x, size_t n, uint32_t bucket, void* stream);
int b2_c_lp_s(b2_comm_t comm, float* x, size_t n, int codec, float* delta, size_t delta_len,
              float* eps, size_t eps_len, uint32_t bucket, void* stream);
int b2_d_fp_s(b2_comm_t comm, float* x, size_t n, const int* nbrs, int n_nbrs, int mode,
              uint32_t bucket, void* stream);
/* hierarchical_c (collectives.hpp:80-82, collectives.cpp:290-385) over ONE
 * node -- every rank of the communicator shares the NVLink domain: the
 * reference sums the members in fp64 in ascending rank order from +0.0 and
 * rounds once, with no compression whatever the codec (collectives.cpp:
 * 377-380), which is C_FP_S's fold for two or more ranks and (float)(0.0 +
 * (double)x) for one.  (Node layouts spanning several nodes need an
 * inter-node transport, which this path does not have.) */
int b2_hierarchical_c(b2_comm_t comm, float* x, size_t n, uint32_t bucket, void* stream);
int b2_c_lp_s_stochastic(b2_comm_t comm, float* x, size_t n, float* delta, size_t delta_len, float* eps,
                         size_t eps_len, uint64_t seed, uint32_t bucket, void* stream);
int b2_d_lp_s_stochastic(b2_comm_t comm, float* x, size_t n, const int* nbrs, int n_nbrs, int mode,
                         uint64_t seed, uint32_t bucket, void* stream);
int b2_d_lp_s(b2_comm_t comm, float* x, size_t n, const int* nbrs, int n_nbrs, int codec,
              int mode, uint32_t bucket, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* B2COMM_H */
