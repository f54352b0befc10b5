/*
 * rcomm_oracle.h -- CPU restatement of the rcomm hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2107_01499_b200/,
 * include/) may link or call this; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg use it, and only as the checker.
 *
 * Every function restates one reference routine (file:line under
 * /root/reference/proj) with the reference's exact float semantics:
 * no FMA, IEEE division, round-half-even, fp64 accumulation in ascending
 * rank order starting from +0.0.
 *
 * Parity pinning: the restatement is checked against the reference's own
 * known-answer tests (tests/golden/kats.json, transcribed with file:line) and
 * against the compiled reference (oracle/_ref/librcomm_ref.so, built from the
 * sources in place by oracle/Makefile) through the fixtures in tests/golden/.
 */
#ifndef RCOMM_ORACLE_H
#define RCOMM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_NONFINITE = -1, ORC_ERR_SIZE = -2 };
enum { ORC_CODEC_IDENTITY = 0, ORC_CODEC_UNIFORM8 = 1, ORC_CODEC_ONEBIT = 2 };
enum { ORC_REDUCE_SUM = 0, ORC_REDUCE_AVERAGE = 1 };

/* collectives.cpp:167-175 */
void orc_partition_range(size_t len, int n, int k, size_t* lo, size_t* sz);

/* kernels.cpp:34-41 (n > 0) */
void orc_minmax(const float* x, size_t n, float* lo, float* hi);
/* kernels.cpp:43-50 */
void orc_quantize_u8(const float* x, uint8_t* out, float min, float inv_step, size_t n);
/* kernels.cpp:52-56 */
void orc_dequantize_u8(const uint8_t* in, float* out, float min, float step, size_t n);

/* codec.cpp:24-27,40-80 (uniform8, nearest).  Returns ORC_ERR_NONFINITE where
 * the reference throws "encode: non-finite input value". */
int orc_u8_encode(const float* x, size_t n, float* lo, float* hi, uint8_t* codes);
/* codec.cpp:81-88 (onebit) with the scalar kernels (kernels.cpp:26-32,
 * 58-63): scale = (float)(sequential fp64 sum of |x|) / (float)n; wire =
 * [scale f32][ceil(n/8) bytes, bit k (LE) = !signbit(x[k])].  Returns
 * ORC_ERR_NONFINITE where the reference throws. */
/* hierarchical_c, collectives.cpp:290-385 (no error feedback); nodes[r] =
 * node of rank r (<= 64 ranks). */
int orc_hierarchical_c(int g, size_t len, float* const* xs, const int* nodes, int codec);

int orc_onebit_encode_wire(const float* x, size_t n, uint8_t* wire);
/* codec.cpp:110-114, kernels.cpp:65-69 */
void orc_onebit_decode_wire(const uint8_t* wire, size_t n, float* out);
/* codec.cpp:93-109 (uniform8) */
void orc_u8_decode(float lo, float hi, const uint8_t* codes, size_t n, float* out);
/* codec.cpp:31-38 + 58-59: exact wire bytes [min f32][max f32][u8 x n] */
int orc_u8_encode_wire(const float* x, size_t n, uint8_t* wire);
/* codec.cpp:125-137 with the uniform8 codec: y = x - delta; P = Q(y);
 * d = D(P); delta = y - d.  decoded may be NULL. */
int orc_u8_compensate_encode(const float* x, float* delta, size_t n, float* lo,
                             float* hi, uint8_t* codes, float* decoded);

/* c_fp_s -> scatter_reduce_fp, collectives.cpp:42-87 / 215-220, restated over
 * all g ranks' buffers at once (xs[r] is rank r's bucket, updated in place). */
void orc_c_fp_s(int g, size_t len, float* const* xs);

/* c_lp_s -> scatter_reduce_lp, collectives.cpp:91-163 / 222-227, restated
 * partition by partition.  codec: ORC_CODEC_IDENTITY, ORC_CODEC_UNIFORM8 or ORC_CODEC_ONEBIT.
 * deltas/eps NULL = stateless; else deltas[r] has len floats and eps[r] has
 * owned_partition_len(len, g, r) floats (ErrorState, codec.hpp:40-47). */
int orc_c_lp_s(int g, size_t len, float* const* xs, int codec,
               float* const* deltas, float* const* eps);

/* d_fp_s for one rank, collectives.cpp:229-258.  nbr_x[i] = x of the i-th
 * entry of the sorted, self-inclusive neighbour list; out may alias self. */
void orc_d_fp_s_rank(size_t len, const float* const* nbr_x, int nnb, int mode,
                     float* out);
/* d_lp_s for one rank, collectives.cpp:260-288: every term, self included,
 * is D(Q(x_j)) over the whole bucket. */
int orc_d_lp_s_rank(size_t len, const float* const* nbr_x, int nnb, int codec,
                    int mode, float* out);

/* ring / full neighbour sets, collectives.cpp:181-193 (random needs
 * libstdc++'s std::shuffle and is served by the product's host layer). */
int orc_topology_neighbors(int kind_ring1_full2, int n, int rank, int* out);

/* Deterministic synthetic gradient: splitmix64 counter hash
 * -> 24-bit value -> uniform in [-1, 1).  Identical formula in the CUDA
 * generator (csrc/synth.cu) so host and device inputs are bit-identical. */
void orc_synth(float* x, size_t n, uint64_t seed, uint64_t offset);

#ifdef __cplusplus
}
#endif
#endif
