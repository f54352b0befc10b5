/*
 * rcomm_oracle.c -- CPU restatement of the rcomm hot path (TEST INFRASTRUCTURE).
 *
 * See rcomm_oracle.h.  Compiled with -O2 -ffp-contract=off and without
 * -ffast-math so that every float expression rounds exactly as the reference
 * (g++ -O2, SSE2/AVX2, no FMA) rounds it.  File:line citations refer to
 * /root/reference/proj.
 */
#include "rcomm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* collectives.cpp:167-175 */
void orc_partition_range(size_t len, int n, int k, size_t* lo, size_t* sz) {
  const size_t base = len / (size_t)n;
  const size_t extra = len % (size_t)n;
  const size_t uk = (size_t)k;
  *lo = uk * base + (uk < extra ? uk : extra);
  *sz = base + (uk < extra ? 1 : 0);
}

/* kernels.cpp:34-41 (scalar backend; AVX2 differs only on +-0 ties) */
void orc_minmax(const float* x, size_t n, float* lo, float* hi) {
  float l = x[0], h = x[0];
  for (size_t k = 1; k < n; ++k) {
    l = x[k] < l ? x[k] : l;
    h = x[k] > h ? x[k] : h;
  }
  *lo = l;
  *hi = h;
}

/* kernels.cpp:43-50: nearbyintf under the default (round-half-even) mode,
 * clamp in float, then convert.  NaN survives the clamp; the x86 conversion
 * of NaN yields 0x80000000 whose low byte is 0 -- spelled out here. */
void orc_quantize_u8(const float* x, uint8_t* out, float min, float inv_step, size_t n) {
  for (size_t k = 0; k < n; ++k) {
    float q = nearbyintf((x[k] - min) * inv_step);
    q = q < 0.0f ? 0.0f : (q > 255.0f ? 255.0f : q);
    out[k] = isnan(q) ? (uint8_t)0 : (uint8_t)q;
  }
}

/* kernels.cpp:52-56: rounded multiply, then rounded add (no FMA) */
void orc_dequantize_u8(const uint8_t* in, float* out, float min, float step, size_t n) {
  for (size_t k = 0; k < n; ++k) {
    const float p = (float)in[k] * step; /* rounded product (no contraction) */
    out[k] = min + p;
  }
}

static int all_finite(const float* x, size_t n) { /* codec.cpp:24-27 */
  for (size_t k = 0; k < n; ++k)
    if (!isfinite(x[k])) return 0;
  return 1;
}

/* codec.cpp:40-80, uniform8 + nearest */
int orc_u8_encode(const float* x, size_t n, float* lo_out, float* hi_out, uint8_t* codes) {
  if (!all_finite(x, n)) return ORC_ERR_NONFINITE;
  float lo = 0.0f, hi = 0.0f;
  if (n) orc_minmax(x, n, &lo, &hi);
  *lo_out = lo;
  *hi_out = hi;
  const float range = hi - lo;
  if (range == 0.0f) {
    if (n) memset(codes, 0, n); /* degenerate range: all codes 0 (codec.cpp:62-64) */
  } else {
    orc_quantize_u8(x, codes, lo, 255.0f / range, n);
  }
  return ORC_OK;
}

/* codec.cpp:93-109, uniform8 */
void orc_u8_decode(float lo, float hi, const uint8_t* codes, size_t n, float* out) {
  const float step = (hi - lo) / 255.0f;
  orc_dequantize_u8(codes, out, lo, step, n);
}

/* codec.cpp:31-38, 58-59: [lo f32 LE][hi f32 LE][codes] */
int orc_u8_encode_wire(const float* x, size_t n, uint8_t* wire) {
  float lo, hi;
  int rc = orc_u8_encode(x, n, &lo, &hi, wire + 8);
  if (rc) return rc;
  memcpy(wire, &lo, 4);
  memcpy(wire + 4, &hi, 4);
  return ORC_OK;
}

/* codec.cpp:125-137 */
int orc_u8_compensate_encode(const float* x, float* delta, size_t n, float* lo,
                             float* hi, uint8_t* codes, float* decoded) {
  float* y = (float*)malloc((n ? n : 1) * sizeof(float));
  float* d = (float*)malloc((n ? n : 1) * sizeof(float));
  for (size_t k = 0; k < n; ++k) y[k] = x[k] - delta[k];
  int rc = orc_u8_encode(y, n, lo, hi, codes);
  if (rc == ORC_OK) {
    orc_u8_decode(*lo, *hi, codes, n, d);
    for (size_t k = 0; k < n; ++k) delta[k] = y[k] - d[k];
    if (decoded) memcpy(decoded, d, n * sizeof(float));
  }
  free(y);
  free(d);
  return rc;
}

/* scatter_reduce_fp, collectives.cpp:42-87.  g == 1 returns x untouched
 * (collectives.cpp:49).  Owner k folds every rank's partition k in ascending
 * rank order into a +0.0-initialised double and rounds once; every rank then
 * holds the owner's float result. */
void orc_c_fp_s(int g, size_t len, float* const* xs) {
  if (g == 1) return;
  for (int k = 0; k < g; ++k) {
    size_t lo, sz;
    orc_partition_range(len, g, k, &lo, &sz);
    for (size_t e = lo; e < lo + sz; ++e) {
      double acc = 0.0;
      for (int j = 0; j < g; ++j) acc += (double)xs[j][e];
      const float r = (float)acc;
      for (int j = 0; j < g; ++j) xs[j][e] = r;
    }
  }
}

/* Identity codec: encode checks finiteness and copies (codec.cpp:41,47-50);
 * decode copies.  Used for the identity-collapse restatement. */
static int enc_dec(int codec, const float* x, size_t n, float* out) {
  if (codec == ORC_CODEC_IDENTITY) {
    if (!all_finite(x, n)) return ORC_ERR_NONFINITE;
    memcpy(out, x, n * sizeof(float));
    return ORC_OK;
  }
  if (codec == ORC_CODEC_ONEBIT) { /* codec.cpp:81-88, 110-114 */
    uint8_t* w = (uint8_t*)malloc(4 + (n + 7) / 8);
    int rc = orc_onebit_encode_wire(x, n, w);
    if (rc == ORC_OK) orc_onebit_decode_wire(w, n, out);
    free(w);
    return rc;
  }
  uint8_t* c = (uint8_t*)malloc(n ? n : 1);
  float lo, hi;
  int rc = orc_u8_encode(x, n, &lo, &hi, c);
  if (rc == ORC_OK) orc_u8_decode(lo, hi, c, n, out);
  free(c);
  return rc;
}

/* scatter_reduce_lp, collectives.cpp:91-163.  Partition k's final value on
 * every rank is D(Q2((float)sum_j D(Q1(x_j|k - delta_j|k)) - eps_k)); the
 * residuals follow compensate_encode (codec.cpp:125-137). */
int orc_c_lp_s(int g, size_t len, float* const* xs, int codec,
               float* const* deltas, float* const* eps) {
  int rc = ORC_OK;
  for (int k = 0; k < g && rc == ORC_OK; ++k) {
    size_t lo, sz;
    orc_partition_range(len, g, k, &lo, &sz);
    double* acc = (double*)calloc(sz ? sz : 1, sizeof(double));
    float* y = (float*)malloc((sz ? sz : 1) * sizeof(float));
    float* d = (float*)malloc((sz ? sz : 1) * sizeof(float));
    for (int j = 0; j < g && rc == ORC_OK; ++j) {
      for (size_t e = 0; e < sz; ++e)
        y[e] = deltas ? xs[j][lo + e] - deltas[j][lo + e] : xs[j][lo + e];
      rc = enc_dec(codec, y, sz, d);
      if (rc) break;
      for (size_t e = 0; e < sz; ++e) {
        if (deltas) deltas[j][lo + e] = y[e] - d[e];
        acc[e] += (double)d[e]; /* kernels.cpp:14-16, ranks ascending */
      }
    }
    if (rc == ORC_OK) {
      for (size_t e = 0; e < sz; ++e) {
        const float s = (float)acc[e];
        y[e] = eps ? s - eps[k][e] : s;
      }
      rc = enc_dec(codec, y, sz, d);
      if (rc == ORC_OK) {
        for (size_t e = 0; e < sz; ++e) {
          if (eps) eps[k][e] = y[e] - d[e];
          for (int j = 0; j < g; ++j) xs[j][lo + e] = d[e];
        }
      }
    }
    free(acc);
    free(y);
    free(d);
  }
  return rc;
}

/* hierarchical_c, collectives.cpp:290-385 (no error feedback).  nodes[r] is
 * rank r's node; members of a node ascending, leader = lowest member. */
int orc_hierarchical_c(int g, size_t len, float* const* xs, const int* nodes, int codec) {
  int node_ids[64], L = 0, rc = ORC_OK;
  for (int r = 0; r < g; ++r) { /* distinct nodes, ascending (std::map order, 303-308) */
    int seen = 0;
    for (int i = 0; i < L; ++i) seen |= node_ids[i] == nodes[r];
    if (!seen) node_ids[L++] = nodes[r];
  }
  for (int i = 1; i < L; ++i) /* insertion sort */
    for (int j = i; j > 0 && node_ids[j - 1] > node_ids[j]; --j) {
      int t = node_ids[j]; node_ids[j] = node_ids[j - 1]; node_ids[j - 1] = t;
    }
  double* acc = (double*)calloc((size_t)L * (len ? len : 1), sizeof(double));
  int leaders[64];
  for (int i = 0; i < L; ++i) {
    double* a = acc + (size_t)i * len;
    leaders[i] = -1;
    for (int r = 0; r < g; ++r) /* members in rank order (322-334) */
      if (nodes[r] == node_ids[i]) {
        if (leaders[i] < 0) leaders[i] = r;
        for (size_t e = 0; e < len; ++e) a[e] += (double)xs[r][e];
      }
  }
  /* leaders sorted ascending by rank (308) */
  for (int i = 1; i < L; ++i)
    for (int j = i; j > 0 && leaders[j - 1] > leaders[j]; --j) {
      int t = leaders[j]; leaders[j] = leaders[j - 1]; leaders[j - 1] = t;
      for (size_t e = 0; e < len; ++e) {
        double d = acc[(size_t)j * len + e];
        acc[(size_t)j * len + e] = acc[(size_t)(j - 1) * len + e];
        acc[(size_t)(j - 1) * len + e] = d;
      }
    }
  if (L > 1 && codec == ORC_CODEC_IDENTITY) {
    /* fp64 partials: owner k's part = its own acc, then the other leaders'
     * in leader order (350-357); every leader ends with all parts (360-372) */
    double* fin = (double*)malloc((len ? len : 1) * sizeof(double));
    for (int k = 0; k < L; ++k) {
      size_t lo, m;
      orc_partition_range(len, L, k, &lo, &m);
      for (size_t e = 0; e < m; ++e) {
        double part = acc[(size_t)k * len + lo + e];
        for (int j = 0; j < L; ++j)
          if (j != k) part += acc[(size_t)j * len + lo + e];
        fin[lo + e] = part;
      }
    }
    for (int i = 0; i < L; ++i)
      for (size_t e = 0; e < len; ++e) xs[leaders[i]][e] = (float)fin[e];
    free(fin);
  } else {
    for (int i = 0; i < L; ++i)
      for (size_t e = 0; e < len; ++e) xs[leaders[i]][e] = (float)acc[(size_t)i * len + e];
    if (L > 1) { /* scatter_reduce_lp over the leader group (375) */
      float* lx[64];
      for (int i = 0; i < L; ++i) lx[i] = xs[leaders[i]];
      rc = orc_c_lp_s(L, len, lx, codec, NULL, NULL);
    }
  }
  /* leaders send x down to their members (382-383) */
  for (int r = 0; r < g; ++r) {
    int lead = -1;
    for (int i = 0; i < L && lead < 0; ++i)
      if (nodes[leaders[i]] == nodes[r]) lead = leaders[i];
    if (lead != r) memcpy(xs[r], xs[lead], len * sizeof(float));
  }
  free(acc);
  return rc;
}

/* d_fp_s, collectives.cpp:229-258 (one rank) */
void orc_d_fp_s_rank(size_t len, const float* const* nbr_x, int nnb, int mode,
                     float* out) {
  const double inv = mode == ORC_REDUCE_AVERAGE ? 1.0 / (double)nnb : 1.0;
  for (size_t e = 0; e < len; ++e) {
    double acc = 0.0;
    for (int i = 0; i < nnb; ++i) acc += (double)nbr_x[i][e];
    out[e] = (float)(acc * inv);
  }
}

/* d_lp_s, collectives.cpp:260-288 (one rank) */
int orc_d_lp_s_rank(size_t len, const float* const* nbr_x, int nnb, int codec,
                    int mode, float* out) {
  const double inv = mode == ORC_REDUCE_AVERAGE ? 1.0 / (double)nnb : 1.0;
  double* acc = (double*)calloc(len ? len : 1, sizeof(double));
  float* d = (float*)malloc((len ? len : 1) * sizeof(float));
  int rc = ORC_OK;
  for (int i = 0; i < nnb && rc == ORC_OK; ++i) {
    rc = enc_dec(codec, nbr_x[i], len, d);
    if (rc == ORC_OK)
      for (size_t e = 0; e < len; ++e) acc[e] += (double)d[e];
  }
  if (rc == ORC_OK)
    for (size_t e = 0; e < len; ++e) out[e] = (float)(acc[e] * inv);
  free(acc);
  free(d);
  return rc;
}

static int cmp_int(const void* a, const void* b) {
  return *(const int*)a - *(const int*)b;
}

/* collectives.cpp:181-193 */
int orc_topology_neighbors(int kind_ring1_full2, int n, int rank, int* out) {
  if (rank < 0 || rank >= n) return ORC_ERR_SIZE;
  if (kind_ring1_full2 == 2) {
    for (int i = 0; i < n; ++i) out[i] = i;
    return n;
  }
  int v[3] = {(rank + n - 1) % n, rank, (rank + 1) % n};
  qsort(v, 3, sizeof(int), cmp_int);
  int m = 0;
  for (int i = 0; i < 3; ++i)
    if (m == 0 || out[m - 1] != v[i]) out[m++] = v[i];
  return m;
}

static uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void orc_synth(float* x, size_t n, uint64_t seed, uint64_t offset) {
  const uint64_t key = splitmix64(seed);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t h = splitmix64(key + offset + i);
    const int32_t m = (int32_t)(h >> 40); /* 24 bits */
    x[i] = (float)(m - 8388608) * 1.1920928955078125e-07f;
  }
}

/* ------------------------------------------------------------- onebit */
/* codec.cpp:81-88 + kernels.cpp:26-32 (sum_abs, scalar: sequential fp64) and
 * 58-63 (sign_pack) */
int orc_onebit_encode_wire(const float* x, size_t n, uint8_t* wire) {
  for (size_t k = 0; k < n; ++k)
    if (!isfinite(x[k])) return ORC_ERR_NONFINITE; /* codec.cpp:24-27 */
  double s = 0.0;
  for (size_t k = 0; k < n; ++k) s += fabs((double)x[k]);
  const float scale = n ? (float)s / (float)n : 0.0f;
  memcpy(wire, &scale, 4);
  const size_t nbytes = (n + 7) / 8;
  for (size_t b = 0; b < nbytes; ++b) wire[4 + b] = 0;
  for (size_t k = 0; k < n; ++k)
    if (!signbit(x[k])) wire[4 + k / 8] |= (uint8_t)(1u << (k % 8));
  return 0;
}

/* codec.cpp:110-114, kernels.cpp:65-69 (sign_unpack) */
void orc_onebit_decode_wire(const uint8_t* wire, size_t n, float* out) {
  float scale;
  memcpy(&scale, wire, 4);
  for (size_t k = 0; k < n; ++k) out[k] = ((wire[4 + k / 8] >> (k % 8)) & 1u) ? scale : -scale;
}
