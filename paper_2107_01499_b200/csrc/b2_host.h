// b2_host.h -- host-side helpers shared by the translation units of libb2comm.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "b2comm.h"

namespace b2 {

void set_error(const char* fmt, ...);

#define B2_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::b2::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),    \
                      __FILE__, __LINE__);                                       \
      return B2_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

#define B2_REQUIRE(cond, ...)         \
  do {                                \
    if (!(cond)) {                    \
      ::b2::set_error(__VA_ARGS__);   \
      return B2_ERR_INVALID;          \
    }                                 \
  } while (0)

// Persistent-grid size for a kernel: SMs x resident CTAs per SM.
int persistent_grid(const void* func, int threads, size_t smem = 0);
int sm_count();
// A persistent grid restricted to an SM budget (sms > 0): whole CTAs-per-SM
// multiples of at most `sms` SMs.
inline int budget_grid(int grid, int sms) {
  const int per_sm = grid / (sm_count() > 0 ? sm_count() : 1);
  return sms > 0 && sms < sm_count() ? sms * (per_sm > 0 ? per_sm : 1) : grid;
}
// Resident CTAs per SM of `func` at `threads` threads (cached per device).
int occupancy(const void* func, int threads, size_t smem = 0);
// Opt a ring kernel into the 192 KB dynamic shared memory (once per device).
cudaError_t ensure_ring_smem(const void* fn);

}  // namespace b2
