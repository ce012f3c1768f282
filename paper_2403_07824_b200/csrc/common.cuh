// common.cuh — shared device helpers for the vqpc kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "vqpc.h"

#define VQPC_FULL_MASK 0xffffffffu

// Device-side bounds and invariant checks of the check build (-DVQPC_CHECKS,
// tools/checks_build.sh): a violated condition prints its location and traps, so
// the test that triggered it fails loudly. Compiled out of the product build. (The
// pool's compute-sanitizer is disabled; this build is the memory-safety evidence.)
#ifdef VQPC_CHECKS
#include <cstdio>
#define VQPC_DCHECK(cond)                                                                     \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("VQPC_DCHECK failed at %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                    \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define VQPC_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

namespace vqpc {

// double shuffles (two 32-bit SHFLs each)
__device__ __forceinline__ double shfl_down(double v, int off) {
  return __shfl_down_sync(VQPC_FULL_MASK, v, off);
}
__device__ __forceinline__ double shfl_up(double v, int off) {
  return __shfl_up_sync(VQPC_FULL_MASK, v, off);
}
__device__ __forceinline__ double shfl_xor(double v, int off) {
  return __shfl_xor_sync(VQPC_FULL_MASK, v, off);
}

// Butterfly all-reduce: every lane ends with bit-identical sums (IEEE addition
// is commutative, so partner lanes compute the same value at every level).
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += shfl_xor(v, off);
  return v;
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace vqpc
