// Shared device helpers: error plumbing for the C ABI and the reference's
// counter-based RNG restated for the device.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "gosh_b200.h"

// Exported C-ABI entry points (the library is built -fvisibility=hidden).
#define GB_API extern "C" __attribute__((visibility("default")))

namespace gb {

void set_error(const char *fmt, ...);

#define GB_CUDA_TRY(expr)                                                    \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) {                                                 \
      ::gb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                      cudaGetErrorString(_e));                               \
      return GB_E_CUDA;                                                      \
    }                                                                        \
  } while (0)

#define GB_CHECK_LAUNCH() GB_CUDA_TRY(cudaGetLastError())

#define GB_REQUIRE(cond, ...)                                                \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ::gb::set_error(__VA_ARGS__);                                          \
      return GB_E_INVALID;                                                   \
    }                                                                        \
  } while (0)

inline cudaStream_t as_stream(void *h) { return reinterpret_cast<cudaStream_t>(h); }

int num_sms();

// ---------------------------------------------------------------------------
// RNG: splitmix64 streams of _rng.py:14-49.  All arithmetic mod 2^64; the
// draw_below conversion is (int64)(f64(x>>11) * 2^-53 * f64(n)) with
// round-to-nearest multiplies, exactly as numba evaluates _rng.py:46-49.
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // _rng.py:14
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;    // _rng.py:15
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;    // _rng.py:16

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += kGolden;
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream,
                                                        uint64_t step, uint64_t vertex) {
  uint64_t h = mix64(seed ^ (stream * kGolden));
  h = mix64(h ^ step);
  return mix64(h ^ vertex);
}

__host__ __device__ __forceinline__ uint64_t draw_u64(uint64_t key, uint64_t ctr) {
  return mix64(key ^ (ctr * kMix1));
}

__device__ __forceinline__ double draw_unit(uint64_t key, uint64_t ctr) {
  return __dmul_rn(__ull2double_rn(draw_u64(key, ctr) >> 11), 1.0 / 9007199254740992.0);
}

__device__ __forceinline__ int64_t draw_below(uint64_t key, uint64_t ctr, int64_t n) {
  return (int64_t)__dmul_rn(draw_unit(key, ctr), __ll2double_rn(n));
}

}  // namespace gb
