// Shared helpers for the sm_100a kernels of libssmquant_sm100.so.
// Numerics follow the oracle contract (oracle/qblock.py header): IEEE f32 division,
// round-half-to-even, explicit __fmul_rn/__fadd_rn where the oracle's op order is
// the parity contract (no FMA contraction there).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/ssmquant_sm100.h"

namespace sq {

void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define SQ_REQUIRE(cond, code, ...)        \
  do {                                     \
    if (!(cond)) {                         \
      ::sq::set_error(__VA_ARGS__);        \
      return (code);                       \
    }                                      \
  } while (0)

__device__ __forceinline__ int8_t quant8(float v, float s) {
  float q = rintf(__fdiv_rn(v, s));
  q = fminf(fmaxf(q, -128.f), 127.f);
  return (int8_t)q;
}

__device__ __forceinline__ float silu_f(float v) {
  return __fdiv_rn(v, __fadd_rn(1.0f, expf(-v)));
}

// LEDGER G14: log1p(exp(x)), identity above 20.
__device__ __forceinline__ float softplus_f(float v) {
  return v > 20.f ? v : log1pf(expf(v));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace sq
