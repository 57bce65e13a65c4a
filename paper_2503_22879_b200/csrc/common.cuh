// Shared helpers for the sm_100a kernels of libssmquant_sm100.so.
// Numerics follow the oracle contract (oracle/qblock.py header): IEEE f32 division,
// round-half-to-even, explicit __fmul_rn/__fadd_rn where the oracle's op order is
// the parity contract (no FMA contraction there).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>

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

// SiLU with a rounded reciprocal instead of the IEEE division (<= 2 ulp from silu_f).
__device__ __forceinline__ float silu_fast(float v) {
  return __fmul_rn(v, __frcp_rn(__fadd_rn(1.0f, expf(-v))));
}

// SiLU with the hardware exp2 / reciprocal approximations (a few ulp from silu_f); for
// values that are requantized right away, where it moves a code only at a rounding tie.
__device__ __forceinline__ float silu_approx(float v) { return __fdividef(v, 1.0f + __expf(-v)); }

// quant8(v, s) without the IEEE division or FRND on the common path: t = v * (1/s) is
// clamped to [-129, 128] and rounded half-to-even with the 1.5 * 2^23 magic add; t lies
// within a few ulp of v/s, so unless t sits within 1e-4 of a rounding tie (|t - v/s| <= 4e-5 for |t| <= 129) (detected, and
// then recomputed with the exact division) the code is bit-identical to quant8.
__device__ __forceinline__ int8_t quant8_inv(float v, float s, float inv_s) {
  const float t = fminf(fmaxf(__fmul_rn(v, inv_s), -129.f), 128.f);
  const float r = __fadd_rn(t, 12582912.0f);
  int q = __float_as_int(r) - 0x4B400000;
  if (fabsf(__fsub_rn(t, __fsub_rn(r, 12582912.0f))) > 0.4999f) q = (int)rintf(__fdiv_rn(v, s));
  return (int8_t)max(-128, min(127, q));
}

// Branch-free first pass of quant8_inv: returns the code from v * (1/s) and flags (tie=true)
// values within 1e-4 of a rounding tie, which the caller recomputes with quant8 (exact), so
// the codes stay bit-identical to quant8 while the common path has no division or branch.
// Clamping t to [-128, 127] before rounding equals rounding then clamping (integer bounds,
// monotone rint), so no integer clamp is needed; a clamped t is never flagged as a tie, and
// near ±127.5 / -128.5 both roundings clamp to the same code.
__device__ __forceinline__ int8_t quant8_fast(float v, float inv_s, bool& tie) {
  const float t = fminf(fmaxf(__fmul_rn(v, inv_s), -128.f), 127.f);
  const float r = __fadd_rn(t, 12582912.0f);
  tie |= fabsf(__fsub_rn(t, __fsub_rn(r, 12582912.0f))) > 0.4999f;
  return (int8_t)(__float_as_int(r) - 0x4B400000);
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

int launch_group_sum(const int8_t* codes, int64_t ld, int M, int K, int32_t* gsum, int64_t ldg, cudaStream_t st);
// int8 SSD chunk scan (ssd_chunk.cu); SQ_ERR_ARG when the shape is not eligible
int launch_ssd_chunk(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
                     const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                     int8_t* state, int state_in, float* y, int64_t ldy, cudaStream_t st);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- programmatic dependent launch (PDL) --------------------------------------------
// Kernels on the decode path are launched with programmatic stream serialization: the
// next kernel's CTAs may start (prologue, TMEM/smem setup, read-only weight prefetch)
// while this one drains.  Rule: everything a kernel does before pdl_wait() touches only
// read-only data (weights, scales) and on-chip memory; pdl_wait() returns once the
// previous grid has completed and its writes are visible.  Pointers to data produced by
// an earlier grid must NOT be `const __restrict__`: nvcc turns those loads into
// LDG.CONSTANT and hoists them above griddepcontrol.wait (seen in SASS).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// SQ_PDL: bitmask of kernel classes launched with PDL (default PDL_GEMM; 0 disables)
enum { PDL_ROW = 1, PDL_PREP = 2, PDL_RING = 4, PDL_NORM = 8, PDL_GEMM = 16 };
bool pdl_enabled(int cls);

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(int cls, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(cls) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace sq
