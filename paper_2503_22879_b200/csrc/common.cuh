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

// 4 int8 codes -> 2 x float2 (exact): each byte, biased to unsigned, becomes the low mantissa
// byte of 2^23 (PRMT), then 2^23 + 128 is subtracted with one packed add.
__device__ __forceinline__ void s8x4_f2x2(uint32_t u, float2& a, float2& b) {
  const uint32_t v = u ^ 0x80808080u;
  const float2 bias = make_float2(-8388736.0f, -8388736.0f);
  a = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7540)),
                             __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7541))), bias);
  b = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7542)),
                             __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7543))), bias);
}
__device__ __forceinline__ float ex2_approx(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
// SiLU of a channel pair with packed f32x2 math around the two MUFU ops (silu_approx form)
__device__ __forceinline__ float2 silu2_approx(float2 v) {
  const float2 t = __fmul2_rn(v, make_float2(-1.4426950408889634f, -1.4426950408889634f));
  const float2 d = __fadd2_rn(make_float2(ex2_approx(t.x), ex2_approx(t.y)), make_float2(1.f, 1.f));
  return __fmul2_rn(v, make_float2(rcp_approx(d.x), rcp_approx(d.y)));
}

// quant8_fast on four values held as two float2 (packed multiply / magic-number rint);
// returns the packed little-endian codes and ORs the tie flag (see quant8_fast).
__device__ __forceinline__ uint32_t quant8x4_fast(float2 v0, float2 v1, float2 inv0, float2 inv1, bool& tie) {
  const float2 RM = make_float2(12582912.0f, 12582912.0f), NRM = make_float2(-12582912.0f, -12582912.0f);
  const float2 M1 = make_float2(-1.f, -1.f);
  float2 t0 = __fmul2_rn(v0, inv0), t1 = __fmul2_rn(v1, inv1);
  t0.x = fminf(fmaxf(t0.x, -128.f), 127.f);
  t0.y = fminf(fmaxf(t0.y, -128.f), 127.f);
  t1.x = fminf(fmaxf(t1.x, -128.f), 127.f);
  t1.y = fminf(fmaxf(t1.y, -128.f), 127.f);
  const float2 r0 = __fadd2_rn(t0, RM), r1 = __fadd2_rn(t1, RM);
  const float2 d0 = __ffma2_rn(__fadd2_rn(r0, NRM), M1, t0), d1 = __ffma2_rn(__fadd2_rn(r1, NRM), M1, t1);
  tie |= fmaxf(fmaxf(fabsf(d0.x), fabsf(d0.y)), fmaxf(fabsf(d1.x), fabsf(d1.y))) > 0.4999f;
  // code bytes = low bytes of the rint bit patterns (0x4B400000 has a zero low byte)
  return __byte_perm(__byte_perm(__float_as_uint(r0.x), __float_as_uint(r0.y), 0x0040),
                     __byte_perm(__float_as_uint(r1.x), __float_as_uint(r1.y), 0x0040), 0x5410);
}

// LEDGER G14: log1p(exp(x)), identity above 20.
__device__ __forceinline__ float softplus_f(float v) {
  return v > 20.f ? v : log1pf(expf(v));
}

// softplus on the SFU (ex2 / lg2 approximations): identity above 20, e^v below -10 (relative error
// < e^v / 2 there), log(1 + e^v) between; a few ulp from softplus_f elsewhere.  For operands that
// feed tolerance-compared float math (the Mamba1 scan's Δ), not bit-exact paths.
__device__ __forceinline__ float softplus_approx(float v) {
  if (v > 20.f) return v;
  const float e = __expf(v);
  return v < -10.f ? e : __logf(1.f + e);
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
int launch_ssd_chunk_tc(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
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

// SQ_PDL_MASK (capi.cu): bitmask of kernel classes launched with PDL (default PDL_GEMM | PDL_PREP |
// PDL_RING | PDL_SMALL | PDL_SMALL8; 0 disables)
// PDL_SMALL: the f32 (W4A16) b=1 chain; PDL_SMALL8: the int8 b=1 chain
enum { PDL_ROW = 1, PDL_PREP = 2, PDL_RING = 4, PDL_NORM = 8, PDL_GEMM = 16, PDL_SMALL = 32, PDL_SMALL8 = 64 };
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
