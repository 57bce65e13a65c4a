// K5: depthwise causal conv1d on int8 codes + SiLU + requant (Quamba2 W8A8 conv,
// PAPER.md:302), prefill and decode-update variants.
//
// Layout: codes tokens-major [B*T x C] (C = d_inner + 2GN, contiguous, coalesced over c);
// cache [B x (Kc-1) x C] int8 = the last Kc-1 input codes (exact — no requant error).
// Math per (t, c) exactly as the oracle (oracle/qblock.py _conv_a8):
//   v_j = f32(q_j) * s_in[c];  acc = bias[c];  acc = acc + w[c,j]*v_j  (j ascending, unfused)
//   out = clamp(rint(silu(acc) / s_out[c]))
// HBM-bound: each code is read once by the thread that owns its (segment, channel) plus
// Kc-1 halo reads that hit L1/L2.
#include "common.cuh"

namespace sq {

constexpr int kMaxK = 8;
constexpr int kSeg = 64;   // tokens per thread in the prefill kernel

template <typename TIn, typename TOut, bool Q>
__global__ void conv1d_prefill_kernel(const TIn* x, int64_t ldx, const float* __restrict__ w,
                                      const float* __restrict__ bias, const float* __restrict__ s_in,
                                      const float* __restrict__ s_out, int B, int T, int C, int Kc,
                                      const TIn* cache, int cache_in, TOut* out, int64_t ldo) {
  pdl_trigger();
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int seg = blockIdx.y;
  const int b = blockIdx.z;
  if (c >= C) return;
  const int t0 = seg * kSeg;
  if (t0 >= T) return;
  const int t1 = min(T, t0 + kSeg);
  const float si = Q ? s_in[c] : 1.f;
  const float so = Q ? s_out[c] : 1.f;
  float wc[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) wc[j] = j < Kc ? w[c * Kc + j] : 0.f;
  const float bc = bias[c];
  float win[kMaxK];  // win[Kc-1] is the newest
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) win[j] = 0.f;
  // initial window: inputs t0-Kc+1 .. t0-1
  for (int j = 0; j < Kc - 1; ++j) {
    const int t = t0 - (Kc - 1) + j;
    float v = 0.f;
    if (t >= 0) {
      v = Q ? __fmul_rn((float)x[((int64_t)b * T + t) * ldx + c], si) : (float)x[((int64_t)b * T + t) * ldx + c];
    } else if (cache_in) {
      const int cj = (Kc - 1) + t;  // index into cache window
      TIn cv = cache[((int64_t)b * (Kc - 1) + cj) * C + c];
      v = Q ? __fmul_rn((float)cv, si) : (float)cv;
    }
    win[j] = v;
  }
  for (int t = t0; t < t1; ++t) {
    const TIn xv = x[((int64_t)b * T + t) * ldx + c];
    win[Kc - 1] = Q ? __fmul_rn((float)xv, si) : (float)xv;
    float acc = bc;
    for (int j = 0; j < Kc; ++j) acc = __fadd_rn(acc, __fmul_rn(wc[j], win[j]));
    const float sv = silu_f(acc);
    if (Q)
      reinterpret_cast<int8_t*>(out)[((int64_t)b * T + t) * ldo + c] = quant8(sv, so);
    else
      reinterpret_cast<float*>(out)[((int64_t)b * T + t) * ldo + c] = sv;
    for (int j = 0; j < Kc - 1; ++j) win[j] = win[j + 1];
  }
}

// int8 prefill, 4 channels per thread (one 32-bit load/store per token row, a warp moves
// 128 contiguous bytes), kSeg4 tokens per thread in sub-blocks of 8 rows whose loads are
// issued before any math.  Same op order as the scalar kernel; SiLU from the hardware
// exp2 / reciprocal approximations and the division-free quantizer with its exact tie
// fallback (codes move only at rounding ties).
constexpr int kSeg4 = 32;
template <int KC>
__global__ void __launch_bounds__(128) conv1d_prefill4_kernel(const int8_t* __restrict__ x, int64_t ldx,
                                                              const float* __restrict__ w,
                                                              const float* __restrict__ bias,
                                                              const float* __restrict__ s_in,
                                                              const float* __restrict__ s_out, int T, int C,
                                                              int8_t* __restrict__ cache, int cache_in,
                                                              int8_t* __restrict__ out, int64_t ldo) {
  const int c0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const int b = blockIdx.z;
  if (c0 >= C) return;
  const int t0 = blockIdx.y * kSeg4;
  const int t1 = min(T, t0 + kSeg4);
  // channel pairs (c0, c0+1) and (c0+2, c0+3) as float2 lanes
  float2 wc[2][KC], si[2], iso[2], bc[2];
  float so[4];
#pragma unroll
  for (int pr = 0; pr < 2; ++pr) {
    const int ca = c0 + 2 * pr, cb = ca + 1;
#pragma unroll
    for (int j = 0; j < KC; ++j) wc[pr][j] = make_float2(w[ca * KC + j], w[cb * KC + j]);
    si[pr] = make_float2(s_in[ca], s_in[cb]);
    so[2 * pr] = s_out[ca];
    so[2 * pr + 1] = s_out[cb];
    iso[pr] = make_float2(__frcp_rn(so[2 * pr]), __frcp_rn(so[2 * pr + 1]));
    bc[pr] = make_float2(bias[ca], bias[cb]);
  }
  // win[pr][j]: dequantised input at token t-KC+1+j; slot KC-1 is the newest.
  float2 win[2][KC];
#pragma unroll
  for (int pr = 0; pr < 2; ++pr)
#pragma unroll
    for (int j = 0; j < KC; ++j) win[pr][j] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 1; j < KC; ++j) {   // tokens t0-KC+j, j = 1..KC-1
    const int t = t0 - KC + j;
    uint32_t u = 0;
    if (t >= 0)
      u = *reinterpret_cast<const uint32_t*>(x + ((int64_t)b * T + t) * ldx + c0);
    else if (cache_in)
      u = *reinterpret_cast<const uint32_t*>(cache + ((int64_t)b * (KC - 1) + (KC - 1 + t)) * C + c0);
    float2 q[2];
    s8x4_f2x2(u, q[0], q[1]);
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
#pragma unroll
      for (int k = 0; k < KC - 1; ++k) win[pr][k] = win[pr][k + 1];
      win[pr][KC - 1] = __fmul2_rn(q[pr], si[pr]);
    }
  }
  if (blockIdx.y == 0 && KC > 1) {
    // the first segment owns the cache: only its threads read the old window (above, their own
    // 4 channels), so they alone may overwrite it with the sequence's last KC-1 input codes
    // (for T < KC-1 the kept old entries are read before any write)
    uint32_t nv[KC > 1 ? KC - 1 : 1];
#pragma unroll
    for (int j = 0; j < KC - 1; ++j) {
      const int t = T - (KC - 1) + j;
      nv[j] = t >= 0 ? *reinterpret_cast<const uint32_t*>(x + ((int64_t)b * T + t) * ldx + c0)
            : cache_in ? *reinterpret_cast<const uint32_t*>(cache + ((int64_t)b * (KC - 1) + (KC - 1 + t)) * C + c0)
                       : 0u;
    }
#pragma unroll
    for (int j = 0; j < KC - 1; ++j)
      *reinterpret_cast<uint32_t*>(cache + ((int64_t)b * (KC - 1) + j) * C + c0) = nv[j];
  }
  const float2 RM = make_float2(12582912.0f, 12582912.0f), NRM = make_float2(-12582912.0f, -12582912.0f);
  for (int tb = t0; tb < t1; tb += 8) {
    uint32_t u[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      u[i] = tb + i < t1 ? __ldg(reinterpret_cast<const uint32_t*>(x + ((int64_t)b * T + tb + i) * ldx + c0)) : 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (tb + i >= t1) break;
      float2 q[2], sv[2];
      s8x4_f2x2(u[i], q[0], q[1]);
      uint32_t packed = 0;
      bool tie = false;
      int qi[4];
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
#pragma unroll
        for (int k = 0; k < KC - 1; ++k) win[pr][k] = win[pr][k + 1];
        win[pr][KC - 1] = __fmul2_rn(q[pr], si[pr]);
        float2 acc = bc[pr];
#pragma unroll
        for (int j = 0; j < KC; ++j) acc = __fadd2_rn(acc, __fmul2_rn(wc[pr][j], win[pr][j]));
        sv[pr] = silu2_approx(acc);
        // quant8_fast on the pair: t = v / s (by reciprocal), magic-number rint, tie flag
        float2 t = __fmul2_rn(sv[pr], iso[pr]);
        // rint as an int, saturated by cvt.pack.sat below instead of clamping to [-128, 127] and
        // packing bytes (bit-identical codes).  Only the low side is clamped, at -2^22: the magic
        // add then keeps r > 0, so every t <= -128.5 saturates to -128 and every t >= 127.5 to 127
        t.x = fmaxf(t.x, -4194304.f);
        t.y = fmaxf(t.y, -4194304.f);
        const float2 r = __fadd2_rn(t, RM);
        const float2 d = __ffma2_rn(__fadd2_rn(r, NRM), make_float2(-1.f, -1.f), t);   // t - rint(t)
        tie |= fabsf(d.x) > 0.4999f || fabsf(d.y) > 0.4999f;
        qi[2 * pr] = __float_as_int(r.x) - 0x4B400000;
        qi[2 * pr + 1] = __float_as_int(r.y) - 0x4B400000;
      }
      {
        uint32_t hi;
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(qi[3]), "r"(qi[2]));
        asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(packed) : "r"(qi[1]), "r"(qi[0]), "r"(hi));
      }
      if (tie) {
        packed = (uint32_t)(uint8_t)quant8(sv[0].x, so[0]) | ((uint32_t)(uint8_t)quant8(sv[0].y, so[1]) << 8) |
                 ((uint32_t)(uint8_t)quant8(sv[1].x, so[2]) << 16) | ((uint32_t)(uint8_t)quant8(sv[1].y, so[3]) << 24);
      }
      *reinterpret_cast<uint32_t*>(out + ((int64_t)b * T + tb + i) * ldo + c0) = packed;
    }
  }
}

// Final cache window = last Kc-1 entries of (old cache ++ x).  Separate launch so the
// prefill kernel's reads of the old cache never race with these writes.
template <typename T_>
__global__ void conv1d_cache_kernel(const T_* x, int64_t ldx, int B, int T, int C, int Kc, T_* cache,
                                    int cache_in) {
  pdl_trigger();
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (c >= C) return;
  T_ nv[kMaxK];
  for (int j = 0; j < Kc - 1; ++j) {
    const int t = T - (Kc - 1) + j;  // position in x, negative -> old cache
    if (t >= 0)
      nv[j] = x[((int64_t)b * T + t) * ldx + c];
    else
      nv[j] = cache_in ? cache[((int64_t)b * (Kc - 1) + (Kc - 1 + t)) * C + c] : (T_)0;
  }
  for (int j = 0; j < Kc - 1; ++j) cache[((int64_t)b * (Kc - 1) + j) * C + c] = nv[j];
}

// f32 decode step (T = 1): the window is the cache (or zeros) + the new input; the output and the
// shifted cache in one launch (conv1d_prefill_kernel's op order: acc = b + Σ_j w_j·win_j, SiLU)
__global__ void conv1d_update_f32_kernel(const float* x, int64_t ldx, const float* __restrict__ w,
                                         const float* __restrict__ bias, int B, int C, int Kc, float* cache,
                                         int cache_in, float* out, int64_t ldo) {
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (c >= C) return;
  float wc[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) wc[j] = j < Kc ? w[c * Kc + j] : 0.f;
  const float bc = bias[c];
  pdl_wait();   // x and the cache come from earlier grids
  float* cr = cache + (int64_t)b * (Kc - 1) * C + c;
  float win[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) win[j] = (j < Kc - 1 && cache_in) ? cr[(int64_t)j * C] : 0.f;
  win[Kc - 1] = x[(int64_t)b * ldx + c];
  float acc = bc;
  for (int j = 0; j < Kc; ++j) acc = __fadd_rn(acc, __fmul_rn(wc[j], win[j]));
  out[(int64_t)b * ldo + c] = silu_f(acc);
  for (int j = 0; j < Kc - 1; ++j) cr[(int64_t)j * C] = win[j + 1];
}

__global__ void conv1d_update_kernel(const int8_t* x, int64_t ldx, const float* __restrict__ w,
                                     const float* __restrict__ bias, const float* __restrict__ s_in,
                                     const float* __restrict__ s_out, int B, int C, int Kc, int8_t* cache,
                                     int8_t* out, int64_t ldo) {
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (c >= C) return;
  // parameters before the grid dependency wait (static); codes and cache after it
  const float si = s_in[c], so = s_out[c], bc = bias[c];
  float wc[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) wc[j] = j < Kc ? w[c * Kc + j] : 0.f;
  pdl_wait();
  int8_t* cr = cache + (int64_t)b * (Kc - 1) * C + c;
  int8_t q[kMaxK];
  for (int j = 0; j < Kc - 1; ++j) q[j] = cr[(int64_t)j * C];
  q[Kc - 1] = x[(int64_t)b * ldx + c];
  float acc = bc;
  for (int j = 0; j < Kc; ++j) acc = __fadd_rn(acc, __fmul_rn(wc[j], __fmul_rn((float)q[j], si)));
  out[(int64_t)b * ldo + c] = quant8(silu_f(acc), so);
  for (int j = 0; j < Kc - 1; ++j) cr[(int64_t)j * C] = q[j + 1];
}

}  // namespace sq

using namespace sq;

extern "C" int sq_conv1d_int8(const int8_t* x, int64_t ldx, const float* w, const float* bias, const float* s_in,
                              const float* s_out, int B, int T, int C, int Kc, int8_t* cache, int cache_in,
                              int8_t* out, int64_t ldo, void* stream) {
  SQ_REQUIRE(B >= 0 && T >= 0 && C > 0 && Kc >= 1 && Kc <= kMaxK, SQ_ERR_SHAPE,
             "sq_conv1d_int8: bad shape (Kc=%d)", Kc);
  if (B == 0 || T == 0) return SQ_OK;
  cudaStream_t st = as_stream(stream);
  if (Kc == 4 && C % 4 == 0 && ldx % 4 == 0 && ldo % 4 == 0 && ((uintptr_t)x & 3) == 0 && ((uintptr_t)out & 3) == 0) {
    dim3 g((C / 4 + 127) / 128, (T + kSeg4 - 1) / kSeg4, B);
    conv1d_prefill4_kernel<4><<<g, 128, 0, st>>>(x, ldx, w, bias, s_in, s_out, T, C, cache, cache_in, out, ldo);
    return check_launch("sq_conv1d_int8");   // the cache window is written by the first segment
  } else {
    dim3 g((C + 127) / 128, (T + kSeg - 1) / kSeg, B);
    launch_k(PDL_SMALL, conv1d_prefill_kernel<int8_t, int8_t, true>, g, dim3(128), 0, st, x, ldx, w, bias, s_in, s_out, B, T, C, Kc, cache,
                                                                   cache_in, out, ldo);
  }
  if (Kc > 1) launch_k(PDL_SMALL, conv1d_cache_kernel<int8_t>, dim3((C + 127) / 128, B), dim3(128), 0, st, x, ldx, B, T, C, Kc, cache, cache_in);
  return check_launch("sq_conv1d_int8");
}

extern "C" int sq_conv1d_f32(const float* x, int64_t ldx, const float* w, const float* bias, int B, int T, int C,
                             int Kc, float* cache, int cache_in, float* out, int64_t ldo, void* stream) {
  SQ_REQUIRE(B >= 0 && T >= 0 && C > 0 && Kc >= 1 && Kc <= kMaxK, SQ_ERR_SHAPE, "sq_conv1d_f32: bad shape");
  if (B == 0 || T == 0) return SQ_OK;
  cudaStream_t st = as_stream(stream);
  if (T == 1 && Kc > 1) {   // decode step: output + cache shift in one launch
    launch_k(PDL_SMALL, conv1d_update_f32_kernel, dim3((C + 127) / 128, B), dim3(128), 0, st, x, ldx, w, bias, B, C, Kc,
             cache, cache_in, out, ldo);
    return check_launch("sq_conv1d_f32");
  }
  dim3 g((C + 127) / 128, (T + kSeg - 1) / kSeg, B);
  launch_k(PDL_SMALL, conv1d_prefill_kernel<float, float, false>, g, dim3(128), 0, st, x, ldx, w, bias, (const float*)nullptr, (const float*)nullptr, B, T, C, Kc, cache,
                                                                cache_in, out, ldo);
  if (Kc > 1) launch_k(PDL_SMALL, conv1d_cache_kernel<float>, dim3((C + 127) / 128, B), dim3(128), 0, st, x, ldx, B, T, C, Kc, cache, cache_in);
  return check_launch("sq_conv1d_f32");
}

extern "C" int sq_conv1d_update_int8(const int8_t* x, int64_t ldx, const float* w, const float* bias,
                                     const float* s_in, const float* s_out, int B, int C, int Kc, int8_t* cache,
                                     int8_t* out, int64_t ldo, void* stream) {
  SQ_REQUIRE(B >= 0 && C > 0 && Kc >= 1 && Kc <= kMaxK, SQ_ERR_SHAPE, "sq_conv1d_update_int8: bad shape");
  if (B == 0) return SQ_OK;
  launch_k(PDL_SMALL8, conv1d_update_kernel, dim3((C + 127) / 128, B), dim3(128), 0, as_stream(stream), x, ldx, w, bias, s_in, s_out, B, C,
                                                                                 Kc, cache, out, ldo);
  return check_launch("sq_conv1d_update_int8");
}
