/*
 * ssmquant_sm100.h — C-ABI of libssmquant_sm100.so, the B200 (sm_100a) hot path of
 * Quamba2's quantized Mamba block forward (arXiv 2503.22879).
 *
 * Every entry point replaces one step of the reference contract's quantized block
 * (/root/reference/SPEC.md; the reference ships no implementation of it):
 *
 *   sq_rmsnorm_quant          model pre-norm + per-tensor int8 quant of the block input u
 *                             ("quantize ... u", LEDGER G5, G8)
 *   sq_gemm_w8a8/sq_gemm_w4a8 in_proj / out_proj / x_proj / dt_proj / head:
 *                             tensor.matmul (pkg/src/ssmquant/tensor.py:33-54) on quantized
 *                             operands + quantizer.fuse_scales + requant
 *   sq_gemv_w4a16             W4A16 projections ("dequantizes weights into the float path",
 *                             SPEC.md:329)
 *   sq_conv1d_int8            ssm_block.causal_conv1d on int8 codes,
 *                             + SiLU + requant to clustered x / per-state-group B,C scales
 *   sq_conv1d_update_int8     the same with cache stepping (decode)
 *   sq_ssd_scan_int8          ssm_block.ssd_chunked / selective_scan for
 *                             Mamba2, int8 operands, fp32 state, gated output, int8 final state
 *   sq_selective_scan_int8    Mamba1 selective_scan
 *   sq_state_update_int8      decode-time stepping of SsmState
 *   sq_gate_norm_had_quant    RMSNorm + hadamard.hadamard_quantize
 *
 *   sq_repack_w4 / sq_unpack_w4   u4packed <-> kernel layout
 *
 * Conventions: all pointers are device pointers owned by the caller; the library never
 * allocates device memory and keeps no global mutable state except a thread-local
 * last-error string.  Row-major, tokens-major activations; `ld*` are row strides in
 * elements.  `stream` is a cudaStream_t.  Launches are asynchronous.  Return 0 on
 * success or a negative sq_status (mapped by the Python layer onto
 * ssmquant.errors: SQ_ERR_SHAPE -> ShapeError, SQ_ERR_LAYOUT -> LayoutError,
 * SQ_ERR_CUDA / SQ_ERR_ARCH -> RuntimeError).
 */
#ifndef SSMQUANT_SM100_H
#define SSMQUANT_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SQ_ABI_VERSION 8

typedef enum {
  SQ_OK = 0,
  SQ_ERR_SHAPE = -1,
  SQ_ERR_LAYOUT = -2,
  SQ_ERR_CUDA = -3,
  SQ_ERR_ARCH = -4,
  SQ_ERR_ARG = -5
} sq_status;

/* GEMM epilogues.  y[m,n] = f32(acc[m,n]) * alpha[n] with acc the exact int32 sum. */
typedef enum {
  SQ_EPI_I32 = 0,    /* out int32 [M x N] = acc                                    */
  SQ_EPI_F32 = 1,    /* out f32   [M x N] = y                                      */
  SQ_EPI_QUANT = 2,  /* out int8  [M x N] = clamp(rint(y / col_scale[n]), -128, 127) */
  SQ_EPI_RESID = 3   /* out f32   [M x N] += y   (residual stream, in place)         */
} sq_epilogue;

int sq_abi_version(void);
const char* sq_last_error(void);
/* 1 if the current device is sm_100 (B200-class) and the kernels can run. */
int sq_device_supported(void);

/* ---- weights ---------------------------------------------------------------------- */
/* u4packed [N x K/2] (low nibble = even k) -> kernel layout `dst` (sq_w4_bytes(N,K) bytes). */
int64_t sq_w4_bytes(int N, int K);
int sq_repack_w4(const uint8_t* u4packed, int N, int K, uint8_t* dst, void* stream);
int sq_unpack_w4(const uint8_t* src, int N, int K, uint8_t* u4packed, void* stream);

/* ---- model glue --------------------------------------------------------------------- */
/* out[m,:] = clamp(rint((x[m,:] * rsqrt(mean x^2 + eps)) * gamma / s));  gsum (optional)
 * receives the sums of the output codes over every 128-wide block, int32 [M x D/128]. */
int sq_rmsnorm_quant(const float* x, int64_t ldx, const float* gamma, float eps, float s,
                     int M, int D, int8_t* out, int64_t ldo, int32_t* gsum, int64_t ldg, void* stream);
/* out[m,:] = x[m,:] * rsqrt(mean x^2 + eps) * gamma (f32) */
int sq_rmsnorm_f32(const float* x, int64_t ldx, const float* gamma, float eps,
                   int M, int D, float* out, int64_t ldo, void* stream);
/* out[m,:] = clamp(rint(x[m,:] / s))  (quantizer.quantize, PerTensor) */
int sq_quantize_f32(const float* x, int64_t ldx, float s, int M, int D, int8_t* out, int64_t ldo, void* stream);
/* h[m,:] = codes[tok[m],:] * row_scale[tok[m]] */
int sq_embed_int8(const int8_t* codes, const float* row_scale, const int32_t* tok, int M, int D,
                  float* h, void* stream);
/* 4-bit embedding: h[m,:] = v(tok[m],:) * row_scale[tok[m]], v from u4packed rows [V x D/2] */
int sq_embed_u4(const uint8_t* packed, const float* row_scale, const int32_t* tok, int M, int D,
                float* h, void* stream);
/* tok[m] = argmax_n logits[m, n] (lowest index on ties) */
int sq_argmax_f32(const float* logits, int64_t ld, int M, int N, int32_t* tok, void* stream);

/* ---- projections ------------------------------------------------------------------ */
int sq_gemm_w8a8(const int8_t* a, int64_t lda, const int8_t* w /*[N x K]*/, const float* alpha,
                 int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
                 void* stream);
/* W4A8 with SPEC per-group float weight scales (LEDGER G11):
 *   y[m,n] = f32(s_a * p[m,n]),  p = fma(w_scale[n,g], f32(acc_g[m,n]), p) over groups g ascending
 *            (f32, one rounding per group),  acc_g = sum_{k in g} a[m,k] * w4[n,k] (int32)
 * When the kernel splits K over a cluster (sq_gemm_w4a8_splits(M,N,K) > 1), each split sums its own
 * groups from 0 and the partials are added in split order.  w_scale is the tiled layout written by
 * sq_tile_group_scales; SQ_EPI_I32 is not defined for per-group scales (SQ_ERR_ARG). */
int sq_gemm_w4a8(const int8_t* a, int64_t lda, const uint8_t* w4 /*repacked*/,
                 const float* w_scale /*tiled [ceil(N/128)][K/group][128]*/, int group, float s_a,
                 int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
                 void* stream);
int sq_gemm_w4a8_splits(int M, int N, int K);
/* group scales [N x G] row-major -> tiled [ceil(N/128)][G][128] (sq_group_scale_elems floats) */
int64_t sq_group_scale_elems(int N, int G);
int sq_tile_group_scales(const float* s_group, int N, int G, float* dst, void* stream);
/* W4A16: y[m,n] (+)= sum_g s_group[n,g] * sum_{k in g} w4[n,k] * bf16(x'[m,k])  (f32 accumulation;
 * x is f32 in memory and rounded to bf16, RN, on load; resid!=0 adds in place).  With norm_w
 * (nullable) x' = RMSNorm(x) = x * rsqrt(mean_k x^2 + eps) * norm_w (sq_rmsnorm_f32's math), else
 * x' = x.  w4 is the sq_repack_w4a16 layout (sq_w4a16_bytes): mma.sync bf16 fragment order when
 * K % 64 == 0 and group is 64 or 128, else row-major u4packed. */
int64_t sq_w4a16_bytes(int N, int K, int group);
int sq_repack_w4a16(const uint8_t* u4packed, int N, int K, int group, uint8_t* dst, void* stream);
int sq_gemv_w4a16(const float* x, int64_t ldx, const float* norm_w /*[K] or NULL*/, float eps,
                  const uint8_t* w4 /*sq_repack_w4a16 layout*/,
                  const float* s_group /*[N x K/group]*/, int group, int M, int N, int K,
                  float* out, int64_t ldo, int resid, void* stream);
/* sq_gemv_w4a16 with the depthwise causal conv (T = 1 decode update) fused into
 * the epilogue: for output columns n in [c0, c0 + C) the token's conv channel c = n - c0 takes
 * win = cache[m][0..Kc-2][c] | out[m][n], writes silu(bias[c] + Σ_j w[c][j]·win[j]) (unfused f32,
 * j ascending, as sq_conv1d_f32) to conv_out[m][c] and shifts the cache; the GEMV output itself
 * is written as before.  Replaces the sq_conv1d_f32 (T=1) launch of the W4A16 decode step. */
typedef struct {
  const float* w;      /* [C x Kc] */
  const float* b;      /* [C]      */
  int kc, c0, C;
  float* cache;        /* [M x (Kc-1) x C] */
  int cache_in;
  float* out;          /* [M x ldo]       */
  int64_t ldo;
} sq_conv_epilogue;
int sq_gemv_w4a16_conv(const float* x, int64_t ldx, const float* norm_w, float eps, const uint8_t* w4,
                       const float* s_group, int group, int M, int N, int K, float* out, int64_t ldo, int resid,
                       const sq_conv_epilogue* conv, void* stream);

/* ---- causal conv1d (+SiLU +requant) ------------------------------------------------- */
/* x codes [B*T x C] (row stride ldx), cache codes [B x (Kc-1) x C] (read as the initial
 * window if cache_in, always written with the final window), out codes [B*T x C]. */
int sq_conv1d_int8(const int8_t* x, int64_t ldx, const float* w /*[C x Kc]*/, const float* bias,
                   const float* s_in, const float* s_out, int B, int T, int C, int Kc,
                   int8_t* cache, int cache_in, int8_t* out, int64_t ldo, void* stream);
int sq_conv1d_update_int8(const int8_t* x, int64_t ldx, const float* w, const float* bias,
                          const float* s_in, const float* s_out, int B, int C, int Kc,
                          int8_t* cache, int8_t* out, int64_t ldo, void* stream);
/* fp32 variants (W4A16 float path): x/out f32, cache f32 */
int sq_conv1d_f32(const float* x, int64_t ldx, const float* w, const float* bias, int B, int T,
                  int C, int Kc, float* cache, int cache_in, float* out, int64_t ldo, void* stream);

/* ---- scans ------------------------------------------------------------------------ */
/* Mamba2 parameters shared by prefill and decode. */
typedef struct {
  int n_heads, head_dim, d_state, n_groups;
  const int32_t* head_group;   /* [nh] state group of each head                        */
  const float* A;              /* [nh] (= -exp(a_log))                                 */
  const float* D;              /* [nh]                                                 */
  const float* dt_bias;        /* [nh]                                                 */
  float s_dt, s_z;             /* per-tensor scales of the dt and z in_proj slices     */
  const float* s_x;            /* [nh*P] clustered x scales (conv output)              */
  const float* s_B;            /* [G]                                                  */
  const float* s_C;            /* [G]                                                  */
  const float* s_h;            /* [nh*P] cached-state scales (ClusterMap cells)        */
} sq_mamba2_params;

/* Prefill: codes x [B*T x nh*P], B/C [B*T x G*N], dt [B*T x nh], z [B*T x nh*P]
 * (row strides ldx/ldbc/lddt/ldz), state [B x nh x P x N] int8 (read if state_in,
 * written with the final state), y f32 [B*T x nh*P] gated by SiLU(z). */
int sq_ssd_scan_int8(const sq_mamba2_params* p, int B, int T,
                     const int8_t* x, int64_t ldx, const int8_t* Bm, const int8_t* Cm, int64_t ldbc,
                     const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                     int8_t* state, int state_in, float* y, int64_t ldy, int chunk, void* stream);
/* Decode (T=1): same operands, state updated in place. */
int sq_state_update_int8(const sq_mamba2_params* p, int B,
                         const int8_t* x, int64_t ldx, const int8_t* Bm, const int8_t* Cm, int64_t ldbc,
                         const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                         int8_t* state, float* y, int64_t ldy, void* stream);
/* W4A16 float path: f32 operands, f32 state [B x nh x P x N]. T=1 is decode. */
int sq_ssd_scan_f32(const sq_mamba2_params* p, int B, int T,
                    const float* x, int64_t ldx, const float* Bm, const float* Cm, int64_t ldbc,
                    const float* dt, int64_t lddt, const float* z, int64_t ldz,
                    float* state, int state_in, float* y, int64_t ldy, void* stream);

/* Mamba2 decode step (K5 decode + K9 + K6), the SSM half of a block for one token per
 * sequence, from the in_proj requant codes zx[b] = z | x | B | C | dt:
 *   conv-cache stepping + SiLU + requant of x, B, C  (ssm_block.causal_conv1d with cache,
 *   SPEC.md:281-289; same int8 math as sq_conv1d_update_int8), dequantised with the
 *   clustered x / per-group B,C scales into the f32 workspace `ws` together with the
 *   per-channel scan scalars,
 *   int8 SSM state update h' = exp(dt*A) h + dt*x*B, y = C.h' + D*x, y*SiLU(z)
 *   (selective_scan T=1) -> y,
 *   RMSNorm over d_inner + Sylvester FWHT + quant with s_y -> yq.
 * Three launches on `stream` (four with yq_gsum unless the 8192-wide Hadamard norm emits the
 * sums: sq_mamba2_decode_launches).  State and conv cache are updated in place; ws
 * (sq_mamba2_decode_ws_bytes) and y [B x d_inner] f32 are caller-owned (y holds the gated SSM
 * output). */
typedef struct {
  sq_mamba2_params ssm;
  int conv_kernel;
  const float* conv_w;      /* [conv_dim x conv_kernel]                              */
  const float* conv_b;      /* [conv_dim]                                            */
  const float* conv_s_in;   /* [conv_dim] scales of the in_proj x|B|C codes          */
  const float* conv_s_out;  /* [conv_dim] clustered x scales | per-group B, C scales */
  const float* norm_w;      /* [d_inner]                                             */
  float eps, s_y;
  int hadamard;
} sq_mamba2_decode_params;

int64_t sq_mamba2_decode_ws_bytes(const sq_mamba2_decode_params* p, int B);
int sq_mamba2_decode_launches(const sq_mamba2_decode_params* p, int B, int with_gsum);
int sq_mamba2_decode_step_int8(const sq_mamba2_decode_params* p, int B, const int8_t* zx, int64_t ldzx,
                               int8_t* conv_cache /*[B x (Kc-1) x conv_dim]*/, int8_t* state,
                               void* ws, float* y, int64_t ldy, int8_t* yq, int64_t ldyq,
                               int32_t* yq_gsum /*optional [B x d_inner/128]*/, int64_t ldg, void* stream);

typedef struct {
  int d_inner, d_state;
  const float* A;              /* [d_inner x N]                                        */
  const float* D;              /* [d_inner]                                            */
  const float* dt_bias;        /* [d_inner]                                            */
  float s_dt, s_z, s_B, s_C;
  const float* s_x;            /* [d_inner]                                            */
  const float* s_h;            /* [d_inner]                                            */
} sq_mamba1_params;

/* Mamba1 W8A8 decode step (T = 1, B <= 8), SSM half of a block in ONE launch (decode_m1.cu):
 * conv update + cache shift -> x_proj -> dt_proj (both W8A8 int8 [N x K] row-major, EPI_QUANT
 * epilogue quant8(f32(acc)*alpha[n], cs[n])) -> int8 scan step -> gated RMSNorm + FWHT + quant.
 * Replaces sq_conv1d_update_int8 + 2x sq_gemm_w8a8 + sq_selective_scan_int8 (T=1) +
 * sq_gate_norm_had_quant on the reference's decode path.
 * zx [B x 2*d_inner] in_proj codes (z | x); ws: sq_mamba1_decode_ws_bytes bytes, 16-B aligned,
 * ZEROED ONCE before first use (grid barrier counters, self-resetting); yq [B x d_inner]. */
typedef struct {
  sq_mamba1_params ssm;
  int conv_kernel;
  const float* conv_w;        /* [d_inner x conv_kernel]                              */
  const float* conv_b;        /* [d_inner]                                            */
  const float* conv_s_in;     /* [d_inner] in_proj x code scales                      */
  const float* conv_s_out;    /* [d_inner] conv output scales                         */
  int dt_rank;
  const int8_t* xproj_w;      /* [dt_rank + 2N x d_inner]                             */
  const float* xproj_alpha;   /* [dt_rank + 2N]  s_w[n] * s_a                          */
  const float* xproj_cs;      /* [dt_rank + 2N]  output code scales                   */
  const int8_t* dtproj_w;     /* [d_inner x dt_rank]                                  */
  const float* dtproj_alpha;  /* [d_inner]                                            */
  const float* dtproj_cs;     /* [d_inner]                                            */
  const float* norm_w;        /* [d_inner]                                            */
  float eps, s_y;
  int hadamard;
} sq_mamba1_decode_params;

int64_t sq_mamba1_decode_ws_bytes(const sq_mamba1_decode_params* p, int B);
/* Whole Mamba1 W8A8 decode layer in ONE launch (B <= 8): the model's pre-norm + quant of the
 * residual stream h (sq_rmsnorm_quant's math and order), in_proj (W8, EPI_QUANT), the SSM half of
 * sq_mamba1_decode_step_int8, and out_proj (W8, EPI_RESID into h).  Replaces the four launches
 * sq_rmsnorm_quant + sq_gemm_w8a8 + sq_mamba1_decode_step_int8 + sq_gemm_w8a8 of a layer.
 * ws as sq_mamba1_decode_ws_bytes (zeroed once). */
typedef struct {
  const float* ln_w;          /* [d_model] the model's pre-norm weight */
  float ln_eps, s_u;          /* its eps; in_proj input code scale     */
  int d_model;
  const int8_t* in_w;         /* [2*d_inner x d_model]                 */
  const float* in_alpha;      /* [2*d_inner]                           */
  const float* in_cs;         /* [2*d_inner] output code scales        */
  const int8_t* out_w;        /* [d_model x d_inner]                   */
  const float* out_alpha;     /* [d_model]                             */
} sq_mamba1_layer_params;
int sq_mamba1_decode_layer_int8(const sq_mamba1_decode_params* p, const sq_mamba1_layer_params* lp, int B,
                                float* h, int64_t ldh, int8_t* conv_cache, int8_t* state, void* ws, void* stream);

int sq_mamba1_decode_step_int8(const sq_mamba1_decode_params* p, int B, const int8_t* zx, int64_t ldzx,
                               int8_t* conv_cache /*[B x (Kc-1) x d_inner]*/, int8_t* state /*[B x d_inner x 16]*/,
                               void* ws, int8_t* yq, int64_t ldyq, void* stream);

/* Mamba1 prefill (T>=1; T=1 is decode): codes x [B*T x d], dt [B*T x d], B/C [B*T x N]
 * (row stride ldbc, C at +N), z [B*T x d]; state int8 [B x d x N].  ws (16-B aligned,
 * sq_selective_scan_int8_ws_bytes, may be NULL) enables the time-chunked two-pass scan for long
 * prompts (two launches instead of one). */
int64_t sq_selective_scan_int8_ws_bytes(const sq_mamba1_params* p, int B, int T);
int sq_selective_scan_int8(const sq_mamba1_params* p, int B, int T,
                           const int8_t* x, int64_t ldx, const int8_t* dt, int64_t lddt,
                           const int8_t* BC, int64_t ldbc, const int8_t* z, int64_t ldz,
                           int8_t* state, int state_in, float* y, int64_t ldy, void* ws, void* stream);

/* Mamba1 W4A16 scan on floats: x / dt_raw / z [B*T x d], B|C rows [B*T x 2N] (stride ldbc,
 * C at +N), state f32 [B x d x N].  Replaces the reference's float selective_scan for the
 * Mamba1 W4A16 profile. */
int sq_selective_scan_f32(const sq_mamba1_params* p, int B, int T,
                          const float* x, int64_t ldx, const float* dt, int64_t lddt,
                          const float* BC, int64_t ldbc, const float* z, int64_t ldz,
                          float* state, int state_in, float* y, int64_t ldy, void* stream);

/* ---- gated-norm + Hadamard + quant ------------------------------------------------ */
/* out[m,:] = clamp(rint(H_blk (y*rsqrt(mean y^2+eps)*gamma) / s_y)); hadamard=0 skips H. */
int sq_gate_norm_had_quant(const float* y, int64_t ldy, const float* gamma, float eps, float s_y,
                           int hadamard, int M, int D, int8_t* out, int64_t ldo, void* stream);

/* ---- SPEC float ops (ssm_block.discretize / selective_scan / ssd_chunked) --
 * Δ = softplus(dt_raw + dt_bias) [M x H];  Ȧ = exp(Δ·A) [M x H x N] (A [H x N]; Mamba2: N = 1). */
int sq_discretize_f32(const float* dt_raw, int64_t ld, const float* dt_bias, const float* A, int M, int H, int N,
                      float* dA, float* delta, void* stream);
/* Recurrence on precomputed Ȧ / Δ (selective_scan(x, Ȧ, Δ, B, C, D, z, state)); z may be NULL
 * (no gate).  Mamba2 form: Ȧ, Δ [B*T x nh] (row stride lddt), B/C [B*T x G*N] per state group;
 * the params' A / dt_bias are unused.  Mamba1 form: Ȧ [B*T x d_inner x N] dense, Δ [B*T x d_inner]. */
int sq_selective_scan2_pre_f32(const sq_mamba2_params* p, int B, int T, const float* x, int64_t ldx,
                               const float* dA, const float* delta, int64_t lddt, const float* Bm,
                               const float* Cm, int64_t ldbc, const float* z, int64_t ldz, float* state,
                               int state_in, float* y, int64_t ldy, void* stream);
int sq_selective_scan1_pre_f32(const sq_mamba1_params* p, int B, int T, const float* x, int64_t ldx,
                               const float* dA, const float* delta, int64_t lddt, const float* Bm,
                               const float* Cm, int64_t ldbc, const float* z, int64_t ldz, float* state,
                               int state_in, float* y, int64_t ldy, void* stream);

#ifdef __cplusplus
}
#endif
#endif
