// Mamba2 decode step (PAPER.md:771-774
// int8 cached state): the SSM half of a block for one token per sequence, three launches:
//
//  K5d  prep_kernel        conv-cache stepping + SiLU + requant of every x|B|C channel
//                            (4 channels per thread, all loads issued up front), then the
//                            per-row scan scalars (x̂, Δx̂/s_h, SiLU(ẑ), s_h) and per-head
//                            (Ȧ, D) packed per (sequence, head) and the dequantised B̂|Ĉ
//                            packed per (sequence, group) into an f32 workspace, laid out so
//                            each state tile's operands are three contiguous bulk copies.
//  K9   state_ring_kernel    persistent, 2 CTAs/SM; a producer warp streams (state tile
//                            8 KB, row scalars 1 KB, B̂|Ĉ 1 KB) per (sequence, head) with
//                            1-D bulk TMA into an 8-deep smem ring, 8 consumer warps update
//                            and release slots through per-slot mbarriers (no block-wide
//                            barriers), so HBM always has ~80 KB per CTA in flight.  h' is
//                            computed in "scaled units" t = h'/s_h = Ȧ·q + (Δx̂/s_h)·B̂ with
//                            packed f32x2 FMAs; the requant is a magic-number rint (FADD2) +
//                            cvt.pack.sat, exact because |Δx̂/s_h·B̂| is clamped to 2^21
//                            (saturation keeps the sign); y = s_h·Σ t·Ĉ + D·x̂, gated by SiLU(ẑ).
//  K6   norm_had8192_kernel  d_inner = 8192: one CTA per row, FWHT in three register phases
//                            joined by two swizzled smem transposes;
//       norm_had_kernel      other widths: one thread-block cluster per sequence (CL <= 8 CTAs of <= 1024
//                            channels): Σy² reduced across the cluster in f64 (rank order),
//                            r·γ, Sylvester FWHT stages in the oracle's order — in registers,
//                            shuffles, smem, and across CTAs through DSMEM for Hadamard
//                            blocks wider than a CTA — then rint(v / s_y) -> yq.
// Numerics vs the oracle (oracle/qblock.py decode_step_batched): conv codes op-for-op; state
// codes and yq within one quantization step (fused FMA / scaled-unit update, f32 y sum);
// tested with mismatch fractions in tests/test_gpu_decode.py.
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace sq {
using namespace sm100;

constexpr int DS_P = 64;
// profiling builds only (-DSQ_DECODE_STAGES=m): bitmask of the launches issued, 1 prep | 2 state | 4 norm
#ifndef SQ_DECODE_STAGES
#define SQ_DECODE_STAGES 7
#endif
constexpr int DS_MAXCH = 1024;   // channels per norm CTA
constexpr int ST_THREADS = 256;
constexpr int ST_HEADS = 4;      // heads per state CTA

__device__ __forceinline__ float s8_raw(uint32_t u_xor80, int i) {
  // 2^23 + 128 + (signed byte i of the original word); subtract 8388736 for the value
  uint32_t bits;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bits) : "r"(u_xor80), "r"(0x4B000000u), "r"(0x7440u | (uint32_t)i));
  return __int_as_float(bits);
}

__device__ __forceinline__ uint32_t pack4_sat(int q0, int q1, int q2, int q3) {
  uint32_t hi, out;
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, 0;" : "=r"(hi) : "r"(q3), "r"(q2));
  asm("cvt.pack.sat.s8.s32.b32 %0, %1, %2, %3;" : "=r"(out) : "r"(q1), "r"(q0), "r"(hi));
  return out;
}

__device__ __forceinline__ float4 ld_dsmem_f32x4(uint32_t addr) {
  float4 v;
  asm("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ double ld_dsmem_f64_nv(uint32_t addr) {
  double v;
  asm("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float fget(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }

// One conv output code for channel c (sq_conv1d_update_int8's exact op order), shifting
// the cache window.  Generic kernel size.
__device__ __forceinline__ int8_t conv_step(const sq_mamba2_decode_params& P, int Kc, int c, int C,
                                            int8_t* __restrict__ cache_b, int8_t xnew) {
  const float si = P.conv_s_in[c];
  float acc = P.conv_b[c];
  int8_t prev = 0;
  for (int j = 0; j < Kc; ++j) {
    const int8_t q = j < Kc - 1 ? cache_b[(int64_t)j * C + c] : xnew;
    acc = __fadd_rn(acc, __fmul_rn(P.conv_w[c * Kc + j], __fmul_rn((float)q, si)));
    if (j > 0) cache_b[(int64_t)(j - 1) * C + c] = q;
    prev = q;
  }
  (void)prev;
  return quant8(silu_f(acc), P.conv_s_out[c]);
}

// Four consecutive channels c..c+3 with Kc = 4.  The layer's constants (taps, bias, scales)
// are loaded before the grid-dependency wait; the codes after it.  Same per-channel op order
// as the oracle (acc = b + Σ_j w_j·(q_j·s_in), IEEE RN each) computed as packed f32x2 pairs,
// SiLU from the MUFU exp2 / reciprocal, and the division-free quantizer with its exact tie
// fallback.
struct Conv4Params {
  float4 t0, t1, t2, t3, bi, si, so;
};
__device__ __forceinline__ Conv4Params conv4_params(const sq_mamba2_decode_params& P, int c) {
  const float4* wt = reinterpret_cast<const float4*>(P.conv_w + (int64_t)c * 4);
  return {__ldg(wt), __ldg(wt + 1), __ldg(wt + 2), __ldg(wt + 3),
          __ldg(reinterpret_cast<const float4*>(P.conv_b + c)), __ldg(reinterpret_cast<const float4*>(P.conv_s_in + c)),
          __ldg(reinterpret_cast<const float4*>(P.conv_s_out + c))};
}
__device__ __forceinline__ uint32_t conv4_compute(const Conv4Params& k, uint32_t w0, uint32_t w1, uint32_t w2,
                                                  uint32_t w3) {
  // taps of channel pairs (c, c+1) and (c+2, c+3), tap j
  const float2 wa[4] = {make_float2(k.t0.x, k.t1.x), make_float2(k.t0.y, k.t1.y), make_float2(k.t0.z, k.t1.z),
                        make_float2(k.t0.w, k.t1.w)};
  const float2 wb[4] = {make_float2(k.t2.x, k.t3.x), make_float2(k.t2.y, k.t3.y), make_float2(k.t2.z, k.t3.z),
                        make_float2(k.t2.w, k.t3.w)};
  const uint32_t win[4] = {w0, w1, w2, w3};
  const float2 sia = make_float2(k.si.x, k.si.y), sib = make_float2(k.si.z, k.si.w);
  float2 acca = make_float2(k.bi.x, k.bi.y), accb = make_float2(k.bi.z, k.bi.w);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float2 qa, qb;
    s8x4_f2x2(win[j], qa, qb);
    acca = __fadd2_rn(acca, __fmul2_rn(wa[j], __fmul2_rn(qa, sia)));
    accb = __fadd2_rn(accb, __fmul2_rn(wb[j], __fmul2_rn(qb, sib)));
  }
  const float2 va = silu2_approx(acca), vb = silu2_approx(accb);
  bool tie = false;
  // reciprocal estimates are within ~1 ulp: quant8_fast's tie window (1e-4 of a step) covers it
  uint32_t code = quant8x4_fast(va, vb, make_float2(rcp_approx(k.so.x), rcp_approx(k.so.y)),
                                make_float2(rcp_approx(k.so.z), rcp_approx(k.so.w)), tie);
  if (tie)
    code = (uint32_t)(uint8_t)quant8(va.x, k.so.x) | ((uint32_t)(uint8_t)quant8(va.y, k.so.y) << 8) |
           ((uint32_t)(uint8_t)quant8(vb.x, k.so.z) << 16) | ((uint32_t)(uint8_t)quant8(vb.y, k.so.w) << 24);
  return code;
}


// ------------------------------------------------------------------ decode workspace layout
// per (sequence, head): ROWF floats = x̂[64] | Δx̂/s_h[64] | SiLU(ẑ)[64] | s_h[64] | Ȧ, D, 0, 0
// per (sequence, group): B̂[N] | Ĉ[N], each in the consumer's bank-conflict-free order:
//   n = chunk*CPT + 4e + j  lives at  (e*8 + chunk)*4 + j   (CPT = N/8 columns per thread)
constexpr int DS_ROWF = 4 * DS_P + 4;
__host__ __device__ inline int64_t ds_rows_floats(int B, int nh) { return (int64_t)B * nh * DS_ROWF; }
__host__ __device__ inline int64_t ds_ws_floats(int B, int nh, int G, int N) {
  return ds_rows_floats(B, nh) + (int64_t)B * G * 2 * N;
}
__device__ __forceinline__ int bc_swz(int n, int N) {
  const int cpt = N / 8;
  const int chunk = n / cpt, r = n % cpt, e = r >> 2, j = r & 3;
  return ((e * 8 + chunk) << 2) + j;
}

// ------------------------------------------------------------------ K5d: conv + scan operands
__global__ void __launch_bounds__(256) prep_kernel(const sq_mamba2_decode_params P, int C, int di, int GN,
                                                  const int8_t* zx, int64_t ldzx,
                                                  int8_t* __restrict__ cache, float* __restrict__ ws, int B,
                                                  int vec) {
  const sq_mamba2_params& S = P.ssm;
  const int N = S.d_state, nh = S.n_heads;
  const int b = blockIdx.y;
  const int Kc = P.conv_kernel;
  pdl_trigger();
  const int8_t* zrow = zx + (int64_t)b * ldzx;
  int8_t* cache_b = cache + (int64_t)b * (Kc - 1) * C;
  float* rows_b = ws + (int64_t)b * nh * DS_ROWF;
  float* bc_b = ws + ds_rows_floats(B, nh) + (int64_t)b * 2 * GN;
  const int step = vec ? 4 : 1;
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * step;
  if (vec && c < C) {   // four consecutive channels, one head (x) or one group run of B / C
    // layer constants first (no grid in the chain writes them), then wait for the codes
    const Conv4Params kp = conv4_params(P, c);
    const bool isx = c < di;
    const int h = isx ? c / DS_P : 0;
    float4 sh = make_float4(0.f, 0.f, 0.f, 0.f);
    float dtb = 0.f, Ah = 0.f, Dh = 0.f, sBg = 1.f;
    if (isx) {
      sh = __ldg(reinterpret_cast<const float4*>(S.s_h + c));
      dtb = S.dt_bias[h];
      Ah = S.A[h];
      Dh = S.D[h];
      sBg = S.s_B[S.head_group[h]];
    }
    pdl_wait();
    const uint32_t w0 = *reinterpret_cast<const uint32_t*>(cache_b + c);
    const uint32_t w1 = *reinterpret_cast<const uint32_t*>(cache_b + C + c);
    const uint32_t w2 = *reinterpret_cast<const uint32_t*>(cache_b + 2 * C + c);
    const uint32_t w3 = *reinterpret_cast<const uint32_t*>(zrow + di + c);
    const uint32_t zc = isx ? *reinterpret_cast<const uint32_t*>(zrow + c) : 0u;
    const int8_t dcode = isx ? zrow[2 * di + 2 * GN + h] : (int8_t)0;
    *reinterpret_cast<uint32_t*>(cache_b + c) = w1;
    *reinterpret_cast<uint32_t*>(cache_b + C + c) = w2;
    *reinterpret_cast<uint32_t*>(cache_b + 2 * C + c) = w3;
    const uint32_t code = conv4_compute(kp, w0, w1, w2, w3);
    const float4 so = kp.so;
    const float4 v = make_float4(__fmul_rn((float)(int8_t)code, so.x), __fmul_rn((float)(int8_t)(code >> 8), so.y),
                                 __fmul_rn((float)(int8_t)(code >> 16), so.z), __fmul_rn((float)(int8_t)(code >> 24), so.w));
    if (isx) {   // x channels: the scan's per-row operands
      const int p = c % DS_P;
      const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dcode, S.s_dt), dtb));
      const float rsmax = 2097152.0f / (128.0f * sBg);   // |rs·B̂| <= 2^21
      float* rf = rows_b + (int64_t)h * DS_ROWF;
      auto rs = [&](float xh, float s) {
        return fminf(fmaxf(__fmul_rn(__fmul_rn(delta, xh), __frcp_rn(s)), -rsmax), rsmax);
      };
      const float2 za = silu2_approx(__fmul2_rn(make_float2((float)(int8_t)zc, (float)(int8_t)(zc >> 8)),
                                                make_float2(S.s_z, S.s_z)));
      const float2 zb = silu2_approx(__fmul2_rn(make_float2((float)(int8_t)(zc >> 16), (float)(int8_t)(zc >> 24)),
                                                make_float2(S.s_z, S.s_z)));
      *reinterpret_cast<float4*>(rf + p) = v;
      *reinterpret_cast<float4*>(rf + DS_P + p) = make_float4(rs(v.x, sh.x), rs(v.y, sh.y), rs(v.z, sh.z), rs(v.w, sh.w));
      *reinterpret_cast<float4*>(rf + 2 * DS_P + p) = make_float4(za.x, za.y, zb.x, zb.y);
      *reinterpret_cast<float4*>(rf + 3 * DS_P + p) = sh;
      if (p == 0) {
        rf[4 * DS_P] = expf(__fmul_rn(delta, Ah));
        rf[4 * DS_P + 1] = Dh;
      }
    } else {        // B | C channels: four consecutive n of one group land contiguously
      const int j = c - di;
      const int isC = j >= GN ? 1 : 0;
      const int jj = j - isC * GN;
      const int g = jj / N, n = jj % N;
      *reinterpret_cast<float4*>(bc_b + (int64_t)g * 2 * N + isC * N + bc_swz(n, N)) = v;
    }
    return;
  }
  pdl_wait();
  if (c >= C) return;
  const int8_t q = conv_step(P, Kc, c, C, cache_b, zrow[di + c]);
  if (c < di) {
    const int h = c / DS_P;
    const float delta = softplus_f(__fadd_rn(__fmul_rn((float)zrow[2 * di + 2 * GN + h], S.s_dt), S.dt_bias[h]));
    const float rsmax = 2097152.0f / (128.0f * S.s_B[S.head_group[h]]);
    float* rf = rows_b + (int64_t)h * DS_ROWF;
    const int p = c % DS_P;
    const float xh = __fmul_rn((float)q, P.conv_s_out[c]);
    const float sh = S.s_h[c];
    rf[p] = xh;
    rf[DS_P + p] = fminf(fmaxf(__fmul_rn(__fmul_rn(delta, xh), __frcp_rn(sh)), -rsmax), rsmax);
    rf[2 * DS_P + p] = silu_approx(__fmul_rn((float)zrow[c], S.s_z));
    rf[3 * DS_P + p] = sh;
    if (p == 0) {
      rf[4 * DS_P] = expf(__fmul_rn(delta, S.A[h]));
      rf[4 * DS_P + 1] = S.D[h];
    }
  } else {
    const int j = c - di;
    const int isC = j >= GN ? 1 : 0;
    const int jj = j - isC * GN;
    const int g = jj / N, n = jj % N;
    bc_b[(int64_t)g * 2 * N + isC * N + bc_swz(n, N)] = __fmul_rn((float)q, P.conv_s_out[c]);
  }
}

// ------------------------------------------------------------------ K9: streaming state update
constexpr int SR_CONSUMERS = 8;
constexpr int SR_THREADS = (SR_CONSUMERS + 1) * 32;
#ifndef SQ_SR_NSLOT
#define SQ_SR_NSLOT 8
#endif
constexpr int SR_NSLOT = SQ_SR_NSLOT;   // state-tile ring depth per CTA (two per SM); same-box sweep 6 / 8 / 10 -> 15.19k / 15.52k / 15.13k tok/s
template <int N>
struct SrCfg {
  static constexpr int TILE = DS_P * N;
  static constexpr int ROWB = DS_ROWF * 4;
  static constexpr int BCB = 2 * N * 4;
  static constexpr int SLOT = TILE + ROWB + BCB;
  static constexpr int SMEM = SR_NSLOT * SLOT + 2 * SR_NSLOT * 8 + 128;
};

template <int N>
__global__ void __launch_bounds__(SR_THREADS, 2) state_ring_kernel(const sq_mamba2_params S, int B,
                                                                  const float* __restrict__ ws,
                                                                  int8_t* __restrict__ state, float* __restrict__ y,
                                                                  int64_t ldy) {
  using Cfg = SrCfg<N>;
  constexpr int CPT = N / 8;   // state columns per thread
  constexpr int VW = CPT / 4;  // 32-bit words per row piece
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SR_NSLOT * Cfg::SLOT);
  uint64_t* empty = full + SR_NSLOT;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nh = S.n_heads, GN = S.n_groups * N;
  const int ntiles_all = B * nh;
  const int ntiles = (ntiles_all - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  pdl_trigger();
  if (tid == 0) {
    for (int i = 0; i < SR_NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], SR_CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();   // prep outputs (ws) and the state: produced / last written by earlier grids
  const float* bc_all = ws + ds_rows_floats(B, nh);
  if (warp == SR_CONSUMERS) {
    // ---------------- producer: state tile + row scalars + B̂|Ĉ of the head's group
    if (lane == 0) {
      for (int i = 0; i < ntiles; ++i) {
        const int t = blockIdx.x + i * gridDim.x;
        const int b = t / nh, h = t % nh;
        const int slot = i % SR_NSLOT;
        if (i >= SR_NSLOT) mbar_wait(&empty[slot], ((i / SR_NSLOT) - 1) & 1);
        uint8_t* dst = smem + slot * Cfg::SLOT;
        mbar_arrive_expect_tx(&full[slot], Cfg::SLOT);
        bulk_load(dst, state + (int64_t)t * Cfg::TILE, Cfg::TILE, &full[slot]);
        bulk_load(dst + Cfg::TILE, ws + (int64_t)t * DS_ROWF, Cfg::ROWB, &full[slot]);
        bulk_load(dst + Cfg::TILE + Cfg::ROWB, bc_all + ((int64_t)b * S.n_groups + S.head_group[h]) * 2 * N,
                  Cfg::BCB, &full[slot]);
      }
    }
    return;
  }
  // ---------------- consumers: thread = (row quad rq, column chunk); rows rq and rq + 32
  const int chunk = tid & 7, rq = tid >> 3;
  const float2 MG = make_float2(-8388736.0f, -8388736.0f);
  const float2 RM = make_float2(12582912.0f, 12582912.0f);
  const int gstep = gridDim.x;
  const int db = gstep / nh, dh = gstep % nh;   // tile t -> (b, h) advanced incrementally
  int b = blockIdx.x / nh, h = blockIdx.x % nh;
  const uint32_t full0 = smem_u32(full);
  for (int i = 0; i < ntiles; ++i) {
    const int t = b * nh + h;
    const int slot = i % SR_NSLOT;
    const uint8_t* sl = smem + slot * Cfg::SLOT;
    const float* rf = reinterpret_cast<const float*>(sl + Cfg::TILE);
    const float* bcs = reinterpret_cast<const float*>(sl + Cfg::TILE + Cfg::ROWB);
    mbar_wait_addr(full0 + slot * 8, (i / SR_NSLOT) & 1);
    float2 bv[CPT / 2], cv[CPT / 2];
#pragma unroll
    for (int e = 0; e < CPT / 4; ++e) {
      const float4 b4 = *reinterpret_cast<const float4*>(bcs + ((e * 8 + chunk) << 2));
      const float4 c4 = *reinterpret_cast<const float4*>(bcs + N + ((e * 8 + chunk) << 2));
      bv[e * 2] = make_float2(b4.x, b4.y);
      bv[e * 2 + 1] = make_float2(b4.z, b4.w);
      cv[e * 2] = make_float2(c4.x, c4.y);
      cv[e * 2 + 1] = make_float2(c4.z, c4.w);
    }
    const float dA = rf[4 * DS_P], Dh = rf[4 * DS_P + 1];
    const float2 dA2 = make_float2(dA, dA);
    int8_t* st = state + (int64_t)t * Cfg::TILE + chunk * CPT;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int R = rq + 32 * k;
      const float rs = rf[DS_P + R];
      const float2 rs2 = make_float2(rs, rs);
      uint32_t raw[VW];
      if constexpr (VW == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(sl + R * N + chunk * CPT);
        raw[0] = v.x; raw[1] = v.y; raw[2] = v.z; raw[3] = v.w;
      } else {
        const uint2 v = *reinterpret_cast<const uint2*>(sl + R * N + chunk * CPT);
        raw[0] = v.x; raw[1] = v.y;
      }
      uint32_t outw[VW];
      float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int e = 0; e < VW; ++e) {
        const uint32_t u = raw[e] ^ 0x80808080u;
        int qi[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; i2 += 2) {
          const int n2 = e * 2 + i2 / 2;
          const float2 hq = __fadd2_rn(make_float2(s8_raw(u, i2), s8_raw(u, i2 + 1)), MG);
          const float2 tt = __ffma2_rn(dA2, hq, __fmul2_rn(rs2, bv[n2]));
          acc2 = __ffma2_rn(tt, cv[n2], acc2);
          const float2 rr = __fadd2_rn(tt, RM);   // bits = 0x4B400000 + rint(t), |t| < 2^22
          qi[i2] = __float_as_int(rr.x) - 0x4B400000;
          qi[i2 + 1] = __float_as_int(rr.y) - 0x4B400000;
        }
        outw[e] = pack4_sat(qi[0], qi[1], qi[2], qi[3]);
      }
      if constexpr (VW == 4)
        *reinterpret_cast<uint4*>(st + R * N) = make_uint4(outw[0], outw[1], outw[2], outw[3]);
      else
        *reinterpret_cast<uint2*>(st + R * N) = make_uint2(outw[0], outw[1]);
      float acc = __fadd_rn(acc2.x, acc2.y);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (chunk == 0)
        y[(int64_t)b * ldy + h * DS_P + R] =
            __fmul_rn(__fadd_rn(__fmul_rn(rf[3 * DS_P + R], acc), __fmul_rn(Dh, rf[R])), rf[2 * DS_P + R]);
    }
    fence_proxy_async_smem();   // our generic reads of the slot precede the next bulk copy into it
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    h += dh;
    b += db;
    if (h >= nh) {
      h -= nh;
      ++b;
    }
  }
}

// ------------------------------------------------------------------ K6: norm + FWHT + quant
// cluster of `cl` CTAs per sequence, CTA r owns channels [r*CH, (r+1)*CH), E = CH/256 each thread
__global__ void __launch_bounds__(256) norm_had_kernel(const sq_mamba2_decode_params P, int di, int CH, int cl,
                                                      int blk, const float* y, int64_t ldy,
                                                      int8_t* __restrict__ yq, int64_t ldyq) {
  __shared__ __align__(16) float ys[DS_MAXCH];
  __shared__ double red[9];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = cl > 1 ? (int)cluster_rank() : 0;
  const int b = blockIdx.y;
  const int c0 = rank * CH;
  const int E = CH / 256;
  pdl_trigger();
  pdl_wait();
  float v[4];
  double ss = 0.0;
  const float* yr = y + (int64_t)b * ldy + c0 + tid * E;
  if (E == 4) {
    const float4 q = *reinterpret_cast<const float4*>(yr);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) v[e] = yr[e];
  }
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (e < E) ss += (double)v[e] * (double)v[e];
  ss = warp_sum_d(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    red[8] = t;
  }
  double tot = 0.0;
  if (cl > 1) {
    cluster_sync();
    const uint32_t ra = smem_u32(red + 8);
    double parts[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) parts[r] = r < cl ? ld_dsmem_f64_nv(map_peer(ra, r)) : 0.0;
#pragma unroll
    for (int r = 0; r < 8; ++r) tot += parts[r];
  } else {
    __syncthreads();
    tot = red[8];
  }
  const float ms = (float)(tot / (double)di);
  const float rf = __fdiv_rn(1.0f, sqrtf(__fadd_rn(ms, P.eps)));
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (e < E) v[e] = __fmul_rn(__fmul_rn(v[e], rf), P.norm_w[c0 + tid * E + e]);
  const int hb = P.hadamard ? blk : 1;
  const int hin = hb < CH ? hb : CH;   // stages h < hin stay inside the CTA
#pragma unroll
  for (int h = 1; h < 4; h <<= 1)
    if (h < E && h < hin) {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < E && (e & h) == 0) {
          const float x0 = v[e], x1 = v[e + h];
          v[e] = __fadd_rn(x0, x1);
          v[e + h] = __fsub_rn(x0, x1);
        }
    }
  for (int m = 1; m < 32 && E * m < hin; m <<= 1) {
    const bool upper = (lane & m) != 0;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) {
        const float o = __shfl_xor_sync(0xffffffffu, v[e], m);
        v[e] = upper ? __fsub_rn(o, v[e]) : __fadd_rn(v[e], o);
      }
  }
  if (32 * E < hin) {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) ys[tid * E + e] = v[e];
    __syncthreads();
    for (int h = 32 * E, lg = __ffs(32 * E) - 1; h < hin; h <<= 1, ++lg) {
      for (int idx = tid; idx < CH / 2; idx += 256) {
        const int i0 = ((idx >> lg) << (lg + 1)) | (idx & (h - 1));
        const float x0 = ys[i0], x1 = ys[i0 + h];
        ys[i0] = __fadd_rn(x0, x1);
        ys[i0 + h] = __fsub_rn(x0, x1);
      }
      __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) v[e] = ys[tid * E + e];
  }
  if (hb > CH) {   // stages across the cluster: the Hadamard block spans nb CTAs
    const int nb = hb / CH;
    const int base = (rank / nb) * nb;
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) ys[tid * E + e] = v[e];
    cluster_sync();
    float w[8][4];
    const uint32_t ad = smem_u32(ys + tid * E);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < nb) {
        if (E == 4) {
          const float4 q = ld_dsmem_f32x4(map_peer(ad, base + j));
          w[j][0] = q.x; w[j][1] = q.y; w[j][2] = q.z; w[j][3] = q.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < E) w[j][e] = ld_dsmem_f32(map_peer(ad + e * 4, base + j));
        }
      }
#pragma unroll
    for (int h = 1; h < 8; h <<= 1)
      if (h < nb) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < nb && (j & h) == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x0 = w[j][e], x1 = w[j + h][e];
              w[j][e] = __fadd_rn(x0, x1);
              w[j + h][e] = __fsub_rn(x0, x1);
            }
          }
      }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (base + j == rank) {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = w[j][e];
      }
  }
  int8_t* yo = yq + (int64_t)b * ldyq + c0 + tid * E;
  if (E == 4) {
    *reinterpret_cast<uint32_t*>(yo) = (uint32_t)(uint8_t)quant8(v[0], P.s_y) |
                                       ((uint32_t)(uint8_t)quant8(v[1], P.s_y) << 8) |
                                       ((uint32_t)(uint8_t)quant8(v[2], P.s_y) << 16) |
                                       ((uint32_t)(uint8_t)quant8(v[3], P.s_y) << 24);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (e < E) yo[e] = quant8(v[e], P.s_y);
  }
  if (cl > 1) cluster_sync();   // peers may still be reading this CTA's smem
}

// ------------------------------------------------------------------ K6 (d_inner = 8192): one CTA per row
// 256 threads x 32 values.  The 13 Sylvester stages run in three register phases, bits
// [0,5) on each thread's contiguous 32 values, bits [5,10) and [10,13) after two swizzled
// smem transposes (chunk q of 4 floats stored at q ^ ((q >> 3) & 7): conflict-free for the
// contiguous, stride-32 and stride-1024 access patterns).  Same butterflies, same order as
// the oracle; the RMS sum is f64.
__device__ __forceinline__ int had_swz(int i) {   // float index -> swizzled float index
  const int q = i >> 2;
  return ((q ^ ((q >> 3) & 7)) << 2) | (i & 3);
}

// One Sylvester stage of stride h (h >= 2) over 32 register values with packed f32x2 ops:
// lanes (e, e+1) and (e+h, e+h+1) butterfly together; a - b as fma(b, -1, a) rounds like
// the oracle's f32 subtraction.
template <int H>
__device__ __forceinline__ void had_stage32(float (&v)[32]) {
  const float2 M1 = make_float2(-1.f, -1.f);
#pragma unroll
  for (int e = 0; e < 32; e += 2)
    if ((e & H) == 0) {
      const float2 a = make_float2(v[e], v[e + 1]), b = make_float2(v[e + H], v[e + H + 1]);
      const float2 s = __fadd2_rn(a, b), d = __ffma2_rn(b, M1, a);
      v[e] = s.x; v[e + 1] = s.y; v[e + H] = d.x; v[e + H + 1] = d.y;
    }
}
__device__ __forceinline__ void had_stage32_h1(float (&v)[32]) {
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    const float x0 = v[e], x1 = v[e + 1];
    v[e] = __fadd_rn(x0, x1);
    v[e + 1] = __fsub_rn(x0, x1);
  }
}
__device__ __forceinline__ void had_5stages(float (&v)[32]) {
  had_stage32_h1(v);
  had_stage32<2>(v);
  had_stage32<4>(v);
  had_stage32<8>(v);
  had_stage32<16>(v);
}

__global__ void __launch_bounds__(256) norm_had8192_kernel(const sq_mamba2_decode_params P, const float* y,
                                                          int64_t ldy, int8_t* __restrict__ yq, int64_t ldyq,
                                                          int32_t* __restrict__ gsum, int64_t ldg) {
  constexpr int D = 8192;
  __shared__ __align__(16) float buf[D];
  __shared__ double red[8];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int b = blockIdx.x;
  float v[32];
  const float4* src = reinterpret_cast<const float4*>(y + (int64_t)b * ldy + t * 32);
  const float4* gam = reinterpret_cast<const float4*>(P.norm_w + t * 32);
  float4 gm[8];
  pdl_trigger();
#pragma unroll
  for (int j = 0; j < 8; ++j) gm[j] = __ldg(gam + j);
  pdl_wait();
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 q = src[j];
    v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
  }
  double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < 32; ++e) s4[e & 3] += (double)v[e] * (double)v[e];
  double ss = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  ss = warp_sum_d(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float isy = __frcp_rn(P.s_y);
  const float ms = (float)(tot / (double)D);
  const float rf = __fdiv_rn(1.0f, sqrtf(__fadd_rn(ms, P.eps)));
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 g = gm[j];
    v[4 * j] = __fmul_rn(__fmul_rn(v[4 * j], rf), g.x);
    v[4 * j + 1] = __fmul_rn(__fmul_rn(v[4 * j + 1], rf), g.y);
    v[4 * j + 2] = __fmul_rn(__fmul_rn(v[4 * j + 2], rf), g.z);
    v[4 * j + 3] = __fmul_rn(__fmul_rn(v[4 * j + 3], rf), g.w);
  }
  int8_t* out = yq + (int64_t)b * ldyq;
  if (!P.hadamard) {
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      w[j] = (uint32_t)(uint8_t)quant8_inv(v[4 * j], P.s_y, isy) | ((uint32_t)(uint8_t)quant8_inv(v[4 * j + 1], P.s_y, isy) << 8) |
             ((uint32_t)(uint8_t)quant8_inv(v[4 * j + 2], P.s_y, isy) << 16) | ((uint32_t)(uint8_t)quant8_inv(v[4 * j + 3], P.s_y, isy) << 24);
    *reinterpret_cast<uint4*>(out + t * 32) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(out + t * 32 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
    return;
  }
  // phase A: bits 0..4 (contiguous values of this thread)
  had_5stages(v);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<float4*>(buf + had_swz(t * 32 + 4 * j)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  __syncthreads();
  // phase B: bits 5..9; thread holds i = (t_hi << 10) | (k << 5) | t_lo
  const int tlo = t & 31, thi = t >> 5;
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = buf[had_swz((thi << 10) | (k << 5) | tlo)];
  had_5stages(v);
#pragma unroll
  for (int k = 0; k < 32; ++k) buf[had_swz((thi << 10) | (k << 5) | tlo)] = v[k];
  __syncthreads();
  // phase C: bits 10..12; thread holds i = (m << 10) | (t << 2) | j
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const float4 q = *reinterpret_cast<const float4*>(buf + had_swz((m << 10) | (t << 2)));
    v[4 * m] = q.x; v[4 * m + 1] = q.y; v[4 * m + 2] = q.z; v[4 * m + 3] = q.w;
  }
  // stages h = 4, 8, 16 in units of the 4-value groups (value index 4m + j): packed pairs
  had_stage32<4>(v);
  had_stage32<8>(v);
  had_stage32<16>(v);
  const float2 is2 = make_float2(isy, isy);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    bool tie = false;
    uint32_t code = quant8x4_fast(make_float2(v[4 * m], v[4 * m + 1]), make_float2(v[4 * m + 2], v[4 * m + 3]), is2,
                                  is2, tie);
    if (tie)   // rare: a value within 1e-4 of a rounding tie -> exact division
      code = (uint32_t)(uint8_t)quant8(v[4 * m], P.s_y) | ((uint32_t)(uint8_t)quant8(v[4 * m + 1], P.s_y) << 8) |
             ((uint32_t)(uint8_t)quant8(v[4 * m + 2], P.s_y) << 16) |
             ((uint32_t)(uint8_t)quant8(v[4 * m + 3], P.s_y) << 24);
    *reinterpret_cast<uint32_t*>(out + ((m << 10) | (t << 2))) = code;
    if (gsum) {   // 128-wide block (m << 3) | warp holds exactly this warp's 32 x 4 codes
      int cs = __dp4a((int)code, 0x01010101, 0);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, o);
      if (lane == 0) gsum[(int64_t)b * ldg + ((m << 3) | warp)] = cs;
    }
  }
}

}  // namespace sq

using namespace sq;

extern "C" int64_t sq_mamba2_decode_ws_bytes(const sq_mamba2_decode_params* p, int B) {
  if (!p || B < 0) return -1;
  return ds_ws_floats(B, p->ssm.n_heads, p->ssm.n_groups, p->ssm.d_state) * 4;
}

extern "C" int sq_mamba2_decode_launches(const sq_mamba2_decode_params* p, int B, int with_gsum) {
  if (!p || B < 0) return -1;
  if (B == 0) return 0;
  const int di = p->ssm.n_heads * DS_P;
  // prep + state ring + norm, plus the group-sum pass unless the 8192-wide Hadamard norm fuses it
  return 3 + (with_gsum && !(di == 8192 && p->hadamard));
}

extern "C" int sq_mamba2_decode_step_int8(const sq_mamba2_decode_params* p, int B, const int8_t* zx, int64_t ldzx,
                                          int8_t* conv_cache, int8_t* state, void* ws, float* y, int64_t ldy,
                                          int8_t* yq, int64_t ldyq, int32_t* yq_gsum, int64_t ldg, void* stream) {
  SQ_REQUIRE(p && B >= 0 && ws && y && yq, SQ_ERR_ARG, "sq_mamba2_decode_step_int8: bad args");
  const sq_mamba2_params& S = p->ssm;
  SQ_REQUIRE(S.head_dim == DS_P, SQ_ERR_SHAPE, "sq_mamba2_decode_step_int8: head_dim must be 64 (got %d)", S.head_dim);
  SQ_REQUIRE(S.d_state == 64 || S.d_state == 128, SQ_ERR_SHAPE,
             "sq_mamba2_decode_step_int8: d_state must be 64 or 128 (got %d)", S.d_state);
  SQ_REQUIRE(p->conv_kernel >= 1 && p->conv_kernel <= 8, SQ_ERR_SHAPE, "sq_mamba2_decode_step_int8: conv kernel");
  SQ_REQUIRE((reinterpret_cast<uintptr_t>(state) & 15) == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0,
             SQ_ERR_LAYOUT, "sq_mamba2_decode_step_int8: state / ws must be 16-B aligned");
  const int di = S.n_heads * DS_P;
  const int GN = S.n_groups * S.d_state;
  const int C = di + 2 * GN;
  // norm CTAs: <= 1024 channels each, at most 8 per cluster, a multiple of 256 channels
  int CH = 0;
  for (int ch = 256; ch <= DS_MAXCH; ch += 256)
    if (di % ch == 0 && di / ch <= 8) {
      CH = ch;
      break;
    }
  SQ_REQUIRE(CH > 0, SQ_ERR_SHAPE, "sq_mamba2_decode_step_int8: d_inner=%d has no <=8-CTA split", di);
  const int cl = di / CH;
  const int blk = di & -di;
  SQ_REQUIRE(blk <= CH || (blk % CH == 0 && blk / CH <= cl), SQ_ERR_SHAPE,
             "sq_mamba2_decode_step_int8: Hadamard block %d vs CTA width %d", blk, CH);
  SQ_REQUIRE(ldy % 4 == 0 && ldyq % 4 == 0, SQ_ERR_LAYOUT, "sq_mamba2_decode_step_int8: ldy / ldyq alignment");
  if (B == 0) return SQ_OK;
  cudaStream_t st = as_stream(stream);
  float* wsf = reinterpret_cast<float*>(ws);
  constexpr int stages = SQ_DECODE_STAGES;
  const int vec = p->conv_kernel == 4 && C % 4 == 0 && ldzx % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(zx) & 3) == 0 && (reinterpret_cast<uintptr_t>(conv_cache) & 3) == 0;
  const int per_blk = vec ? 1024 : 256;
  if (stages & 1)
    launch_k(PDL_PREP, prep_kernel, dim3((C + per_blk - 1) / per_blk, B), dim3(256), 0, st, *p, C, di, GN, zx, ldzx, conv_cache,
             wsf, B, vec);
  auto ring = [&](auto kern, int smem) {
    // per device (a process may drive several GPUs): smem attribute + resident-CTA count
    static std::once_flag once[2][64];
    static int grid_cache[2][64];
    int dev = 0;
    cudaGetDevice(&dev);
    const int kind = smem == SrCfg<128>::SMEM ? 1 : 0;
    std::call_once(once[kind][dev & 63], [&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int per_sm = 0, sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SR_THREADS, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
      grid_cache[kind][dev & 63] = sms * per_sm;
    });
    const int g = grid_cache[kind][dev & 63];
    const int tiles = B * S.n_heads;
    launch_k(PDL_RING, kern, dim3(tiles < g ? tiles : g), dim3(SR_THREADS), smem, st, S, B, (const float*)wsf, state, y, ldy);
  };
  if (stages & 2) {
    if (S.d_state == 128)
      ring(state_ring_kernel<128>, SrCfg<128>::SMEM);
    else
      ring(state_ring_kernel<64>, SrCfg<64>::SMEM);
  }
  if (!(stages & 4)) return check_launch("sq_mamba2_decode_step_int8");
  SQ_REQUIRE(!yq_gsum || (di % 128 == 0 && ldg >= di / 128), SQ_ERR_SHAPE, "sq_mamba2_decode_step_int8: ldg");
  if (di == 8192 && ldy % 4 == 0 && ldyq % 16 == 0) {
    launch_k(PDL_NORM, norm_had8192_kernel, dim3(B), dim3(256), 0, st, *p, (const float*)y, ldy, yq, ldyq,
             p->hadamard ? yq_gsum : nullptr, ldg);
    if (yq_gsum && !p->hadamard) return launch_group_sum(yq, ldyq, B, di, yq_gsum, ldg, st);
    return check_launch("sq_mamba2_decode_step_int8");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, B, 1);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (cl > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cl;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled(PDL_NORM)) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, norm_had_kernel, *p, di, CH, cl, blk, (const float*)y, ldy, yq, ldyq);
  if (e != cudaSuccess) {
    set_error("sq_mamba2_decode_step_int8 launch: %s", cudaGetErrorString(e));
    return SQ_ERR_CUDA;
  }
  if (yq_gsum) return launch_group_sum(yq, ldyq, B, di, yq_gsum, ldg, st);
  return check_launch("sq_mamba2_decode_step_int8");
}


