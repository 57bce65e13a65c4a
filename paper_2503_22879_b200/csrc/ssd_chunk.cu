// K7: int8 SSD chunk scan for Mamba2 prefill on the tensor cores (ssm_block.ssd_chunked,
// SPEC.md:308-316; "8-bit SSD"; Table 3 shapes PAPER.md:254).
//
// One CTA per (sequence, head), 4 warps, chunks of Q = 64 tokens processed in order.  Warp w
// owns the state rows p = 16w .. 16w+15: its slice of H [P=64 x N] stays in MMA accumulator
// registers across chunks, and it produces the transposed outputs Yᵀ[p, t] for those rows:
//
//   CB[t,s]  = Ĉ_t · B̂_s                        int8 x int8 -> int32 (m16n8k32), exact; warp w
//                                                computes rows t = 16w.., all s
//   W[t,s]   = CB s_B s_C e^{cs_t - cs_s} Δ_s  (s <= t)   -> fp16, shared with all warps
//   Y_diagᵀ  = X̂ᵀ · Wᵀ                          fp16 (x codes exact) -> f32, × s_x[p]
//   Y_offᵀ   = H · Ĉᵀ                           fp16 (H rounded to fp16; the accumulator
//                                                fragments are reused as the A operand)
//                                                -> f32, × e^{cs_t} s_C
//   y[t,p]   = (Y_diag + Y_off + D x̂) · SiLU(ẑ)   (SiLU from a 256-entry table of the z codes)
//   H        = e^{cs_Q} H + Σ_s (e^{cs_Q-cs_s} Δ_s s_x[p] s_B x_s[p]) B_s
//              the float weights are split fp16 hi + lo, so the state update keeps ~f32
//              precision (two m16n8k16 MMAs per step) and the int8 state codes written at
//              the end stay within one step of the sequential f32 recurrence.
// cs = cumulative Δ·A inside the chunk (f32).
//
// Data movement: the next chunk's int8 codes are fetched with cp.async into a second raw
// buffer while the current chunk computes; the current chunk's x / B / C codes are widened
// once to fp16 tiles (exact, byte-permute + one HSUB2 per pair) and every fp16 fragment is
// read with ldmatrix (.trans where the reduction runs over tokens).  All padded strides are
// bank-conflict-free for the 8-row ldmatrix phases.  Legacy warp-level mma.sync.
#include <cuda_fp16.h>

#include <mutex>

#include "common.cuh"

namespace sq {

constexpr int SC_Q = 64;       // chunk length
constexpr int SC_P = 64;       // head_dim
constexpr int SC_THREADS = 256;   // 8 warps: (row group w = warp & 3) x (state half nh = warp >> 2)

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_i8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"((uint32_t)__cvta_generic_to_shared(p)));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t h2(float lo, float hi) {   // pack two f32 as fp16x2 (lo in low half)
  const __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ float2 f2(uint32_t v) { return __half22float2(*reinterpret_cast<const __half2*>(&v)); }
// four int8 codes -> two fp16x2 (exact): bytes biased to unsigned, placed under the fp16
// exponent of 1024 (0x64xx = 1024 + byte), then 1152 = 1024 + 128 subtracted.
__device__ __forceinline__ void s8x4_h2x2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t u = w ^ 0x80808080u;
  uint32_t a = __byte_perm(u, 0x64646464u, 0x4140), b = __byte_perm(u, 0x64646464u, 0x4342);
  const __half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
  const __half2 ha = __hsub2(*reinterpret_cast<__half2*>(&a), bias);
  const __half2 hb = __hsub2(*reinterpret_cast<__half2*>(&b), bias);
  lo = *reinterpret_cast<const uint32_t*>(&ha);
  hi = *reinterpret_cast<const uint32_t*>(&hb);
}

template <int N>
struct ScSmem {
  static constexpr int RP = N + 16;       // raw int8 row bytes of B / C codes (conflict-free m16n8k32 loads)
  static constexpr int HP = N + 8;        // fp16 row elements of B / C tiles (conflict-free ldmatrix)
  static constexpr int XP = SC_P + 8;     // fp16 row elements of X / W tiles
  struct Raw {
    int8_t B[SC_Q][RP];                   // B codes [s][n]
    int8_t C[SC_Q][RP];                   // C codes [t][n]
    int8_t X[SC_Q][SC_P];                 // x codes [s][p]
    int8_t Z[SC_Q][SC_P + 16];            // z codes [t][p]
  };
  Raw raw[2];                             // cp.async double buffer (chunk c and c+1)
  __half Bh[SC_Q][HP];                    // B codes [s][n] as fp16
  __half Ch[SC_Q][HP];                    // C codes [t][n] as fp16
  union {
    struct {
      __half Xh[SC_Q][XP];                // x codes [s][p] as fp16
      __half Wh[SC_Q][XP];                // W [t][s] fp16
    };
    float Ys[SC_Q][SC_P + 4];             // pre-gate outputs [t][p], after the Y MMAs
  };
  float cs[SC_Q], dlt[SC_Q], wgt[SC_Q], et[SC_Q];
  float lut[256];                         // SiLU(z_code s_z), indexed by code + 128
};

template <int N>
__global__ void __launch_bounds__(SC_THREADS, 2)
    ssd_chunk_kernel(sq_mamba2_params p, int T, const int8_t* x, int64_t ldx, const int8_t* Bm, const int8_t* Cm,
                     int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                     int8_t* __restrict__ state, int state_in, float* __restrict__ y, int64_t ldy) {
  using S = ScSmem<N>;
  constexpr int NTH = N / 16;             // n-tiles (8 columns) of this warp's state half
  extern __shared__ __align__(16) uint8_t smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const int h = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int w = warp & 3, nh = warp >> 2;    // rows p (and t for C·Bᵀ) 16w..16w+15; state columns half nh
  const int g4 = lane >> 2, t4 = lane & 3;   // fragment row / column-pair indices
  const int mi = lane >> 3, r8 = lane & 7;   // ldmatrix: matrix index / row within it
  const int grp = p.head_group[h];
  const float A = p.A[h], Dh = p.D[h], dtb = p.dt_bias[h];
  const float sB = p.s_B[grp], sC = p.s_C[grp];
  const float sBC = __fmul_rn(sB, sC);
  const int ch0 = h * SC_P;
  const int64_t tok0 = (int64_t)b * T;
  const int n0 = nh * (N / 2);               // first state column of this warp

  // async fetch of one chunk's codes into raw buffer `buf` (rows past T zero-filled)
  auto fetch = [&](int c0, int buf) {
    typename S::Raw& R = sm.raw[buf];
    const int Qc = min(SC_Q, T - c0);
    for (int i = tid; i < SC_Q * (N / 16); i += SC_THREADS) {
      const int r = i / (N / 16), c16 = (i % (N / 16)) * 16;
      const int64_t tok = tok0 + c0 + min(r, Qc - 1);
      cp_async16(&R.B[r][c16], Bm + tok * ldbc + grp * N + c16, r < Qc);
      cp_async16(&R.C[r][c16], Cm + tok * ldbc + grp * N + c16, r < Qc);
    }
    for (int i = tid; i < SC_Q * (SC_P / 16); i += SC_THREADS) {
      const int r = i / (SC_P / 16), c16 = (i % (SC_P / 16)) * 16;
      const int64_t tok = tok0 + c0 + min(r, Qc - 1);
      cp_async16(&R.X[r][c16], x + tok * ldx + ch0 + c16, r < Qc);
      cp_async16(&R.Z[r][c16], z + tok * ldz + ch0 + c16, r < Qc);
    }
    cp_async_commit();
  };
  fetch(0, 0);

  const int pr0 = 16 * w + g4, pr1 = pr0 + 8;
  const float sx0 = p.s_x[ch0 + pr0], sx1 = p.s_x[ch0 + pr1];
  const float sh0 = p.s_h[ch0 + pr0], sh1 = p.s_h[ch0 + pr1];
  float H[NTH][4];   // this warp's slice: rows pr0 / pr1, columns n0 + 8j + 2t4 (+1)
  int8_t* st = state + ((int64_t)b * p.n_heads + h) * SC_P * N;
#pragma unroll
  for (int j = 0; j < NTH; ++j) {
    const int n = n0 + 8 * j + 2 * t4;
    if (state_in) {
      H[j][0] = __fmul_rn((float)st[pr0 * N + n], sh0);
      H[j][1] = __fmul_rn((float)st[pr0 * N + n + 1], sh0);
      H[j][2] = __fmul_rn((float)st[pr1 * N + n], sh1);
      H[j][3] = __fmul_rn((float)st[pr1 * N + n + 1], sh1);
    } else {
      H[j][0] = H[j][1] = H[j][2] = H[j][3] = 0.f;
    }
  }
  for (int i = tid; i < 256; i += SC_THREADS) sm.lut[i] = silu_fast(__fmul_rn((float)(i - 128), p.s_z));
  const float f0 = __fmul_rn(sx0, sB), f1 = __fmul_rn(sx1, sB);
  // per-token Δ code of this thread's token (tid < 64), prefetched one chunk ahead
  // (addresses clamped instead of predicated: no select waits on the load; rows past Qc get Δ = 0)
  int8_t dcode = tid < SC_Q ? dt[(tok0 + min(tid, T - 1)) * lddt + h] : 0;

  int buf = 0;
  for (int c0 = 0; c0 < T; c0 += SC_Q, buf ^= 1) {
    const int Qc = min(SC_Q, T - c0);
    cp_async_wait_all();
    __syncthreads();   // raw[buf] landed for every thread; previous chunk fully consumed
    if (c0 + SC_Q < T) fetch(c0 + SC_Q, buf ^ 1);
    const typename S::Raw& R = sm.raw[buf];
    if (tid < SC_Q) {
      float dA_log = 0.f, dl = 0.f;
      if (tid < Qc) {
        const float draw = __fadd_rn(__fmul_rn((float)dcode, p.s_dt), dtb);
        dl = softplus_f(draw);
        dA_log = __fmul_rn(dl, A);
      }
      sm.dlt[tid] = dl;
      sm.cs[tid] = dA_log;
      dcode = dt[(tok0 + min(c0 + SC_Q + tid, T - 1)) * lddt + h];
    }
    // widen this chunk's x / B / C codes to fp16 tiles: 8 codes (8 B) -> 8 halves (16 B) per
    // thread, consecutive threads on consecutive 16 B (conflict-free stores)
    for (int i = tid; i < SC_Q * (N / 8); i += SC_THREADS) {
      const int r = i / (N / 8), c8 = (i % (N / 8)) * 8;
      const uint2 bv = *reinterpret_cast<const uint2*>(&R.B[r][c8]);
      const uint2 cv = *reinterpret_cast<const uint2*>(&R.C[r][c8]);
      uint4 o;
      s8x4_h2x2(bv.x, o.x, o.y); s8x4_h2x2(bv.y, o.z, o.w);
      *reinterpret_cast<uint4*>(&sm.Bh[r][c8]) = o;
      s8x4_h2x2(cv.x, o.x, o.y); s8x4_h2x2(cv.y, o.z, o.w);
      *reinterpret_cast<uint4*>(&sm.Ch[r][c8]) = o;
    }
    for (int i = tid; i < SC_Q * (SC_P / 8); i += SC_THREADS) {
      const int r = i / (SC_P / 8), c8 = (i % (SC_P / 8)) * 8;
      const uint2 xv = *reinterpret_cast<const uint2*>(&R.X[r][c8]);
      uint4 o;
      s8x4_h2x2(xv.x, o.x, o.y); s8x4_h2x2(xv.y, o.z, o.w);
      *reinterpret_cast<uint4*>(&sm.Xh[r][c8]) = o;
    }
    __syncthreads();   // dlt / cs / fp16 tiles visible
    if (warp == 0) {   // inclusive prefix sum of Δ·A over the chunk (sequential order, f32)
      float v0 = sm.cs[lane], v1 = sm.cs[lane + 32];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float a0 = __shfl_up_sync(0xffffffffu, v0, o), a1 = __shfl_up_sync(0xffffffffu, v1, o);
        if (lane >= o) {
          v0 += a0;
          v1 += a1;
        }
      }
      v1 += __shfl_sync(0xffffffffu, v0, 31);
      sm.cs[lane] = v0;
      sm.cs[lane + 32] = v1;
      // state-update weights e^{cs_Q - cs_s} Δ_s (padded tokens have Δ = 0); Y_off column
      // scales e^{cs_t} s_C
      const float csQ = __shfl_sync(0xffffffffu, v1, 31);
      sm.wgt[lane] = __fmul_rn(expf(__fsub_rn(csQ, v0)), sm.dlt[lane]);
      sm.wgt[lane + 32] = __fmul_rn(expf(__fsub_rn(csQ, v1)), sm.dlt[lane + 32]);
      sm.et[lane] = __fmul_rn(__expf(v0), sC);
      sm.et[lane + 32] = __fmul_rn(__expf(v1), sC);
    }
    // ---------------- CB = C · Bᵀ (int8, exact): rows t = 16w + {g4, g4+8}, s-tiles 4nh..4nh+3
    const int tr0 = 16 * w + g4, tr1 = tr0 + 8;
    int cb[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) cb[j][0] = cb[j][1] = cb[j][2] = cb[j][3] = 0;
#pragma unroll
    for (int kk = 0; kk < N / 32; ++kk) {
      uint32_t a[4];
      a[0] = *reinterpret_cast<const uint32_t*>(&R.C[tr0][32 * kk + 4 * t4]);
      a[1] = *reinterpret_cast<const uint32_t*>(&R.C[tr1][32 * kk + 4 * t4]);
      a[2] = *reinterpret_cast<const uint32_t*>(&R.C[tr0][32 * kk + 16 + 4 * t4]);
      a[3] = *reinterpret_cast<const uint32_t*>(&R.C[tr1][32 * kk + 16 + 4 * t4]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int jg = 4 * nh + j;
        if (jg <= 2 * w + 1)   // s-tiles past this warp's last row are causally masked
          mma_i8(cb[j], a, *reinterpret_cast<const uint32_t*>(&R.B[8 * jg + g4][32 * kk + 4 * t4]),
                 *reinterpret_cast<const uint32_t*>(&R.B[8 * jg + g4][32 * kk + 16 + 4 * t4]));
      }
    }
    __syncthreads();   // cs / wgt / et visible
    // ---------------- W = CB s_B s_C e^{cs_t - cs_s} Δ_s (causal) -> fp16 tile [t][s]
    {
      const float cst0 = sm.cs[tr0], cst1 = sm.cs[tr1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int jg = 4 * nh + j;
        const int s0 = 8 * jg + 2 * t4, s1 = s0 + 1;
        uint32_t wv0 = 0, wv1 = 0;
        if (jg <= 2 * w + 1) {
          const float css0 = sm.cs[s0], css1 = sm.cs[s1], d0 = sm.dlt[s0], d1 = sm.dlt[s1];
          float w00 = __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][0], sBC), __expf(cst0 - css0)), d0);
          float w01 = __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][1], sBC), __expf(cst0 - css1)), d1);
          float w10 = __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][2], sBC), __expf(cst1 - css0)), d0);
          float w11 = __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][3], sBC), __expf(cst1 - css1)), d1);
          w00 = s0 <= tr0 ? w00 : 0.f;
          w01 = s1 <= tr0 ? w01 : 0.f;
          w10 = s0 <= tr1 ? w10 : 0.f;
          w11 = s1 <= tr1 ? w11 : 0.f;
          wv0 = h2(w00, w01);
          wv1 = h2(w10, w11);
        }
        *reinterpret_cast<uint32_t*>(&sm.Wh[tr0][s0]) = wv0;
        *reinterpret_cast<uint32_t*>(&sm.Wh[tr1][s0]) = wv1;
      }
    }
    // X̂ᵀ A fragments (rows p of this warp's group, k = s): Y_diag, the D term and the H update
    uint32_t xa[SC_Q / 16][4];
#pragma unroll
    for (int kk = 0; kk < SC_Q / 16; ++kk)
      ldsm_x4_t(xa[kk], &sm.Xh[16 * kk + (mi >> 1) * 8 + r8][16 * w + (mi & 1) * 8]);
    __syncthreads();   // W visible
    // ---------------- Yᵀ: Y_diag for t-tiles 4nh..4nh+3, Y_off partial over this warp's n half
    float yd[4][4], yo[SC_Q / 8][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) yd[j][0] = yd[j][1] = yd[j][2] = yd[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < SC_Q / 8; ++j) yo[j][0] = yo[j][1] = yo[j][2] = yo[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < SC_Q / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < 4; j += 2) {
        const int jg = 4 * nh + j;
        if (kk > jg / 2) continue;   // W[t][s] = 0 for s > t: t-tiles jg, jg+1 need s < 8jg + 16
        uint32_t bw[4];   // b0,b1 of t-tile jg, then of t-tile jg+1
        ldsm_x4(bw, &sm.Wh[8 * (jg + (mi >> 1)) + r8][16 * kk + (mi & 1) * 8]);
        mma_f16(yd[j], xa[kk], bw[0], bw[1]);
        mma_f16(yd[j + 1], xa[kk], bw[2], bw[3]);
      }
    }
#pragma unroll
    for (int kk = 0; kk < NTH / 2; ++kk) {
      const uint32_t ha[4] = {h2(H[2 * kk][0], H[2 * kk][1]), h2(H[2 * kk][2], H[2 * kk][3]),
                              h2(H[2 * kk + 1][0], H[2 * kk + 1][1]), h2(H[2 * kk + 1][2], H[2 * kk + 1][3])};
#pragma unroll
      for (int j = 0; j < SC_Q / 8; j += 2) {
        uint32_t bc[4];
        ldsm_x4(bc, &sm.Ch[8 * (j + (mi >> 1)) + r8][n0 + 16 * kk + (mi & 1) * 8]);
        mma_f16(yo[j], ha, bc[0], bc[1]);
        mma_f16(yo[j + 1], ha, bc[2], bc[3]);
      }
    }
    // ---------------- epilogue: y[t][p] assembled in smem (over the X / W tiles) in a fixed
    // order — (Y_diag·s_x + (Y_off[n half 0] + Y_off[n half 1])·e^{cs_t} s_C) + D x̂ — then
    // SiLU(ẑ) gating and coalesced 16-byte stores
    __syncthreads();   // every warp done reading Xh / Wh
    if (nh == 1) {
#pragma unroll
      for (int j = 0; j < SC_Q / 8; ++j) {
        const int t = 8 * j + 2 * t4;
        sm.Ys[t][pr0] = yo[j][0];
        sm.Ys[t + 1][pr0] = yo[j][1];
        sm.Ys[t][pr1] = yo[j][2];
        sm.Ys[t + 1][pr1] = yo[j][3];
      }
    }
    __syncthreads();
    auto finish = [&](int j, int jl, float o0, float o1, float o2, float o3) {
      // x codes at (p, t) from the X̂ᵀ fragments: t-tile j = k-step j/2, half j&1
      const float2 xc0 = f2(xa[j >> 1][(j & 1) * 2]), xc1 = f2(xa[j >> 1][(j & 1) * 2 + 1]);
      const int t = 8 * j + 2 * t4;
      const float e0 = sm.et[t], e1 = sm.et[t + 1];
      sm.Ys[t][pr0] = __fadd_rn(__fadd_rn(__fmul_rn(yd[jl][0], sx0), __fmul_rn(o0, e0)), __fmul_rn(Dh, __fmul_rn(xc0.x, sx0)));
      sm.Ys[t + 1][pr0] = __fadd_rn(__fadd_rn(__fmul_rn(yd[jl][1], sx0), __fmul_rn(o1, e1)), __fmul_rn(Dh, __fmul_rn(xc0.y, sx0)));
      sm.Ys[t][pr1] = __fadd_rn(__fadd_rn(__fmul_rn(yd[jl][2], sx1), __fmul_rn(o2, e0)), __fmul_rn(Dh, __fmul_rn(xc1.x, sx1)));
      sm.Ys[t + 1][pr1] = __fadd_rn(__fadd_rn(__fmul_rn(yd[jl][3], sx1), __fmul_rn(o3, e1)), __fmul_rn(Dh, __fmul_rn(xc1.y, sx1)));
    };
    if (nh == 0) {
#pragma unroll
      for (int j = 0; j < SC_Q / 8; ++j) {
        const int t = 8 * j + 2 * t4;
        const float o0 = __fadd_rn(yo[j][0], sm.Ys[t][pr0]), o1 = __fadd_rn(yo[j][1], sm.Ys[t + 1][pr0]);
        const float o2 = __fadd_rn(yo[j][2], sm.Ys[t][pr1]), o3 = __fadd_rn(yo[j][3], sm.Ys[t + 1][pr1]);
        if (j < 4) {
          finish(j, j, o0, o1, o2, o3);
        } else {   // the other half's t-tiles: leave the summed Y_off for it
          sm.Ys[t][pr0] = o0;
          sm.Ys[t + 1][pr0] = o1;
          sm.Ys[t][pr1] = o2;
          sm.Ys[t + 1][pr1] = o3;
        }
      }
    }
    __syncthreads();
    if (nh == 1) {
#pragma unroll
      for (int j = 4; j < SC_Q / 8; ++j) {
        const int t = 8 * j + 2 * t4;
        finish(j, j - 4, sm.Ys[t][pr0], sm.Ys[t + 1][pr0], sm.Ys[t][pr1], sm.Ys[t + 1][pr1]);
      }
    }
    __syncthreads();
    {
      const int p4 = (tid & 15) * 4;
#pragma unroll
      for (int i = 0; i < SC_Q / 16; ++i) {
        const int t = (tid >> 4) + 16 * i;
        if (t < Qc) {
          const float4 v = *reinterpret_cast<const float4*>(&sm.Ys[t][p4]);
          const uint32_t zc = *reinterpret_cast<const uint32_t*>(&R.Z[t][p4]);
          float4 o;
          o.x = __fmul_rn(v.x, sm.lut[(int)(int8_t)(zc) + 128]);
          o.y = __fmul_rn(v.y, sm.lut[(int)(int8_t)(zc >> 8) + 128]);
          o.z = __fmul_rn(v.z, sm.lut[(int)(int8_t)(zc >> 16) + 128]);
          o.w = __fmul_rn(v.w, sm.lut[(int)(int8_t)(zc >> 24) + 128]);
          *reinterpret_cast<float4*>(y + (tok0 + c0 + t) * ldy + ch0 + p4) = o;
        }
      }
    }
    // ---------------- H = e^{cs_Q} H + Σ_s w_s s_x s_B x_s ⊗ B_s   (fp16 hi + lo split of the weights)
    const float eQ = expf(sm.cs[SC_Q - 1]);   // padded tokens carry Δ = 0
#pragma unroll
    for (int j = 0; j < NTH; ++j) {
      H[j][0] = __fmul_rn(H[j][0], eQ);
      H[j][1] = __fmul_rn(H[j][1], eQ);
      H[j][2] = __fmul_rn(H[j][2], eQ);
      H[j][3] = __fmul_rn(H[j][3], eQ);
    }
#pragma unroll
    for (int kk = 0; kk < SC_Q / 16; ++kk) {
      uint32_t ahi[4], alo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {   // a0 (row g, k 2t), a1 (row g+8, k 2t), a2 (row g, k 2t+8), a3 (row g+8, k 2t+8)
        const int s = 16 * kk + ((q & 2) ? 8 : 0) + 2 * t4;
        const float fr = (q & 1) ? f1 : f0;
        const float2 xc = f2(xa[kk][q]);
        const float v0 = __fmul_rn(__fmul_rn(sm.wgt[s], xc.x), fr);
        const float v1 = __fmul_rn(__fmul_rn(sm.wgt[s + 1], xc.y), fr);
        const __half2 hi = __floats2half2_rn(v0, v1);
        const float2 hf = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
        ahi[q] = *reinterpret_cast<const uint32_t*>(&hi);
        alo[q] = *reinterpret_cast<const uint32_t*>(&lo);
      }
      // hi pass over this half's n-tiles, then lo pass: dependent MMAs on one H tile are NTH apart
#pragma unroll
      for (int j = 0; j < NTH; j += 2) {
        uint32_t bb[4];   // b0,b1 of n-tile j, then of n-tile j+1 (stored [s][n] -> .trans)
        ldsm_x4_t(bb, &sm.Bh[16 * kk + (mi & 1) * 8 + r8][n0 + 8 * (j + (mi >> 1))]);
        mma_f16(H[j], ahi, bb[0], bb[1]);
        mma_f16(H[j + 1], ahi, bb[2], bb[3]);
      }
#pragma unroll
      for (int j = 0; j < NTH; j += 2) {
        uint32_t bb[4];
        ldsm_x4_t(bb, &sm.Bh[16 * kk + (mi & 1) * 8 + r8][n0 + 8 * (j + (mi >> 1))]);
        mma_f16(H[j], alo, bb[0], bb[1]);
        mma_f16(H[j + 1], alo, bb[2], bb[3]);
      }
    }
  }
  cp_async_wait_all();
  // ---------------- final state -> int8 codes (ClusterMap-cell scales)
#pragma unroll
  for (int j = 0; j < NTH; ++j) {
    const int n = n0 + 8 * j + 2 * t4;
    st[pr0 * N + n] = quant8(H[j][0], sh0);
    st[pr0 * N + n + 1] = quant8(H[j][1], sh0);
    st[pr1 * N + n] = quant8(H[j][2], sh1);
    st[pr1 * N + n + 1] = quant8(H[j][3], sh1);
  }
}

template <int N>
static int launch_n(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
                    const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                    int8_t* state, int state_in, float* y, int64_t ldy, cudaStream_t st) {
  const int smem = sizeof(ScSmem<N>);
  static std::once_flag once[64];   // per device
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63],
                 [&] { cudaFuncSetAttribute(ssd_chunk_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  ssd_chunk_kernel<N><<<dim3(p->n_heads, B), SC_THREADS, smem, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz,
                                                                    state, state_in, y, ldy);
  return SQ_OK;
}

int launch_ssd_chunk(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
                     const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                     int8_t* state, int state_in, float* y, int64_t ldy, cudaStream_t st) {
  if (p->head_dim != SC_P || (p->d_state != 64 && p->d_state != 128)) return SQ_ERR_ARG;
  if (ldx % 16 || ldbc % 16 || ldz % 16 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(Bm) & 15) || (reinterpret_cast<uintptr_t>(Cm) & 15) ||
      (reinterpret_cast<uintptr_t>(z) & 15))
    return SQ_ERR_ARG;
  if (p->d_state == 128)
    launch_n<128>(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy, st);
  else
    launch_n<64>(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy, st);
  return check_launch("sq_ssd_scan_int8 (chunked)");
}

}  // namespace sq
