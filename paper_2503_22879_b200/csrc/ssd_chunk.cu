// K7: int8 SSD chunk scan for Mamba2 prefill on the tensor cores (ssm_block.ssd_chunked,
// SPEC.md:308-316; "8-bit SSD"; Table 3 shapes PAPER.md:254).
//
// One CTA per (sequence, head), 4 warps, chunks of Q = 64 tokens processed in order with the
// head's state H [P=64 x N] resident in the MMA accumulator registers across chunks:
//
//   CB[t,s]  = Ĉ_t · B̂_s                       int8 x int8 -> int32 (m16n8k32), exact
//   W[t,s]   = CB · s_B s_C · exp(cs_t - cs_s) · Δ_s   (s <= t)     f32 -> fp16, kept in
//              registers: the CB accumulator fragments are reused as the A operand
//   Y_diag   = W · Xcodes                      fp16 x fp16 (x codes exact) -> f32, × s_x[p]
//   Y_off    = exp(cs_t) s_C · (Ccodes · Hᵀ)   fp16 (H rounded to fp16) -> f32
//   y        = (Y_diag + Y_off + D x̂) · SiLU(ẑ)
//   H        = exp(cs_Q) H + Σ_s (e^{cs_Q-cs_s} Δ_s s_x[p] s_B x_s[p]) B_s
//              the float weights are split fp16 hi + lo, so the state update keeps ~f32
//              precision (two m16n8k16 MMAs per step) and the int8 state codes written at
//              the end stay within one step of the sequential f32 recurrence.
// cs = cumulative Δ·A inside the chunk (f32).  Legacy warp-level mma.sync; the operands are
// staged in padded (bank-conflict-free) shared memory and converted to fp16 on the fly.
#include <cuda_fp16.h>

#include "common.cuh"

namespace sq {

constexpr int SC_Q = 64;       // chunk length
constexpr int SC_P = 64;       // head_dim
constexpr int SC_THREADS = 128;

__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_i8(int (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ uint32_t h2(float lo, float hi) {   // pack two f32 as fp16x2 (lo in low half)
  const __half2 v = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t s8pair_h2(const int8_t* p) {   // two consecutive int8 -> fp16x2 (exact)
  return h2((float)p[0], (float)p[1]);
}

template <int N>
struct ScSmem {
  static constexpr int CP = N + 16;       // padded row bytes of C / B codes [t][n]
  static constexpr int TP = SC_Q + 8;     // padded row bytes of transposed codes [*][s]
  int8_t Cs[SC_Q][CP];                    // C codes [t][n]
  int8_t Bs[SC_Q][CP];                    // B codes [s][n]
  int8_t BT[N][TP];                       // B codes [n][s]
  int8_t XT[SC_P][TP];                    // x codes [p][s]
  int8_t Zs[SC_Q][SC_P + 16];             // z codes [t][p]
  __half Hs[SC_P][N + 8];                 // H (fp16 copy) [p][n]
  float cs[SC_Q], dlt[SC_Q], wgt[SC_Q];
  float sxs[SC_P];                        // clustered x scales of the head's channels
  float gz[SC_Q][SC_P + 1];               // SiLU(ẑ) [t][p]
};

template <int N>
__global__ void __launch_bounds__(SC_THREADS) ssd_chunk_kernel(sq_mamba2_params p, int T, const int8_t* x, int64_t ldx,
                                                              const int8_t* Bm, const int8_t* Cm, int64_t ldbc,
                                                              const int8_t* dt, int64_t lddt, const int8_t* z,
                                                              int64_t ldz, int8_t* __restrict__ state, int state_in,
                                                              float* __restrict__ y, int64_t ldy) {
  using S = ScSmem<N>;
  constexpr int NT = N / 8;               // n-tiles of the state (8 columns each)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const int h = blockIdx.x, b = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g4 = lane >> 2, t4 = lane & 3;   // fragment row / column-pair indices
  const int grp = p.head_group[h];
  const float A = p.A[h], Dh = p.D[h], dtb = p.dt_bias[h];
  const float sB = p.s_B[grp], sC = p.s_C[grp];
  const float sBC = __fmul_rn(sB, sC);
  const int ch0 = h * SC_P;
  // this warp's 16 state rows p = 16*warp + {g4, g4+8}; H fragments over all N columns
  const int pr0 = 16 * warp + g4, pr1 = pr0 + 8;
  const float sx0 = p.s_x[ch0 + pr0], sx1 = p.s_x[ch0 + pr1];
  const float sh0 = p.s_h[ch0 + pr0], sh1 = p.s_h[ch0 + pr1];
  float H[NT][4];
  int8_t* st = state + ((int64_t)b * p.n_heads + h) * SC_P * N;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int n = 8 * j + 2 * t4;
    if (state_in) {
      H[j][0] = __fmul_rn((float)st[pr0 * N + n], sh0);
      H[j][1] = __fmul_rn((float)st[pr0 * N + n + 1], sh0);
      H[j][2] = __fmul_rn((float)st[pr1 * N + n], sh1);
      H[j][3] = __fmul_rn((float)st[pr1 * N + n + 1], sh1);
    } else {
      H[j][0] = H[j][1] = H[j][2] = H[j][3] = 0.f;
    }
  }
  // per-thread y rows t = 16*warp + {g4, g4+8}; columns p = 8*j + 2*t4 (+1)
  const int tr0 = 16 * warp + g4, tr1 = tr0 + 8;
  if (tid < SC_P) sm.sxs[tid] = p.s_x[ch0 + tid];

  for (int c0 = 0; c0 < T; c0 += SC_Q) {
    const int Qc = min(SC_Q, T - c0);
    // ---------------- stage the chunk's codes
    __syncthreads();   // previous chunk done with smem
    for (int i = tid; i < SC_Q * (N / 16); i += SC_THREADS) {
      const int r = i / (N / 16), c16 = (i % (N / 16)) * 16;
      int4 bv = make_int4(0, 0, 0, 0), cv = make_int4(0, 0, 0, 0);
      if (r < Qc) {
        const int64_t tok = (int64_t)b * T + c0 + r;
        bv = *reinterpret_cast<const int4*>(Bm + tok * ldbc + grp * N + c16);
        cv = *reinterpret_cast<const int4*>(Cm + tok * ldbc + grp * N + c16);
      }
      *reinterpret_cast<int4*>(&sm.Bs[r][c16]) = bv;
      *reinterpret_cast<int4*>(&sm.Cs[r][c16]) = cv;
      const int8_t* bb = reinterpret_cast<const int8_t*>(&bv);
#pragma unroll
      for (int e = 0; e < 16; ++e) sm.BT[c16 + e][r] = bb[e];
    }
    for (int i = tid; i < SC_Q * (SC_P / 16); i += SC_THREADS) {
      const int r = i / (SC_P / 16), c16 = (i % (SC_P / 16)) * 16;
      int4 xv = make_int4(0, 0, 0, 0), zv = make_int4(0, 0, 0, 0);
      if (r < Qc) {
        const int64_t tok = (int64_t)b * T + c0 + r;
        xv = *reinterpret_cast<const int4*>(x + tok * ldx + ch0 + c16);
        zv = *reinterpret_cast<const int4*>(z + tok * ldz + ch0 + c16);
      }
      *reinterpret_cast<int4*>(&sm.Zs[r][c16]) = zv;
      const int8_t* xb = reinterpret_cast<const int8_t*>(&xv);
#pragma unroll
      for (int e = 0; e < 16; ++e) sm.XT[c16 + e][r] = xb[e];
    }
    if (tid < SC_Q) {
      float dA_log = 0.f, dl = 0.f;
      if (tid < Qc) {
        const float draw = __fadd_rn(__fmul_rn((float)dt[((int64_t)b * T + c0 + tid) * lddt + h], p.s_dt), dtb);
        dl = softplus_f(draw);
        dA_log = __fmul_rn(dl, A);
      }
      sm.dlt[tid] = dl;
      sm.cs[tid] = dA_log;
    }
    __syncthreads();
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
      // state-update weights e^{cs_Q - cs_s} Δ_s (padded tokens have Δ = 0)
      const float csQ = __shfl_sync(0xffffffffu, v1, 31);
      sm.wgt[lane] = __fmul_rn(expf(__fsub_rn(csQ, v0)), sm.dlt[lane]);
      sm.wgt[lane + 32] = __fmul_rn(expf(__fsub_rn(csQ, v1)), sm.dlt[lane + 32]);
    }
    // SiLU(ẑ) table and H (fp16) for Y_off, written from the register-resident state
    for (int i = tid; i < SC_Q * SC_P; i += SC_THREADS) {
      const int t = i / SC_P, pp = i % SC_P;
      sm.gz[t][pp] = silu_fast(__fmul_rn((float)sm.Zs[t][pp], p.s_z));
    }
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int n = 8 * j + 2 * t4;
      *reinterpret_cast<__half2*>(&sm.Hs[pr0][n]) = __floats2half2_rn(H[j][0], H[j][1]);
      *reinterpret_cast<__half2*>(&sm.Hs[pr1][n]) = __floats2half2_rn(H[j][2], H[j][3]);
    }
    __syncthreads();
    const float csQ = sm.cs[SC_Q - 1];   // padded tokens carry Δ = 0

    // ---------------- CB = C · Bᵀ (int8, exact), rows t of this warp, all s
    int cb[SC_Q / 8][4];
#pragma unroll
    for (int j = 0; j < SC_Q / 8; ++j) cb[j][0] = cb[j][1] = cb[j][2] = cb[j][3] = 0;
#pragma unroll
    for (int kk = 0; kk < N / 32; ++kk) {
      uint32_t a[4];
      a[0] = *reinterpret_cast<const uint32_t*>(&sm.Cs[tr0][32 * kk + 4 * t4]);
      a[1] = *reinterpret_cast<const uint32_t*>(&sm.Cs[tr1][32 * kk + 4 * t4]);
      a[2] = *reinterpret_cast<const uint32_t*>(&sm.Cs[tr0][32 * kk + 16 + 4 * t4]);
      a[3] = *reinterpret_cast<const uint32_t*>(&sm.Cs[tr1][32 * kk + 16 + 4 * t4]);
#pragma unroll
      for (int j = 0; j < SC_Q / 8; ++j) {
        uint32_t bf[2];
        bf[0] = *reinterpret_cast<const uint32_t*>(&sm.Bs[8 * j + g4][32 * kk + 4 * t4]);
        bf[1] = *reinterpret_cast<const uint32_t*>(&sm.Bs[8 * j + g4][32 * kk + 16 + 4 * t4]);
        mma_i8(cb[j], a, bf);
      }
    }
    // ---------------- W = CB s_B s_C e^{cs_t - cs_s} Δ_s (causal) -> fp16 A fragments
    const float cst0 = sm.cs[tr0], cst1 = sm.cs[tr1];
    uint32_t wa[SC_Q / 16][4];
#pragma unroll
    for (int j = 0; j < SC_Q / 8; ++j) {
      const int s0 = 8 * j + 2 * t4, s1 = s0 + 1;
      const float css0 = sm.cs[s0], css1 = sm.cs[s1], d0 = sm.dlt[s0], d1 = sm.dlt[s1];
      const float w00 = s0 <= tr0 ? __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][0], sBC), expf(cst0 - css0)), d0) : 0.f;
      const float w01 = s1 <= tr0 ? __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][1], sBC), expf(cst0 - css1)), d1) : 0.f;
      const float w10 = s0 <= tr1 ? __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][2], sBC), expf(cst1 - css0)), d0) : 0.f;
      const float w11 = s1 <= tr1 ? __fmul_rn(__fmul_rn(__fmul_rn((float)cb[j][3], sBC), expf(cst1 - css1)), d1) : 0.f;
      // C-fragment of n-tile j -> A-fragment of k-step j/2 (cols 16kk + {2t4, 2t4+8})
      wa[j >> 1][(j & 1) * 2 + 0] = h2(w00, w01);
      wa[j >> 1][(j & 1) * 2 + 1] = h2(w10, w11);
    }
    // ---------------- Y = W · X  +  C · Hᵀ  (f32 accumulators, rows t, cols p)
    float yd[SC_P / 8][4], yo[SC_P / 8][4];
#pragma unroll
    for (int j = 0; j < SC_P / 8; ++j) {
      yd[j][0] = yd[j][1] = yd[j][2] = yd[j][3] = 0.f;
      yo[j][0] = yo[j][1] = yo[j][2] = yo[j][3] = 0.f;
    }
#pragma unroll
    for (int kk = 0; kk < SC_Q / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < SC_P / 8; ++j) {
        uint32_t bf[2];
        bf[0] = s8pair_h2(&sm.XT[8 * j + g4][16 * kk + 2 * t4]);
        bf[1] = s8pair_h2(&sm.XT[8 * j + g4][16 * kk + 8 + 2 * t4]);
        mma_f16(yd[j], wa[kk], bf);
      }
    }
#pragma unroll
    for (int kk = 0; kk < N / 16; ++kk) {
      uint32_t a[4];
      a[0] = s8pair_h2(&sm.Cs[tr0][16 * kk + 2 * t4]);
      a[1] = s8pair_h2(&sm.Cs[tr1][16 * kk + 2 * t4]);
      a[2] = s8pair_h2(&sm.Cs[tr0][16 * kk + 8 + 2 * t4]);
      a[3] = s8pair_h2(&sm.Cs[tr1][16 * kk + 8 + 2 * t4]);
#pragma unroll
      for (int j = 0; j < SC_P / 8; ++j) {
        uint32_t bf[2];
        bf[0] = *reinterpret_cast<const uint32_t*>(&sm.Hs[8 * j + g4][16 * kk + 2 * t4]);
        bf[1] = *reinterpret_cast<const uint32_t*>(&sm.Hs[8 * j + g4][16 * kk + 8 + 2 * t4]);
        mma_f16(yo[j], a, bf);
      }
    }
    {
      const float e0 = __fmul_rn(expf(cst0), sC), e1 = __fmul_rn(expf(cst1), sC);
#pragma unroll
      for (int j = 0; j < SC_P / 8; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int t = q < 2 ? tr0 : tr1;
          const int pp = 8 * j + 2 * t4 + (q & 1);
          if (t < Qc) {
            const float sxp = sm.sxs[pp];
            const float xh = __fmul_rn((float)sm.XT[pp][t], sxp);
            const float yv = __fadd_rn(__fadd_rn(__fmul_rn(yd[j][q], sxp), __fmul_rn(yo[j][q], q < 2 ? e0 : e1)),
                                       __fmul_rn(Dh, xh));
            y[((int64_t)b * T + c0 + t) * ldy + ch0 + pp] = __fmul_rn(yv, sm.gz[t][pp]);
          }
        }
      }
    }
    // ---------------- H = e^{cs_Q} H + Σ_s w_s s_x s_B x_s ⊗ B_s   (fp16 hi + lo split of the weights)
    const float eQ = expf(csQ);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      H[j][0] = __fmul_rn(H[j][0], eQ);
      H[j][1] = __fmul_rn(H[j][1], eQ);
      H[j][2] = __fmul_rn(H[j][2], eQ);
      H[j][3] = __fmul_rn(H[j][3], eQ);
    }
    const float f0 = __fmul_rn(sx0, sB), f1 = __fmul_rn(sx1, sB);
#pragma unroll
    for (int kk = 0; kk < SC_Q / 16; ++kk) {
      uint32_t ahi[4], alo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int pp = (q & 1) ? pr1 : pr0;
        const int s = 16 * kk + ((q & 2) ? 8 : 0) + 2 * t4;
        const float fr = (q & 1) ? f1 : f0;
        const float v0 = __fmul_rn(__fmul_rn(sm.wgt[s], (float)sm.XT[pp][s]), fr);
        const float v1 = __fmul_rn(__fmul_rn(sm.wgt[s + 1], (float)sm.XT[pp][s + 1]), fr);
        const __half2 hi = __floats2half2_rn(v0, v1);
        const float2 hf = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
        ahi[q] = *reinterpret_cast<const uint32_t*>(&hi);
        alo[q] = *reinterpret_cast<const uint32_t*>(&lo);
      }
      // fragment order: a0 (row g, k 2t), a1 (row g+8, k 2t), a2 (row g, k 2t+8), a3 (row g+8, k 2t+8)
      const uint32_t A_hi[4] = {ahi[0], ahi[1], ahi[2], ahi[3]};
      const uint32_t A_lo[4] = {alo[0], alo[1], alo[2], alo[3]};
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        uint32_t bf[2];
        bf[0] = s8pair_h2(&sm.BT[8 * j + g4][16 * kk + 2 * t4]);
        bf[1] = s8pair_h2(&sm.BT[8 * j + g4][16 * kk + 8 + 2 * t4]);
        mma_f16(H[j], A_hi, bf);
        mma_f16(H[j], A_lo, bf);
      }
    }
  }
  // ---------------- final state -> int8 codes (ClusterMap-cell scales)
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int n = 8 * j + 2 * t4;
    st[pr0 * N + n] = quant8(H[j][0], sh0);
    st[pr0 * N + n + 1] = quant8(H[j][1], sh0);
    st[pr1 * N + n] = quant8(H[j][2], sh1);
    st[pr1 * N + n + 1] = quant8(H[j][3], sh1);
  }
}

int launch_ssd_chunk(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
                     const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                     int8_t* state, int state_in, float* y, int64_t ldy, cudaStream_t st) {
  if (p->head_dim != SC_P || (p->d_state != 64 && p->d_state != 128)) return SQ_ERR_ARG;
  if (ldx % 16 || ldbc % 16 || ldz % 16 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(Bm) & 15) || (reinterpret_cast<uintptr_t>(Cm) & 15) ||
      (reinterpret_cast<uintptr_t>(z) & 15))
    return SQ_ERR_ARG;
  dim3 grid(p->n_heads, B);
  if (p->d_state == 128) {
    const int smem = sizeof(ScSmem<128>);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ssd_chunk_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    ssd_chunk_kernel<128><<<grid, SC_THREADS, smem, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state,
                                                          state_in, y, ldy);
  } else {
    const int smem = sizeof(ScSmem<64>);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ssd_chunk_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    ssd_chunk_kernel<64><<<grid, SC_THREADS, smem, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state,
                                                         state_in, y, ldy);
  }
  return check_launch("sq_ssd_scan_int8 (chunked)");
}

}  // namespace sq
