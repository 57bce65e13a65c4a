// K3: W4A16 projection for small-batch decode — bandwidth-bound int4-weight GEMV
// (PAPER.md:302, 696 Marlin/hgemv lineage; "W4A16 dequantizes weights into
// the float path").
//   y[m,n] = Σ_g s_group[n,g] · Σ_{k∈g} w4[n,k] · x[m,k]
// One warp per output row streams the row's packed nibbles with 16-byte coalesced loads;
// the activation rows (M ≤ 16 per pass) are staged once per CTA in shared memory.
#include "common.cuh"

namespace sq {


// Tiled-layout GEMV (K % 128 == 0; layout of sq_repack_w4): a CTA owns 128 weight rows;
// warp w reads row quadrant (w & 3) and K-half (w >> 2) of every 128-wide K-block, so a
// warp's loads cover 512 contiguous bytes; the activation rows sit in smem (broadcast).
template <int MT>
__global__ void __launch_bounds__(256) gemv_w4a16_tiled_kernel(const float* __restrict__ x, int64_t ldx,
                                                               const uint8_t* __restrict__ w,
                                                               const float* __restrict__ sgrp, int group, int M,
                                                               int N, int K, float* __restrict__ out, int64_t ldo,
                                                               int resid) {
  extern __shared__ float xs[];  // [MT][K]
  __shared__ float part[MT][128];
  for (int i = threadIdx.x; i < MT * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    xs[i] = m < M ? x[(int64_t)m * ldx + k] : 0.f;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, khalf = warp >> 2;
  const int row = q * 32 + lane;
  const int n = blockIdx.x * 128 + row;
  const bool valid = n < N;
  const int nkb = K / 128;
  const int ng = K / group;
  const uint8_t* wsrc = w + (size_t)blockIdx.x * nkb * 8192 + row * 16 + khalf * 2 * 2048;
  const float* srow = sgrp + (size_t)(valid ? n : 0) * ng;
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  constexpr int D = 4;
  int4 buf[D][2];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j < nkb && valid) {
      buf[j][0] = *reinterpret_cast<const int4*>(wsrc + (size_t)j * 8192);
      buf[j][1] = *reinterpret_cast<const int4*>(wsrc + (size_t)j * 8192 + 2048);
    } else {
      buf[j][0] = buf[j][1] = make_int4(0, 0, 0, 0);
    }
  }
  for (int kb0 = 0; kb0 < nkb; kb0 += D) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int kb = kb0 + j;
      if (kb < nkb) {
        int4 cur[2] = {buf[j][0], buf[j][1]};
        if (kb + D < nkb && valid) {
          buf[j][0] = *reinterpret_cast<const int4*>(wsrc + (size_t)(kb + D) * 8192);
          buf[j][1] = *reinterpret_cast<const int4*>(wsrc + (size_t)(kb + D) * 8192 + 2048);
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int k0 = kb * 128 + (khalf * 2 + c) * 32;
          const float s = valid ? srow[k0 / group] : 0.f;
          const uint32_t* pw = reinterpret_cast<const uint32_t*>(&cur[c]);
          float pa[MT];
#pragma unroll
          for (int m = 0; m < MT; ++m) pa[m] = 0.f;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t u = pw[e] ^ 0x88888888u;   // nibble -> v + 8
#pragma unroll
            for (int i4 = 0; i4 < 2; ++i4) {
              float wv[4];
#pragma unroll
              for (int i = 0; i < 4; ++i)
                wv[i] = __uint_as_float(((u >> (8 * i + 4 * i4)) & 0xFu) | 0x4B000000u) - 8388616.0f;   // byte i = e_i | e_{i+4}<<4
#pragma unroll
              for (int m = 0; m < MT; ++m) {
                const float4 xv = *reinterpret_cast<const float4*>(&xs[m * K + k0 + e * 8 + i4 * 4]);
                pa[m] = fmaf(wv[0], xv.x, pa[m]);
                pa[m] = fmaf(wv[1], xv.y, pa[m]);
                pa[m] = fmaf(wv[2], xv.z, pa[m]);
                pa[m] = fmaf(wv[3], xv.w, pa[m]);
              }
            }
          }
#pragma unroll
          for (int m = 0; m < MT; ++m) acc[m] = fmaf(pa[m], s, acc[m]);
        }
      }
    }
  }
  if (khalf == 1) {
#pragma unroll
    for (int m = 0; m < MT; ++m) part[m][row] = acc[m];
  }
  __syncthreads();
  if (khalf == 0 && valid) {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m < M) {
        const float v = acc[m] + part[m][row];
        float* o = out + (int64_t)m * ldo + n;
        *o = resid ? __fadd_rn(*o, v) : v;
      }
    }
  }
}



// Quadrant-split tiled GEMV (K % 128 == 0): a CTA owns one 32-row quadrant of a 128-row
// weight tile (4 CTAs per tile, so small-N projections still fill the GPU); its 8 warps take
// the (k-block, 32-wide chunk) pieces round-robin, lane = row, so each warp load is 512
// contiguous bytes.  Nibbles become floats with a byte-permute into 2^23 + v + 8 and one
// packed subtract; products accumulate in packed f32x2 pairs (short dependency chains); the
// 8 warps' partial row sums are added in fixed warp order (deterministic).
template <int MT, int D>
__global__ void __launch_bounds__(256) gemv_w4a16_q_kernel(const float* x, int64_t ldx,
                                                           const uint8_t* __restrict__ w,
                                                           const float* __restrict__ sgrp, int group, int M, int N,
                                                           int K, float* out, int64_t ldo, int resid) {
  pdl_trigger();
  extern __shared__ __align__(16) float xs[];  // [MT][K]
  __shared__ float part[8][MT][32];
  const int tile = blockIdx.x >> 2, q = blockIdx.x & 3;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = tile * 128 + q * 32 + lane;
  const bool valid = n < N;
  const int nkb = K / 128, ng = K / group;
  const uint8_t* wt = w + (size_t)tile * nkb * 8192 + (q * 32 + lane) * 16;   // + kb*8192 + chunk*2048
  const float* srow = sgrp + (size_t)(valid ? n : 0) * ng;
  const int npieces = nkb * 4;
  // first weight loads before the activation staging (independent of it); D pieces of 512 B
  // in flight per warp (HBM latency × per-SM bandwidth needs tens of KB in flight per SM)
  int4 buf[D];
  float sbuf[D];   // group scale of each in-flight piece, fetched with its weights
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const int pc = warp + 8 * j;
    buf[j] = pc < npieces ? __ldg(reinterpret_cast<const int4*>(wt + (size_t)(pc >> 2) * 8192 + (pc & 3) * 2048))
                          : make_int4(0, 0, 0, 0);
    sbuf[j] = (pc < npieces && valid) ? __ldg(srow + ((pc >> 2) * 128 + (pc & 3) * 32) / group) : 0.f;
  }
  pdl_wait();   // weights and scales above are read-only; x / out come from earlier grids
  // activation staging: batches of 8 loads issued before their smem stores
  for (int i0 = threadIdx.x * 4; i0 < MT * K; i0 += blockDim.x * 4 * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x * 4;
      const int m = i / K, k = i % K;
      v[u] = (i < MT * K && m < M) ? *reinterpret_cast<const float4*>(x + (int64_t)m * ldx + k)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * blockDim.x * 4;
      if (i < MT * K) *reinterpret_cast<float4*>(xs + i) = v[u];
    }
  }
  __syncthreads();
  float acc[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) acc[m] = 0.f;
  const float2 MB = make_float2(-8388616.0f, -8388616.0f);   // 2^23 + 8
  for (int p0 = warp; p0 < npieces; p0 += 8 * D) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int pc = p0 + 8 * j;
      if (pc >= npieces) break;
      const int4 cur = buf[j];
      const float s = sbuf[j];
      const int pn = pc + 8 * D;
      if (pn < npieces) {
        buf[j] = __ldg(reinterpret_cast<const int4*>(wt + (size_t)(pn >> 2) * 8192 + (pn & 3) * 2048));
        sbuf[j] = valid ? __ldg(srow + ((pn >> 2) * 128 + (pn & 3) * 32) / group) : 0.f;
      }
      const int k0 = (pc >> 2) * 128 + (pc & 3) * 32;
      const uint32_t pw[4] = {(uint32_t)cur.x, (uint32_t)cur.y, (uint32_t)cur.z, (uint32_t)cur.w};
      float2 pa[MT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m) pa[m][0] = pa[m][1] = make_float2(0.f, 0.f);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t u = pw[e] ^ 0x88888888u;                       // nibble v -> v + 8
        const uint32_t lo = u & 0x0F0F0F0Fu, hi = (u >> 4) & 0x0F0F0F0Fu;   // elements 0-3 / 4-7
        const float2 w01 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7440)),
                                                  __uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7441))), MB);
        const float2 w23 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7442)),
                                                  __uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7443))), MB);
        const float2 w45 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7440)),
                                                  __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7441))), MB);
        const float2 w67 = __fadd2_rn(make_float2(__uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7442)),
                                                  __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7443))), MB);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const float4 xa = *reinterpret_cast<const float4*>(&xs[m * K + k0 + e * 8]);
          const float4 xb = *reinterpret_cast<const float4*>(&xs[m * K + k0 + e * 8 + 4]);
          pa[m][0] = __ffma2_rn(w01, make_float2(xa.x, xa.y), pa[m][0]);
          pa[m][1] = __ffma2_rn(w23, make_float2(xa.z, xa.w), pa[m][1]);
          pa[m][0] = __ffma2_rn(w45, make_float2(xb.x, xb.y), pa[m][0]);
          pa[m][1] = __ffma2_rn(w67, make_float2(xb.z, xb.w), pa[m][1]);
        }
      }
#pragma unroll
      for (int m = 0; m < MT; ++m)
        acc[m] = fmaf(__fadd_rn(__fadd_rn(pa[m][0].x, pa[m][0].y), __fadd_rn(pa[m][1].x, pa[m][1].y)), s, acc[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < MT; ++m) part[warp][m][lane] = acc[m];
  __syncthreads();
  if (warp == 0 && valid) {
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m < M) {
        float v = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) v = __fadd_rn(v, part[w8][m][lane]);
        float* o = out + (int64_t)m * ldo + n;
        *o = resid ? __fadd_rn(*o, v) : v;
      }
    }
  }
}

template <int MT>
__global__ void __launch_bounds__(256) gemv_w4a16_kernel(const float* __restrict__ x, int64_t ldx,
                                                         const uint8_t* __restrict__ w,
                                                         const float* __restrict__ sgrp, int group, int M, int N,
                                                         int K, float* __restrict__ out, int64_t ldo, int resid) {
  extern __shared__ float xs[];  // [MT][K]
  for (int i = threadIdx.x; i < MT * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    xs[i] = m < M ? x[(int64_t)m * ldx + k] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int ngroups = K / group;
  for (int n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += gridDim.x * warps) {
    const uint8_t* wr = w + (int64_t)n * (K / 2);
    float tot[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) tot[m] = 0.f;
    // each lane handles 32-element chunks (16 packed bytes); a chunk never straddles a group
    for (int c = lane; c < K / 32; c += 32) {
      const int k0 = c * 32;
      const int4 pk = *reinterpret_cast<const int4*>(wr + k0 / 2);
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(&pk);
      float part[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) part[m] = 0.f;
#pragma unroll
      for (int wd = 0; wd < 4; ++wd) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float wv = (float)(((int)(pw[wd] << (28 - 4 * i))) >> 28);
          const int k = k0 + wd * 8 + i;
#pragma unroll
          for (int m = 0; m < MT; ++m) part[m] = fmaf(wv, xs[m * K + k], part[m]);
        }
      }
      const float s = sgrp[(int64_t)n * ngroups + k0 / group];
#pragma unroll
      for (int m = 0; m < MT; ++m) tot[m] = fmaf(part[m], s, tot[m]);
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const float v = warp_sum(tot[m]);
      if (lane == 0 && m < M) {
        float* o = out + (int64_t)m * ldo + n;
        *o = resid ? __fadd_rn(*o, v) : v;
      }
    }
  }
}

}  // namespace sq

using namespace sq;

extern "C" int sq_gemv_w4a16(const float* x, int64_t ldx, const uint8_t* w4, const float* s_group, int group, int M,
                             int N, int K, float* out, int64_t ldo, int resid, void* stream) {
  SQ_REQUIRE(M >= 0 && N > 0 && K > 0 && K % 32 == 0 && group % 32 == 0 && K % group == 0, SQ_ERR_SHAPE,
             "sq_gemv_w4a16: K (%d) and group (%d) must be multiples of 32", K, group);
  cudaStream_t st = as_stream(stream);
  int maxm = (160 * 1024) / (K * 4);
  maxm = maxm >= 8 ? 8 : maxm >= 4 ? 4 : maxm >= 2 ? 2 : 1;
  for (int m0 = 0; m0 < M; m0 += maxm) {
    const int mc = M - m0 < maxm ? M - m0 : maxm;
    const int MT = mc <= 1 ? 1 : (mc <= 2 ? 2 : (mc <= 4 ? 4 : 8));
    const size_t smem = (size_t)MT * K * sizeof(float);
    SQ_REQUIRE(smem <= 200 * 1024, SQ_ERR_SHAPE, "sq_gemv_w4a16: K too large");
    const bool tiled = K % 128 == 0;   // kernel layout of sq_repack_w4
    const bool quad = tiled && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    int blocks = quad ? 4 * ((N + 127) / 128) : tiled ? (N + 127) / 128 : (N + 7) / 8;
    if (!tiled && blocks > 148 * 4) blocks = 148 * 4;
    // few CTAs (small N, e.g. out_proj): each must keep more weight bytes in flight
    const bool deep = MT <= 2 && blocks <= 2 * 148;
#define SQ_GV(MTV)                                                                                  \
  {                                                                                                 \
    auto k = quad ? (deep ? gemv_w4a16_q_kernel<MTV, 16> : gemv_w4a16_q_kernel<MTV, 8>)               \
                  : tiled ? gemv_w4a16_tiled_kernel<MTV> : gemv_w4a16_kernel<MTV>;                    \
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    if (quad)                                                                                       \
      launch_k(PDL_SMALL, k, dim3(blocks), dim3(256), smem, st, x + (int64_t)m0 * ldx, ldx, w4, s_group, \
               group, mc, N, K, out + (int64_t)m0 * ldo, ldo, resid);                               \
    else                                                                                            \
      k<<<blocks, 256, smem, st>>>(x + (int64_t)m0 * ldx, ldx, w4, s_group, group, mc, N, K,        \
                                   out + (int64_t)m0 * ldo, ldo, resid);                            \
  }
    if (MT == 1) SQ_GV(1) else if (MT == 2) SQ_GV(2) else if (MT == 4) SQ_GV(4) else SQ_GV(8)
#undef SQ_GV
  }
  return check_launch("sq_gemv_w4a16");
}
