// K1/K2 fallback: A8 GEMM on the warp-level tensor path (mma.sync m16n8k32 s8), for the
// shapes the tcgen05 kernels do not take (K not a multiple of 128, e.g. Mamba1 dt_proj K=160).
//
//   W8A8:  acc[m,n] = sum_k a[m,k] * w8[n,k] (exact int32);  y = f32(acc) * alpha[n]
//   W4A8:  per 'group'-wide K slice g: acc_g exact int32, promoted p = fma(s_w[n,g], f32(acc_g), p)
//          (ascending g, one rounding), y = p * s_a — the same arithmetic as the tcgen05
//          W4A8 kernel (gemm_w4a8.cu) and the oracle (qblock.qlinear_a8)
//   epilogue : i32 (W8 only) | f32 | int8 requant by col_scale[n] | residual add (sq_epilogue)
//
// Tile 64 tokens x 128 outputs x 64 K, 4 warps (each 64x32), register double-buffered
// global loads, W4 nibbles sign-extended to int8 on the way into shared memory.
#include "common.cuh"

namespace sq {

constexpr int BM = 64, BN = 128, BK = 64, PADK = BK + 16;

__device__ __forceinline__ uint32_t expand_w4x4(uint32_t packed16) {
  // 2 packed bytes (4 nibbles) -> 4 sign-extended int8
  uint32_t out = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int v = ((int)(packed16 << (28 - 4 * i))) >> 28;
    out |= ((uint32_t)v & 0xFFu) << (8 * i);
  }
  return out;
}

__device__ __forceinline__ void mma_s8(int (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <bool W4>
__global__ void __launch_bounds__(128) gemm_a8_mma_kernel(const int8_t* a, int64_t lda,
                                                          const uint8_t* __restrict__ w,
                                                          const float* __restrict__ ws, int group, float s_a,
                                                          const float* __restrict__ alpha, int M, int N, int K,
                                                          int epi, void* out, int64_t ldo,
                                                          const float* __restrict__ col_scale) {
  pdl_trigger();
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  __shared__ __align__(16) int8_t As[BM][PADK];
  __shared__ __align__(16) int8_t Ws[BN][PADK];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int ngroups = W4 ? K / group : 1;

  int acc[4][4][4];
  float facc[4][4][4];   // W4: promoted per-group partial sums
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[i][j][r] = 0;
        facc[i][j][r] = 0.f;
      }

  // per-thread load assignment
  // A: 64 rows x 64 B = 256 x 16B chunks -> 2 per thread
  // W: 128 rows; thread = row; W8: 64 B (4 chunks); W4: 32 B packed (2 chunks)
  int4 ra[2], rw[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = tid + i * 128;
      const int r = c >> 2, kk = (c & 3) * 16;
      const int gm = m0 + r, gk = k0 + kk;
      ra[i] = (gm < M && gk < K) ? *reinterpret_cast<const int4*>(a + (int64_t)gm * lda + gk) : make_int4(0, 0, 0, 0);
    }
    const int gn = n0 + tid;
    if (W4) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int gk = k0 + i * 32;
        int64_t off;
        if (K % 128 == 0) {   // tiled kernel layout (sq_repack_w4): [tile][kb][chunk][row][16B]
          off = ((((int64_t)(gn >> 7) * (K >> 7) + (gk >> 7)) * 4 + ((gk & 127) >> 5)) * 128 + (gn & 127)) * 16;
        } else {
          off = (int64_t)gn * (K / 2) + gk / 2;
        }
        rw[i] = (gn < N && gk < K) ? *reinterpret_cast<const int4*>(w + off) : make_int4(0, 0, 0, 0);
        if (K % 128 == 0) {   // undo the kernel-layout nibble permutation (byte j = e_j | e_{j+4} << 4)
          uint32_t* pw = reinterpret_cast<uint32_t*>(&rw[i]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            uint32_t x = pw[e], lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;
            lo = (lo | (lo >> 4)) & 0x00FF00FFu; lo = (lo | (lo >> 8)) & 0xFFFFu;
            hi = (hi | (hi >> 4)) & 0x00FF00FFu; hi = (hi | (hi >> 8)) & 0xFFFFu;
            pw[e] = lo | (hi << 16);
          }
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int gk = k0 + i * 16;
        rw[i] = (gn < N && gk < K) ? *reinterpret_cast<const int4*>(w + (int64_t)gn * K + gk) : make_int4(0, 0, 0, 0);
      }
    }
  };
  auto sstore = [&]() {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = tid + i * 128;
      *reinterpret_cast<int4*>(&As[c >> 2][(c & 3) * 16]) = ra[i];
    }
    if (W4) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(&rw[i]);
        int4 o0, o1;
        o0.x = expand_w4x4(p[0] & 0xFFFF);
        o0.y = expand_w4x4(p[0] >> 16);
        o0.z = expand_w4x4(p[1] & 0xFFFF);
        o0.w = expand_w4x4(p[1] >> 16);
        o1.x = expand_w4x4(p[2] & 0xFFFF);
        o1.y = expand_w4x4(p[2] >> 16);
        o1.z = expand_w4x4(p[3] & 0xFFFF);
        o1.w = expand_w4x4(p[3] >> 16);
        *reinterpret_cast<int4*>(&Ws[tid][i * 32]) = o0;
        *reinterpret_cast<int4*>(&Ws[tid][i * 32 + 16]) = o1;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) *reinterpret_cast<int4*>(&Ws[tid][i * 16]) = rw[i];
    }
  };

  const int g = lane >> 2, q = lane & 3;
  gload(0);
  for (int k0 = 0; k0 < K; k0 += BK) {
    __syncthreads();
    sstore();
    __syncthreads();
    if (k0 + BK < K) gload(k0 + BK);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 32) {
      uint32_t af[4][4], bf[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = i * 16 + g;
        af[i][0] = *reinterpret_cast<const uint32_t*>(&As[r][ks + q * 4]);
        af[i][1] = *reinterpret_cast<const uint32_t*>(&As[r + 8][ks + q * 4]);
        af[i][2] = *reinterpret_cast<const uint32_t*>(&As[r][ks + 16 + q * 4]);
        af[i][3] = *reinterpret_cast<const uint32_t*>(&As[r + 8][ks + 16 + q * 4]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int nn = warp * 32 + j * 8 + g;
        bf[j][0] = *reinterpret_cast<const uint32_t*>(&Ws[nn][ks + q * 4]);
        bf[j][1] = *reinterpret_cast<const uint32_t*>(&Ws[nn][ks + 16 + q * 4]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) mma_s8(acc[i][j], af[i], bf[j]);
      if (W4 && (k0 + ks + 32) % group == 0 && k0 + ks < K) {
        // group boundary: promote the exact int32 partials with this group's scales
        const int gi = (k0 + ks) / group;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float sc[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int n = n0 + warp * 32 + j * 8 + q * 2 + e;
            sc[e] = n < N ? ws[((int64_t)(n >> 7) * ngroups + gi) * 128 + (n & 127)] : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              facc[i][j][r] = __fmaf_rn(sc[r & 1], (float)acc[i][j][r], facc[i][j][r]);
              acc[i][j][r] = 0;
            }
        }
      }
    }
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int m = m0 + i * 16 + g + (r >> 1) * 8;
        const int n = n0 + warp * 32 + j * 8 + q * 2 + (r & 1);
        if (m >= M || n >= N) continue;
        const int v = acc[i][j][r];
        const int64_t o = (int64_t)m * ldo + n;
        if (!W4 && epi == SQ_EPI_I32) {
          reinterpret_cast<int32_t*>(out)[o] = v;
        } else {
          const float y = W4 ? __fmul_rn(facc[i][j][r], s_a) : __fmul_rn((float)v, alpha[n]);
          if (epi == SQ_EPI_F32)
            reinterpret_cast<float*>(out)[o] = y;
          else if (epi == SQ_EPI_QUANT)
            reinterpret_cast<int8_t*>(out)[o] = quant8(y, col_scale[n]);
          else
            reinterpret_cast<float*>(out)[o] = __fadd_rn(reinterpret_cast<float*>(out)[o], y);
        }
      }
}

int gemm_a8_mma(const int8_t* a, int64_t lda, const uint8_t* w, const float* ws, int group, float s_a, bool w4,
                const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
                cudaStream_t st) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
  if (w4)
    launch_k(PDL_SMALL8, gemm_a8_mma_kernel<true>, grid, dim3(128), 0, st, a, lda, w, ws, group, s_a, alpha, M, N, K,
             epi, out, ldo, col_scale);
  else
    launch_k(PDL_SMALL8, gemm_a8_mma_kernel<false>, grid, dim3(128), 0, st, a, lda, w, ws, group, s_a, alpha, M, N, K,
             epi, out, ldo, col_scale);
  return check_launch("gemm_a8_mma");
}

}  // namespace sq
