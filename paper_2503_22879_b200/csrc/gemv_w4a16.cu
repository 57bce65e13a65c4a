// K3: W4A16 projection for small-batch decode — bandwidth-bound int4-weight GEMV
// (PAPER.md:302, 696 Marlin/hgemv lineage; "W4A16 dequantizes weights into
// the float path").
//   y[m,n] = Σ_g s_group[n,g] · Σ_{k∈g} w4[n,k] · x[m,k]
// One warp per output row streams the row's packed nibbles with 16-byte coalesced loads;
// the activation rows (M ≤ 16 per pass) are staged once per CTA in shared memory.
#include "common.cuh"

namespace sq {

constexpr int kGemvMaxM = 8;

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
  for (int m0 = 0; m0 < M; m0 += kGemvMaxM) {
    const int mc = M - m0 < kGemvMaxM ? M - m0 : kGemvMaxM;
    const int MT = mc <= 1 ? 1 : (mc <= 2 ? 2 : (mc <= 4 ? 4 : 8));
    const size_t smem = (size_t)MT * K * sizeof(float);
    SQ_REQUIRE(smem <= 200 * 1024, SQ_ERR_SHAPE, "sq_gemv_w4a16: K too large");
    int blocks = (N + 7) / 8;
    if (blocks > 148 * 4) blocks = 148 * 4;
#define SQ_GV(MTV)                                                                                  \
  {                                                                                                 \
    auto k = gemv_w4a16_kernel<MTV>;                                                                \
    if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k<<<blocks, 256, smem, st>>>(x + (int64_t)m0 * ldx, ldx, w4, s_group, group, mc, N, K,          \
                                 out + (int64_t)m0 * ldo, ldo, resid);                              \
  }
    if (MT == 1) SQ_GV(1) else if (MT == 2) SQ_GV(2) else if (MT == 4) SQ_GV(4) else SQ_GV(8)
#undef SQ_GV
  }
  return check_launch("sq_gemv_w4a16");
}
