// K3: W4A16 projection for small-batch decode: bandwidth-bound int4-weight x bf16-activation
// GEMV/GEMM (north_star (a); PAPER.md:302, 696 Marlin/hgemv lineage; "W4A16
// dequantizes weights into the float path").
//   y[m,n] = sum_g s_group[n,g] * sum_{k in g} w4[n,k] * bf16(x[m,k])      (f32 accumulation)
// The A16 activations are bf16: x arrives as f32 and is rounded to bf16 (RN) when staged; the
// int4 weights are exact in bf16, so every product is exact and only the f32 summation order
// differs from the oracle (oracle/qblock.py qlinear_a16 rounds x the same way).
//
// With norm_w the input rows are RMS-normalised on the way in (the block's gated norm before
// out_proj, the model's pre-norm before in_proj: one launch fewer each at b=1).
//
// Tensor-core path (K % 64 == 0, group 64 or 128): mma.sync m16n8k16 bf16 -> f32 with the weights
// as the 16-row A operand and up to 8 tokens as the N side.  sq_repack_w4a16 stores the nibbles in
// fragment order -- per (16-row block, 64-wide K quad) one 16-byte word per lane, one 32-bit word
// per k-step whose 4 nibble pairs are the lane's a0..a3 fragments -- so a warp's load is 512
// contiguous bytes and a fragment costs one LOP3 (nibble pair into the mantissa of 128 + u) and one
// bf16 subtract (u + 128 - 136 = v, exact).  Each warp of a CTA owns whole groups of one row block:
// per group a fresh f32 accumulator, then p += s_group * acc; the warps' partial rows are added in
// warp order (deterministic).  Other shapes: one warp per row over row-major u4packed weights.
#include <cuda_bf16.h>

#include "common.cuh"

namespace sq {

constexpr int GV_TOK = 8;   // tokens per pass (the MMA N side)

__device__ __forceinline__ uint32_t bf16_rn_pair(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// (a & 0x000F000F) | c in one LOP3 (c in a register: LOP3 takes a single immediate)
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(d) : "r"(a), "r"(c));   // (a & b) | c
  return d;
}

// 4 bf16x2 A fragments (v = u - 8) from one 32-bit word of 8 offset nibbles u = v + 8:
// the nibble pair goes into the mantissa of bf16 128 + u (one LOP3), then - 136 (exact)
__device__ __forceinline__ void w4_frag(uint32_t w, uint32_t magic, __nv_bfloat162 off, uint32_t (&a)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t t = lop3_and_or(w >> (4 * i), magic);
    const __nv_bfloat162 d = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&t), off);
    a[i] = *reinterpret_cast<const uint32_t*>(&d);
  }
}

// streamed weights: read once, so not allocated in L1
__device__ __forceinline__ uint4 ld_stream(const void* p) {
#ifdef SQ_GV_PROBE_LDG
  return __ldg(reinterpret_cast<const uint4*>(p));
#else
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
#endif
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// grid: one CTA per 32 weight rows (two 16-row MMA blocks per warp share every B fragment);
// NW warps split the K groups (group = 64 * QPG); DG groups of weights (DG * QPG * 2 512-B loads)
// in flight per warp.  smem: x as bf16 [M + 1][K + 8] (row M is zero: the B fragments of absent
// tokens; the pad keeps the B-fragment reads conflict-free) + the warps' partial tiles.
template <int NW, int QPG, int DG>
__global__ void __launch_bounds__(NW * 32) gemv_w4a16_mma_kernel(const float* x, int64_t ldx,
                                                                const float* __restrict__ norm_w, float eps,
                                                                const uint8_t* __restrict__ w,
                                                                const float* __restrict__ sgrp, int M, int N,
                                                                int K, float* out, int64_t ldo, int resid,
                                                                sq_conv_epilogue conv) {
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t gv_smem[];
  const int KP = K + 8;
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(gv_smem);
  float* part = reinterpret_cast<float*>(gv_smem + (size_t)(M + 1) * KP * 2);   // [NW][32][GV_TOK]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  constexpr int GROUP = 64 * QPG;
  const int G = K / GROUP, KQ = K / 64;
  const int g0 = warp * G / NW, g1 = (warp + 1) * G / NW;   // this warp's groups
  // row block r of this CTA: rows rbase + 16 r + {gid, gid + 8}
  const int rbase = blockIdx.x * 32;
  const uint8_t* wq0 = w + ((size_t)(2 * blockIdx.x) * KQ * 32 + lane) * 16;
  const uint8_t* wq1 = wq0 + (size_t)KQ * 512;
  const float* srow[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int n = rbase + 8 * i + gid;   // rows gid, gid + 8, 16 + gid, 24 + gid
    srow[i] = sgrp + (size_t)(n < N ? n : 0) * G;
  }
  // weight prefetch before the grid dependency wait (weights are static): [group][quad][block]
  uint4 buf[DG][QPG][2];
#pragma unroll
  for (int i = 0; i < DG; ++i)
#pragma unroll
    for (int qd = 0; qd < QPG; ++qd) {
      const bool ok = g0 + i < g1;
      const size_t off = (size_t)((g0 + i) * QPG + qd) * 512;
      buf[i][qd][0] = ok ? ld_stream(wq0 + off) : make_uint4(0, 0, 0, 0);
      buf[i][qd][1] = ok ? ld_stream(wq1 + off) : make_uint4(0, 0, 0, 0);
    }
  float sc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sc[i] = g0 < g1 ? __ldg(srow[i] + g0) : 0.f;
  pdl_wait();   // x / out come from earlier grids
  if (norm_w) {
    // fused RMSNorm of the input rows (rmsnorm_f32's math: f64 Σx², r = x·rfac·γ): pass 1 sums
    // the row, pass 2 re-reads it (L1 / L2) and stores bf16(r)
    __shared__ double red[NW];
    __shared__ float rfac_s;
    for (int m = 0; m < M; ++m) {
      const float* xr = x + (int64_t)m * ldx;
      double ss = 0.0;
#pragma unroll 4
      for (int k = threadIdx.x * 4; k < K; k += NW * 32 * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xr + k);
        ss += (double)v.x * (double)v.x + (double)v.y * (double)v.y + (double)v.z * (double)v.z +
              (double)v.w * (double)v.w;
      }
      ss = warp_sum_d(ss);
      if (lane == 0) red[warp] = ss;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < NW; ++i) t += red[i];
        const float ms = (float)(t / (double)K);
        rfac_s = __fdiv_rn(1.0f, sqrtf(__fadd_rn(ms, eps)));
      }
      __syncthreads();
      const float rf = rfac_s;
#pragma unroll 4
      for (int k = threadIdx.x * 4; k < K; k += NW * 32 * 4) {
        const float4 v = *reinterpret_cast<const float4*>(xr + k);
        const float4 g = __ldg(reinterpret_cast<const float4*>(norm_w + k));
        *reinterpret_cast<uint2*>(xs + (size_t)m * KP + k) =
            make_uint2(bf16_rn_pair(__fmul_rn(__fmul_rn(v.x, rf), g.x), __fmul_rn(__fmul_rn(v.y, rf), g.y)),
                       bf16_rn_pair(__fmul_rn(__fmul_rn(v.z, rf), g.z), __fmul_rn(__fmul_rn(v.w, rf), g.w)));
      }
      __syncthreads();   // red / rfac_s reused by the next row
    }
  } else {
  // activation staging (the loads are independent: the compiler keeps several in flight)
#ifndef SQ_GV_PROBE_NOSTAGE   // profiling builds only: x left unstaged
#pragma unroll 4
  for (int i = threadIdx.x * 4; i < M * K; i += NW * 32 * 4) {
    const int m = i / K, k = i - m * K;   // K % 4 == 0: a float4 never straddles rows
    const float4 v = *reinterpret_cast<const float4*>(x + (int64_t)m * ldx + k);
    *reinterpret_cast<uint2*>(xs + (size_t)m * KP + k) = make_uint2(bf16_rn_pair(v.x, v.y), bf16_rn_pair(v.z, v.w));
  }
#endif
  }
  for (int i = threadIdx.x * 2; i < K; i += NW * 32 * 2) *reinterpret_cast<uint32_t*>(xs + (size_t)M * KP + i) = 0u;
  __syncthreads();
  const uint32_t* xrow = reinterpret_cast<const uint32_t*>(xs + (size_t)(gid < M ? gid : M) * KP) + t4;
  const uint32_t magic = 0x43004300u;
  const __nv_bfloat162 off = __floats2bfloat162_rn(136.f, 136.f);
  float p[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
  // one group: QPG quads x 4 k-steps, two row blocks per B fragment; then the promotion
  auto group_step = [&](const uint4 (&cur)[QPG][2], int g) {
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    const uint32_t* xg = xrow + g * (GROUP / 2);
#pragma unroll
    for (int qd = 0; qd < QPG; ++qd) {
      const uint32_t w0[4] = {cur[qd][0].x, cur[qd][0].y, cur[qd][0].z, cur[qd][0].w};
      const uint32_t w1[4] = {cur[qd][1].x, cur[qd][1].y, cur[qd][1].z, cur[qd][1].w};
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint32_t b0 = xg[qd * 32 + s * 8], b1 = xg[qd * 32 + s * 8 + 4];
        uint32_t a[4];
        w4_frag(w0[s], magic, off, a);
        mma_bf16_16816(acc[0], a, b0, b1);
        w4_frag(w1[s], magic, off, a);
        mma_bf16_16816(acc[1], a, b0, b1);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      p[r][0] = fmaf(sc[2 * r], acc[r][0], p[r][0]);
      p[r][1] = fmaf(sc[2 * r], acc[r][1], p[r][1]);
      p[r][2] = fmaf(sc[2 * r + 1], acc[r][2], p[r][2]);
      p[r][3] = fmaf(sc[2 * r + 1], acc[r][3], p[r][3]);
    }
    if (g + 1 < g1) {   // next group's scales
#pragma unroll
      for (int i = 0; i < 4; ++i) sc[i] = __ldg(srow[i] + g + 1);
    }
  };
  int g = g0;
  for (; g + DG <= g1; g += DG) {   // full rounds: each slot is refilled right after its group
#pragma unroll
    for (int i = 0; i < DG; ++i) {
      group_step(buf[i], g + i);
      const int gn = g + DG + i;
      if (gn < g1) {
#pragma unroll
        for (int qd = 0; qd < QPG; ++qd) {
          const size_t off2 = (size_t)(gn * QPG + qd) * 512;
          buf[i][qd][0] = ld_stream(wq0 + off2);
          buf[i][qd][1] = ld_stream(wq1 + off2);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < DG; ++i)   // remainder (< DG groups, already loaded)
    if (g + i < g1) group_step(buf[i], g + i);
  // partial tile of this warp: rows 16 r + gid / + 8, tokens 2 t4, 2 t4 + 1
  float* pw = part + warp * 32 * GV_TOK;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    pw[(16 * r + gid) * GV_TOK + 2 * t4] = p[r][0];
    pw[(16 * r + gid) * GV_TOK + 2 * t4 + 1] = p[r][1];
    pw[(16 * r + gid + 8) * GV_TOK + 2 * t4] = p[r][2];
    pw[(16 * r + gid + 8) * GV_TOK + 2 * t4 + 1] = p[r][3];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * GV_TOK; i += NW * 32) {
    const int rr = i / GV_TOK, m = i % GV_TOK, n = rbase + rr;
    if (m < M && n < N) {
      float v = part[i];
#pragma unroll
      for (int ww = 1; ww < NW; ++ww) v = __fadd_rn(v, part[ww * 32 * GV_TOK + i]);
      float* o = out + (int64_t)m * ldo + n;
      v = resid ? __fadd_rn(*o, v) : v;
      *o = v;
      const int c = n - conv.c0;
      if (c >= 0 && c < conv.C) {   // fused conv update of channel c (sq_conv1d_f32's T = 1 math)
        const int kc = conv.kc;
        float* cr = conv.cache + (int64_t)m * (kc - 1) * conv.C + c;
        float win[8], wc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          wc[j] = j < kc ? __ldg(conv.w + c * kc + j) : 0.f;
          win[j] = (j < kc - 1 && conv.cache_in) ? cr[(int64_t)j * conv.C] : 0.f;
        }
        float acc = __ldg(conv.b + c);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < kc) acc = __fadd_rn(acc, __fmul_rn(wc[j], j == kc - 1 ? v : win[j]));
        conv.out[(int64_t)m * conv.ldo + c] = silu_f(acc);
#pragma unroll
        for (int j = 0; j + 1 < 8; ++j)
          if (j + 1 < kc) cr[(int64_t)j * conv.C] = j + 1 == kc - 1 ? v : win[j + 1];
      }
    }
  }
}

// Fallback (other K / group): one warp per output row, row-major u4packed
// weights (low nibble = even k), bf16-rounded activations in smem.
__global__ void __launch_bounds__(256) gemv_w4a16_rows_kernel(const float* x, int64_t ldx,
                                                              const float* __restrict__ norm_w, float eps,
                                                              const uint8_t* __restrict__ w,
                                                              const float* __restrict__ sgrp, int group, int M,
                                                              int N, int K, float* out, int64_t ldo, int resid) {
  extern __shared__ float xr[];  // [M][K] bf16-rounded, kept in f32
  __shared__ double red[8];
  __shared__ float rfs[GV_TOK];
  if (norm_w) {   // fused RMSNorm (rmsnorm_f32's math) of each input row
    for (int m = 0; m < M; ++m) {
      double ss = 0.0;
      for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const float v = x[(int64_t)m * ldx + k];
        ss += (double)v * (double)v;
      }
      ss = warp_sum_d(ss);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        rfs[m] = __fdiv_rn(1.0f, sqrtf(__fadd_rn((float)(t / (double)K), eps)));
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    float v = x[(int64_t)m * ldx + k];
    if (norm_w) v = __fmul_rn(__fmul_rn(v, rfs[m]), __ldg(norm_w + k));
    xr[i] = __bfloat162float(__float2bfloat16_rn(v));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  const int G = K / group;
  for (int n = blockIdx.x * warps + (threadIdx.x >> 5); n < N; n += gridDim.x * warps) {
    const uint8_t* wr = w + (int64_t)n * (K / 2);
    for (int m = 0; m < M; ++m) {
      float tot = 0.f;
      for (int g = 0; g < G; ++g) {
        float part = 0.f;
        for (int k = g * group + lane; k < (g + 1) * group; k += 32) {
          const int byte = wr[k >> 1];
          const int v = ((k & 1) ? (byte >> 4) : (byte & 0xF)) ^ 8;   // offset nibble -> v + 8
          part = fmaf((float)(v - 8), xr[m * K + k], part);
        }
        tot = fmaf(warp_sum(part), __ldg(sgrp + (int64_t)n * G + g), tot);
      }
      if (lane == 0) {
        float* o = out + (int64_t)m * ldo + n;
        *o = resid ? __fadd_rn(*o, tot) : tot;
      }
    }
  }
}

// SPEC u4packed [N x K/2] (low nibble = even k, two's-complement nibbles) -> the fragment layout:
// [row block][k quad][lane][k-step 0..3] 32-bit words of offset nibbles u = v + 8 (rows >= N zero).
__global__ void repack_w4a16_kernel(const uint8_t* __restrict__ src, int N, int K, uint32_t* __restrict__ dst) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one 32-bit word
  const int KQ = K / 64;
  const int64_t words = (int64_t)((N + 31) / 32) * 2 * KQ * 32 * 4;   // row blocks padded to pairs
  if (idx >= words) return;
  const int s = idx & 3, lane = (idx >> 2) & 31;
  const int64_t qb = idx >> 7;
  const int q = (int)(qb % KQ), rb = (int)(qb / KQ);
  const int gid = lane >> 2, t4 = lane & 3;
  const int k0 = q * 64 + s * 16 + 2 * t4;
  auto nib = [&](int n, int k) -> uint32_t {
    if (n >= N) return 8u;   // v = 0
    const int byte = src[(int64_t)n * (K / 2) + (k >> 1)];
    return (uint32_t)(((k & 1) ? (byte >> 4) : byte) & 0xF) ^ 8u;
  };
  const int r0 = rb * 16 + gid, r1 = r0 + 8;
  uint32_t v = 0;
  // pair i -> bits 4i..4i+3 (first k) and 16+4i..16+4i+3 (second k): a0 (r0, k0), a1 (r1, k0),
  // a2 (r0, k0 + 8), a3 (r1, k0 + 8)
  const int rows[4] = {r0, r1, r0, r1}, ks[4] = {k0, k0, k0 + 8, k0 + 8};
#pragma unroll
  for (int i = 0; i < 4; ++i) v |= (nib(rows[i], ks[i]) << (4 * i)) | (nib(rows[i], ks[i] + 1) << (16 + 4 * i));
  dst[idx] = v;
}

static bool w4a16_mma_layout(int K, int group) { return K % 64 == 0 && (group == 64 || group == 128); }

}  // namespace sq

using namespace sq;

extern "C" int64_t sq_w4a16_bytes(int N, int K, int group) {
  if (N <= 0 || K <= 0 || group <= 0) return -1;
  if (w4a16_mma_layout(K, group)) return (int64_t)((N + 31) / 32) * 32 * K / 2;
  return (int64_t)N * K / 2;
}

extern "C" int sq_repack_w4a16(const uint8_t* u4packed, int N, int K, int group, uint8_t* dst, void* stream) {
  SQ_REQUIRE(u4packed && dst && N > 0 && K > 0 && K % 2 == 0 && group > 0 && K % group == 0, SQ_ERR_SHAPE,
             "sq_repack_w4a16: bad shape N=%d K=%d group=%d", N, K, group);
  cudaStream_t st = as_stream(stream);
  if (!w4a16_mma_layout(K, group)) {
    cudaError_t e = cudaMemcpyAsync(dst, u4packed, (size_t)N * K / 2, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SQ_OK : SQ_ERR_CUDA;
  }
  const int64_t words = (int64_t)((N + 31) / 32) * 2 * (K / 64) * 128;
  repack_w4a16_kernel<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(u4packed, N, K, reinterpret_cast<uint32_t*>(dst));
  return check_launch("sq_repack_w4a16");
}

extern "C" int sq_gemv_w4a16_conv(const float* x, int64_t ldx, const float* norm_w, float eps, const uint8_t* w4,
                                  const float* s_group, int group, int M, int N, int K, float* out, int64_t ldo,
                                  int resid, const sq_conv_epilogue* conv_in, void* stream) {
  sq_conv_epilogue conv{};
  if (conv_in) {
    conv = *conv_in;
    SQ_REQUIRE(conv.w && conv.b && conv.cache && conv.out && conv.kc >= 1 && conv.kc <= 8 && conv.c0 >= 0 &&
                   conv.C > 0 && conv.c0 + conv.C <= N,
               SQ_ERR_SHAPE, "sq_gemv_w4a16_conv: bad conv epilogue (kc %d, columns %d + %d of %d)", conv.kc,
               conv.c0, conv.C, N);
  }
  SQ_REQUIRE(x && w4 && s_group && out && M >= 0 && N > 0 && K > 0 && group > 0 && K % group == 0 && K % 2 == 0,
             SQ_ERR_SHAPE, "sq_gemv_w4a16: bad shape M=%d N=%d K=%d group=%d", M, N, K, group);
  cudaStream_t st = as_stream(stream);
  if (M == 0) return SQ_OK;
  if (w4a16_mma_layout(K, group)) {
    SQ_REQUIRE(ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, SQ_ERR_LAYOUT,
               "sq_gemv_w4a16: x must be 16-B aligned with ldx %% 4 == 0");
    const int cta = (N + 31) / 32;
    for (int m0 = 0; m0 < M; m0 += GV_TOK) {
      const int mc = M - m0 < GV_TOK ? M - m0 : GV_TOK;
      // few CTAs (small N): more warps per CTA, each with its own slice of the groups, so every
      // SM keeps ~16 warps x 4-6 KB of weights in flight
      const int G = K / group;
#ifdef SQ_GV_PROBE_NW   // profiling builds only: fixed warps per CTA
      const int nw = SQ_GV_PROBE_NW;
#else
      const int nw = (cta < 148 && G >= 16) ? 16 : (cta < 3 * 148 && G >= 8) ? 8 : 4;
#endif
      const size_t smem = (size_t)(mc + 1) * (K + 8) * 2 + (size_t)nw * 32 * GV_TOK * 4;
      SQ_REQUIRE(smem <= 227 * 1024, SQ_ERR_SHAPE, "sq_gemv_w4a16: K too large");
      auto launch = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sq_conv_epilogue cv = conv;   // this pass's tokens m0 .. m0 + mc - 1
        if (cv.C > 0) {
          cv.cache += (int64_t)m0 * (cv.kc - 1) * cv.C;
          cv.out += (int64_t)m0 * cv.ldo;
        }
        launch_k(PDL_SMALL, kern, dim3(cta), dim3(nw * 32), smem, st, x + (int64_t)m0 * ldx, ldx, norm_w, eps, w4,
                 s_group, mc, N, K, out + (int64_t)m0 * ldo, ldo, resid, cv);
      };
#ifndef SQ_GV_DG
#define SQ_GV_DG 3
#endif
      if (group == 128) {
        if (nw == 16) launch(gemv_w4a16_mma_kernel<16, 2, SQ_GV_DG>);
        else if (nw == 8) launch(gemv_w4a16_mma_kernel<8, 2, SQ_GV_DG>);
        else launch(gemv_w4a16_mma_kernel<4, 2, SQ_GV_DG>);
      } else {
        if (nw == 16) launch(gemv_w4a16_mma_kernel<16, 1, 6>);
        else if (nw == 8) launch(gemv_w4a16_mma_kernel<8, 1, 6>);
        else launch(gemv_w4a16_mma_kernel<4, 1, 6>);
      }
    }
    return check_launch("sq_gemv_w4a16");
  }
  for (int m0 = 0; m0 < M; m0 += GV_TOK) {
    const int mc = M - m0 < GV_TOK ? M - m0 : GV_TOK;
    const size_t smem = (size_t)mc * K * 4;
    SQ_REQUIRE(smem <= 200 * 1024, SQ_ERR_SHAPE, "sq_gemv_w4a16: K too large");
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(gemv_w4a16_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int blocks = (N + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    gemv_w4a16_rows_kernel<<<blocks, 256, smem, st>>>(x + (int64_t)m0 * ldx, ldx, norm_w, eps, w4, s_group, group,
                                                      mc, N, K, out + (int64_t)m0 * ldo, ldo, resid);
  }
  if (conv.C > 0) {   // the row-major fallback has no fused epilogue: the separate conv update
    const int rc = check_launch("sq_gemv_w4a16");
    if (rc != SQ_OK) return rc;
    return sq_conv1d_f32(out + conv.c0, ldo, conv.w, conv.b, M, 1, conv.C, conv.kc, conv.cache, conv.cache_in,
                         conv.out, conv.ldo, stream);
  }
  return check_launch("sq_gemv_w4a16");
}

extern "C" int sq_gemv_w4a16(const float* x, int64_t ldx, const float* norm_w, float eps, const uint8_t* w4,
                             const float* s_group, int group, int M, int N, int K, float* out, int64_t ldo, int resid,
                             void* stream) {
  return sq_gemv_w4a16_conv(x, ldx, norm_w, eps, w4, s_group, group, M, N, K, out, ldo, resid, nullptr, stream);
}
