// K7 on the 5th-gen tensor cores: int8 SSD chunk scan for Mamba2 prefill with tcgen05.mma
// (ssm_block.ssd_chunked; "8-bit SSD").
//
// One CTA (8 warps: a TMEM lane row per thread pair, column halves split between the pair)
// per (sequence, head), chunks of Q = 128 tokens.
// Every product runs as a 128-row tcgen05.mma with its operands in SW128 K-major shared
// memory tiles and its accumulator in TMEM:
//
//   CB[t,s]    = Ĉ_t · B̂_s                 kind::i8  128x128x128  int32 (exact), TMEM [0,128)
//   Y_off[t,p] = Ĉ_t · H_p                 kind::f16 128x64x128   f32 (H as fp16),  [128,192)
//   W[t,s]     = CB s_B s_C e^{cs_t-cs_s} Δ_s (s <= t)           -> fp16 tile (threads)
//   Y_diag     = W · X̂                     kind::f16 128x64x128   f32 (x codes exact), [192,256)
//   ΔHᵀ[n,p]   = Σ_s B̂_s[n] (w_s s_x[p] s_B x_s[p])   kind::f16 128x64x128 twice (the fp16
//                hi and lo halves of the weights, so the update keeps ~f32 precision), [320,384)
//   Hᵀ         = e^{cs_Q} Hᵀ + ΔHᵀ         threads, TMEM [256,320) (f32 state, never leaves TMEM)
//   y          = (Y_diag s_x + Y_off e^{cs_t} s_C + D x̂) · SiLU(ẑ)  -> staged, coalesced stores
//
// The int8 codes of B and C arrive by cp.async directly in the swizzled operand layout;
// x / z codes are double-buffered; the next chunk's loads overlap the current chunk's
// element-wise phases.  One thread issues the MMAs; tcgen05.commit -> mbarrier hands the
// accumulators back to the four warps.
#include <cuda_fp16.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace sq {
using namespace sm100;

constexpr int TQ = 128;   // chunk length
constexpr int TP = 64;    // head_dim
constexpr int TN = 128;   // d_state
constexpr int TC_SSD_THREADS = 256;   // 8 warps: TMEM lane quadrant (warp & 3) x column half (warp >> 2)

// byte offset of element (row r, byte b) in a SW128 K-major tile of 128-byte rows
__device__ __forceinline__ int sw128(int r, int b) { return r * 128 + ((((b >> 4) ^ (r & 7))) << 4) + (b & 15); }

__host__ __device__ constexpr uint32_t idesc_f16f32(int M, int N) {   // fp16 x fp16 -> f32, K-major
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// MN-major SW128 operand: 128-byte rows along M/N (64 fp16), 8-row (along K) swizzle atoms
// 1024 B apart (SBO); `lbo` bytes between 64-wide M/N blocks.  A K-step of 16 advances 2048 B.
__device__ __forceinline__ uint64_t desc_mn(const void* tile, uint32_t lbo) {
  const uint64_t addr = smem_u32(tile);
  return ((addr >> 4) & 0x3FFFull) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ void cpa16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
// four int8 codes -> two fp16x2 (exact): biased bytes under the fp16 exponent of 1024, minus 1152
__device__ __forceinline__ void s8x4_h2x2_t(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t u = w ^ 0x80808080u;
  uint32_t a = __byte_perm(u, 0x64646464u, 0x4140), b = __byte_perm(u, 0x64646464u, 0x4342);
  const __half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
  const __half2 ha = __hsub2(*reinterpret_cast<__half2*>(&a), bias);
  const __half2 hb = __hsub2(*reinterpret_cast<__half2*>(&b), bias);
  lo = *reinterpret_cast<const uint32_t*>(&ha);
  hi = *reinterpret_cast<const uint32_t*>(&hb);
}
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 v = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// shared memory map (bytes; SW128 tiles 1024-aligned)
struct TcSsdSmem {
  static constexpr int RAWC = 0;                 // C codes [t][n] int8 SW128, buffer k at +k*32 KB
  static constexpr int RAWB = RAWC + 16384;      // B codes [s][n] int8 SW128, buffer k at +k*32 KB
  static constexpr int XR = 80;                  // x code row pitch (64 B + 16: conflict-free row reads)
  static constexpr int RAWX = RAWC + 65536;      // x codes [s][p] int8, 2 buffers 2 x 10 KB
  static constexpr int RAWZ = RAWX + 2 * 128 * XR;   // z codes [t][p] int8, 2 buffers 2 x 8 KB
  static constexpr int CF = RAWZ + 16384;        // C fp16 [t][n] (2 K-blocks), later W [t][s]   32 KB
  static constexpr int BTF = CF + 32768;         // B fp16 [s][n] MN-major (2 n-blocks), later y staging 32 KB
  static constexpr int XTF = BTF + 32768;        // x fp16 [s][p] MN-major                        16 KB
  static constexpr int HF = XTF + 16384;         // H fp16 [n][p] MN-major, later Aw hi [p][s]    16 KB
  static constexpr int AWL = HF + 16384;         // Aw lo fp16 [p][s] (2 K-blocks)                16 KB
  static constexpr int SMALL = AWL + 16384;      // cs, dlt, wgt, et [128] f32; lut [256]; sx [64]
  static constexpr int BAR = SMALL + 4 * 512 + 1024 + 256 + 1024;   // + cs·log2e, s_B s_C Δ [128] each
  static constexpr int BYTES = BAR + 64;
  static constexpr int ALLOC = BYTES + 1024;     // + alignment slack
};

template <int N>
__global__ void __launch_bounds__(TC_SSD_THREADS, 1)
    ssd_chunk_tc_kernel(sq_mamba2_params p, int T, const int8_t* x, int64_t ldx, const int8_t* Bm, const int8_t* Cm,
                        int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                        int8_t* __restrict__ state, int state_in, float* __restrict__ y, int64_t ldy) {
  using L = TcSsdSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(sm);
  float* s_cs = reinterpret_cast<float*>(sm + L::SMALL);
  float* s_dlt = s_cs + TQ;
  float* s_wgt = s_dlt + TQ;
  float* s_et = s_wgt + TQ;
  float* s_lut = s_et + TQ;            // 256
  float* s_sx = s_lut + 256;           // 64
  float* s_cs2 = s_sx + 64;            // cs · log2(e)  [128]
  float* s_db = s_cs2 + TQ;            // s_B s_C Δ     [128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::BAR);   // [0] MMA group 1, [1] MMA group 2
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bar + 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.x, b = blockIdx.y;
  const int grp = p.head_group[h];
  const float A = p.A[h], Dh = p.D[h], dtb = p.dt_bias[h];
  const float sB = p.s_B[grp], sC = p.s_C[grp];
  const float sBC = __fmul_rn(sB, sC);
  const int ch0 = h * TP;
  const int64_t tok0 = (int64_t)b * T;
  const int q4 = warp & 3, hw = warp >> 2;
  const int row = q4 * 32 + lane;                            // TMEM lane (t, n) of this thread
  const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;      // this warp's TMEM lane quadrant

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_holder);
  for (int i = tid; i < 256; i += TC_SSD_THREADS) s_lut[i] = silu_fast(__fmul_rn((float)(i - 128), p.s_z));
  if (tid < TP) s_sx[tid] = p.s_x[ch0 + tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t T_CB = tmem, T_YO = tmem + 128, T_YD = tmem + 192, T_H = tmem + 256, T_DH = tmem + 320;

  // async fetch of one chunk (rows past T zero-filled): B / C straight into their swizzled
  // operand tiles, x / z codes into buffer `buf`
  auto fetch = [&](int c0, int buf) {
    const int Qc = min(TQ, T - c0);
    for (int i = tid; i < TQ * (N / 16); i += TC_SSD_THREADS) {
      const int r = i / (N / 16), c16 = i % (N / 16);
      const int64_t tok = tok0 + c0 + min(r, Qc - 1);
      cpa16(sbase + L::RAWB + buf * 32768 + sw128(r, c16 * 16), Bm + tok * ldbc + grp * N + c16 * 16, r < Qc);
      cpa16(sbase + L::RAWC + buf * 32768 + sw128(r, c16 * 16), Cm + tok * ldbc + grp * N + c16 * 16, r < Qc);
    }
    for (int i = tid; i < TQ * (TP / 16); i += TC_SSD_THREADS) {
      const int r = i / (TP / 16), c16 = (i % (TP / 16)) * 16;
      const int64_t tok = tok0 + c0 + min(r, Qc - 1);
      cpa16(sbase + L::RAWX + buf * 128 * L::XR + r * L::XR + c16, x + tok * ldx + ch0 + c16, r < Qc);
      cpa16(sbase + L::RAWZ + buf * 8192 + r * TP + c16, z + tok * ldz + ch0 + c16, r < Qc);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  fetch(0, 0);

  // initial state: thread n (lane) holds Hᵀ[n][0..63] = code · s_h[p]
  {
    const int n = row;
    int8_t* st = state + ((int64_t)b * p.n_heads + h) * TP * N;
#pragma unroll
    for (int c = hw * 32; c < hw * 32 + 32; c += 16) {
      uint32_t v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        v[j] = __float_as_uint(state_in ? __fmul_rn((float)st[(c + j) * N + n], p.s_h[ch0 + c + j]) : 0.f);
      tmem_st_x16(T_H + lane_off + c, v);
    }
    tmem_wait_st();
  }
  int8_t dcode = tid < TQ ? dt[(tok0 + min(tid, T - 1)) * lddt + h] : 0;   // prefetched one chunk ahead
  const uint64_t dCF = desc_sw128(sm + L::CF), dHF = desc_sw128(sm + L::HF), dAL = desc_sw128(sm + L::AWL);
  const uint64_t dBN = desc_mn(sm + L::BTF, TQ * 128), dXN = desc_mn(sm + L::XTF, TQ * 128);
  const uint64_t dHN = desc_mn(sm + L::HF, N * 128);
  const uint64_t dRC = desc_sw128(sm + L::RAWC), dRB = desc_sw128(sm + L::RAWB);
  constexpr uint32_t ID_I8 = idesc_i8(128, 128);
  constexpr uint32_t ID_BMN = idesc_f16f32(128, 64) | (1u << 16);   // A K-major, B MN-major
  constexpr uint32_t ID_AMN = idesc_f16f32(128, 64) | (1u << 15);   // A MN-major, B K-major
  // descriptor of K-step ks (16 fp16 = 32 B) of a two-block fp16 tile with `rows` rows
  auto kdesc = [](uint64_t d0, int rows, int ks) { return d0 + (uint64_t)((ks >> 2) * rows * 128 >> 4) + 2 * (ks & 3); };

  int buf = 0, ph = 0;
  for (int c0 = 0; c0 < T; c0 += TQ, buf ^= 1, ph ^= 1) {
    const int Qc = min(TQ, T - c0);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();   // this chunk's codes landed; the previous chunk is fully consumed
    if (c0 + TQ < T) fetch(c0 + TQ, buf ^ 1);   // a whole chunk of compute hides the next loads
    const int rbc = buf * 32768;
    const int8_t* rx = reinterpret_cast<const int8_t*>(sm + L::RAWX + buf * 128 * L::XR);
    const int8_t* rz = reinterpret_cast<const int8_t*>(sm + L::RAWZ + buf * 8192);
    // ---- P1: Δ, fp16 operand tiles, H (fp16) for Y_off
    if (tid < TQ) {
      float dl = 0.f, dA = 0.f;
      if (tid < Qc) {
        dl = softplus_f(__fadd_rn(__fmul_rn((float)dcode, p.s_dt), dtb));
        dA = __fmul_rn(dl, A);
      }
      s_dlt[tid] = dl;
      s_cs[tid] = dA;
      dcode = dt[(tok0 + min(c0 + TQ + tid, T - 1)) * lddt + h];
    }
    {   // C fp16 row t (K = n: two 64-wide blocks), this thread's column half
      const int t = row;
#pragma unroll
      for (int c16 = hw * (N / 32); c16 < (hw + 1) * (N / 32); ++c16) {
        const uint4 w = *reinterpret_cast<const uint4*>(sm + L::RAWC + rbc + sw128(t, c16 * 16));
        uint4 o0, o1;
        s8x4_h2x2_t(w.x, o0.x, o0.y); s8x4_h2x2_t(w.y, o0.z, o0.w);
        s8x4_h2x2_t(w.z, o1.x, o1.y); s8x4_h2x2_t(w.w, o1.z, o1.w);
        const int blk = c16 >> 2, b0 = (c16 & 3) * 32;   // 16 codes -> 32 B of fp16
        *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0)) = o0;
        *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0 + 16)) = o1;
      }
    }
    {   // B fp16 [s][n] (MN-major: n-blocks of 64), row s = row, this thread's n half
      const int sr = row;
#pragma unroll
      for (int c16 = hw * (N / 32); c16 < (hw + 1) * (N / 32); ++c16) {
        const uint4 w = *reinterpret_cast<const uint4*>(sm + L::RAWB + rbc + sw128(sr, c16 * 16));
        uint4 o0, o1;
        s8x4_h2x2_t(w.x, o0.x, o0.y); s8x4_h2x2_t(w.y, o0.z, o0.w);
        s8x4_h2x2_t(w.z, o1.x, o1.y); s8x4_h2x2_t(w.w, o1.z, o1.w);
        const int blk = c16 >> 2, b0 = (c16 & 3) * 32;
        *reinterpret_cast<uint4*>(sm + L::BTF + blk * TQ * 128 + sw128(sr, b0)) = o0;
        *reinterpret_cast<uint4*>(sm + L::BTF + blk * TQ * 128 + sw128(sr, b0 + 16)) = o1;
      }
    }
    {   // x fp16 [s][p] (MN-major): row s = row, this thread's 32 codes
      const int sr = row;
      const uint4 w0 = *reinterpret_cast<const uint4*>(rx + sr * L::XR + hw * 32);
      const uint4 w1 = *reinterpret_cast<const uint4*>(rx + sr * L::XR + hw * 32 + 16);
      uint4 o0, o1, o2, o3;
      s8x4_h2x2_t(w0.x, o0.x, o0.y); s8x4_h2x2_t(w0.y, o0.z, o0.w);
      s8x4_h2x2_t(w0.z, o1.x, o1.y); s8x4_h2x2_t(w0.w, o1.z, o1.w);
      s8x4_h2x2_t(w1.x, o2.x, o2.y); s8x4_h2x2_t(w1.y, o2.z, o2.w);
      s8x4_h2x2_t(w1.z, o3.x, o3.y); s8x4_h2x2_t(w1.w, o3.z, o3.w);
      const int b0 = hw * 64;
      *reinterpret_cast<uint4*>(sm + L::XTF + sw128(sr, b0)) = o0;
      *reinterpret_cast<uint4*>(sm + L::XTF + sw128(sr, b0 + 16)) = o1;
      *reinterpret_cast<uint4*>(sm + L::XTF + sw128(sr, b0 + 32)) = o2;
      *reinterpret_cast<uint4*>(sm + L::XTF + sw128(sr, b0 + 48)) = o3;
    }
    {   // H fp16 [n][p] (MN-major): thread n writes its own row, its p half
      const int n = row;
#pragma unroll
      for (int c = hw * 32; c < hw * 32 + 32; c += 16) {
        uint32_t v[16];
        tmem_ld_x16(T_H + lane_off + c, v);
        tmem_wait_ld();
        uint32_t hv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) hv[j] = pack_h2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        *reinterpret_cast<uint4*>(sm + L::HF + sw128(n, c * 2)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        *reinterpret_cast<uint4*>(sm + L::HF + sw128(n, c * 2 + 16)) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    // ---- P2: CB and Y_off on the tensor cores; warp 1 scans Δ·A meanwhile
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < N / 32; ++ks)
        mma_i8_ss(T_CB, dRC + (rbc >> 4) + 2 * ks, dRB + (rbc >> 4) + 2 * ks, ID_I8, ks > 0);
#pragma unroll
      for (int ks = 0; ks < N / 16; ++ks) mma_f16_ss(T_YO, kdesc(dCF, TQ, ks), dHN + 128 * ks, ID_BMN, ks > 0);
      mma_commit(&bar[0]);
    }
    if (warp == 1) {   // inclusive prefix of Δ·A over 128 tokens (4 per lane, in order)
      float v0 = s_cs[4 * lane], v1 = s_cs[4 * lane + 1], v2 = s_cs[4 * lane + 2], v3 = s_cs[4 * lane + 3];
      v1 += v0; v2 += v1; v3 += v2;
      float run = v3;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float a = __shfl_up_sync(0xffffffffu, run, o);
        if (lane >= o) run += a;
      }
      const float off = run - v3;
      v0 += off; v1 += off; v2 += off; v3 += off;
      const float csQ = __shfl_sync(0xffffffffu, v3, 31);
      const float vv[4] = {v0, v1, v2, v3};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int t = 4 * lane + j;
        s_cs[t] = vv[j];
        s_cs2[t] = __fmul_rn(vv[j], 1.4426950408889634f);
        s_db[t] = __fmul_rn(sBC, s_dlt[t]);
        s_wgt[t] = __fmul_rn(expf(__fsub_rn(csQ, vv[j])), s_dlt[t]);
        s_et[t] = __fmul_rn(__expf(vv[j]), sC);
      }
    }
    __syncthreads();   // cs / wgt / et visible
    mbar_wait(&bar[0], ph);
    tc_fence_after();
    // ---- P3: W (from CB) and the state-update weights Aw (hi / lo)
    {
      const int t = row;
      const float2 cst2 = make_float2(s_cs2[t], s_cs2[t]);
      const float2 M1 = make_float2(-1.f, -1.f);
#pragma unroll 1
      for (int c = hw * 64; c < hw * 64 + 64; c += 16) {
        uint32_t o[8];
        const int blk = c >> 6, b0 = (c & 63) * 2;
        if (c > 32 * q4 + 31) {   // s > t for every row of this warp: causally zero
          *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0)) = make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0 + 16)) = make_uint4(0, 0, 0, 0);
          continue;
        }
        uint32_t v[16];
        tmem_ld_x16(T_CB + lane_off + c, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; j += 2) {   // W pair (s, s+1) = CB · 2^{(cs_t - cs_s) log2 e} · s_B s_C Δ_s, packed f32x2
          const int s = c + j;
          const float2 d = __ffma2_rn(*reinterpret_cast<const float2*>(&s_cs2[s]), M1, cst2);
          const float2 e2 = make_float2(ex2_approx(d.x), ex2_approx(d.y));
          const float2 w2 = __fmul2_rn(__fmul2_rn(make_float2((float)(int)v[j], (float)(int)v[j + 1]), e2),
                                       *reinterpret_cast<const float2*>(&s_db[s]));
          o[j >> 1] = pack_h2(s <= t ? w2.x : 0.f, s + 1 <= t ? w2.y : 0.f);
        }
        *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(sm + L::CF + blk * TQ * 128 + sw128(t, b0 + 16)) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
    {   // Aw[p][s] = w_s x_s[p] s_x[p] s_B, split fp16 hi + lo: thread (p, s quarter)
      const int pp = tid & 63, sh = (tid >> 6) * 32;
      const float fr = __fmul_rn(s_sx[pp], sB);
#pragma unroll 2
      for (int s8 = sh; s8 < sh + 32; s8 += 8) {
        uint32_t hi[4], lo[4];
        const float2 fr2 = make_float2(fr, fr);
#pragma unroll
        for (int j = 0; j < 8; j += 2) {   // packed pairs (s, s+1)
          const float2 xv = make_float2((float)rx[(s8 + j) * L::XR + pp], (float)rx[(s8 + j + 1) * L::XR + pp]);
          const float2 v2 = __fmul2_rn(__fmul2_rn(*reinterpret_cast<const float2*>(&s_wgt[s8 + j]), xv), fr2);
          const __half2 hh = __floats2half2_rn(v2.x, v2.y);
          const float2 hf = __half22float2(hh);
          hi[j >> 1] = *reinterpret_cast<const uint32_t*>(&hh);
          const float2 rem = __ffma2_rn(hf, make_float2(-1.f, -1.f), v2);
          lo[j >> 1] = pack_h2(rem.x, rem.y);
        }
        const int off = (s8 >> 6) * TP * 128 + sw128(pp, (s8 & 63) * 2);
        *reinterpret_cast<uint4*>(sm + L::HF + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);   // HF reused as Aw hi
        *reinterpret_cast<uint4*>(sm + L::AWL + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    // ---- P4: Y_diag and ΔHᵀ on the tensor cores
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < TQ / 16; ++ks) mma_f16_ss(T_YD, kdesc(dCF, TQ, ks), dXN + 128 * ks, ID_BMN, ks > 0);
#pragma unroll
      for (int ks = 0; ks < TQ / 16; ++ks) mma_f16_ss(T_DH, dBN + 128 * ks, kdesc(dHF, TP, ks), ID_AMN, ks > 0);
#pragma unroll
      for (int ks = 0; ks < TQ / 16; ++ks) mma_f16_ss(T_DH, dBN + 128 * ks, kdesc(dAL, TP, ks), ID_AMN, 1);
      mma_commit(&bar[1]);
    }
    mbar_wait(&bar[1], ph);
    tc_fence_after();
    // ---- P5: outputs (staged over the Bᵀ tile) and the state update in TMEM
    float* ys = reinterpret_cast<float*>(sm + L::BTF);   // [128][64 + 4]
    {
      const int t = row;
      const float et = s_et[t];
#pragma unroll 1
      for (int c = hw * 32; c < hw * 32 + 32; c += 16) {
        uint32_t vd[16], vo[16];
        tmem_ld_x16(T_YD + lane_off + c, vd);
        tmem_ld_x16(T_YO + lane_off + c, vo);
        const uint4 xq = *reinterpret_cast<const uint4*>(rx + t * L::XR + c);   // this row's 16 x codes
        const int8_t* xb = reinterpret_cast<const int8_t*>(&xq);
        tmem_wait_ld();
        float yv[16];
        const float2 et2 = make_float2(et, et), Dh2 = make_float2(Dh, Dh);
#pragma unroll
        for (int j = 0; j < 16; j += 2) {   // (Y_diag s_x + Y_off e_t) + D x̂, packed over p pairs
          const float2 sx2 = *reinterpret_cast<const float2*>(&s_sx[c + j]);
          const float2 xh = __fmul2_rn(make_float2((float)xb[j], (float)xb[j + 1]), sx2);
          const float2 a = __fmul2_rn(make_float2(__uint_as_float(vd[j]), __uint_as_float(vd[j + 1])), sx2);
          const float2 bo = __fmul2_rn(make_float2(__uint_as_float(vo[j]), __uint_as_float(vo[j + 1])), et2);
          const float2 r2 = __fadd2_rn(__fadd2_rn(a, bo), __fmul2_rn(Dh2, xh));
          yv[j] = r2.x;
          yv[j + 1] = r2.y;
        }
#pragma unroll
        for (int j = 0; j < 16; j += 4)   // 16-B stores: a quarter-warp covers all 32 banks (row pitch 68 floats)
          *reinterpret_cast<float4*>(&ys[t * (TP + 4) + c + j]) = make_float4(yv[j], yv[j + 1], yv[j + 2], yv[j + 3]);
      }
    }
    {
      const float eQ = expf(s_cs[TQ - 1]);   // padded tokens carry Δ = 0
#pragma unroll
      for (int c = hw * 32; c < hw * 32 + 32; c += 16) {
        uint32_t vh[16], vd[16];
        tmem_ld_x16(T_H + lane_off + c, vh);
        tmem_ld_x16(T_DH + lane_off + c, vd);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j)
          vh[j] = __float_as_uint(__fadd_rn(__fmul_rn(__uint_as_float(vh[j]), eQ), __uint_as_float(vd[j])));
        tmem_st_x16(T_H + lane_off + c, vh);
      }
      tmem_wait_st();
    }
    __syncthreads();   // staged outputs visible
    {
      const int p4 = (tid & 15) * 4;
#pragma unroll 4
      for (int i = 0; i < TQ / 16; ++i) {
        const int t = (tid >> 4) + 16 * i;
        if (t < Qc) {
          const float4 v = *reinterpret_cast<const float4*>(&ys[t * (TP + 4) + p4]);
          const uint32_t zc = *reinterpret_cast<const uint32_t*>(rz + t * TP + p4);
          float4 o;
          o.x = __fmul_rn(v.x, s_lut[(int)(int8_t)(zc) + 128]);
          o.y = __fmul_rn(v.y, s_lut[(int)(int8_t)(zc >> 8) + 128]);
          o.z = __fmul_rn(v.z, s_lut[(int)(int8_t)(zc >> 16) + 128]);
          o.w = __fmul_rn(v.w, s_lut[(int)(int8_t)(zc >> 24) + 128]);
          *reinterpret_cast<float4*>(y + (tok0 + c0 + t) * ldy + ch0 + p4) = o;
        }
      }
    }
    tc_fence_before();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // ---- final state -> int8 codes [p][n] (ClusterMap-cell scales)
  {
    const int n = row;
    int8_t* st = state + ((int64_t)b * p.n_heads + h) * TP * N;
    tc_fence_after();
#pragma unroll
    for (int c = hw * 32; c < hw * 32 + 32; c += 16) {
      uint32_t v[16];
      tmem_ld_x16(T_H + lane_off + c, v);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) st[(c + j) * N + n] = quant8(__uint_as_float(v[j]), p.s_h[ch0 + c + j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int launch_ssd_chunk_tc(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx, const int8_t* Bm,
                        const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt, const int8_t* z, int64_t ldz,
                        int8_t* state, int state_in, float* y, int64_t ldy, cudaStream_t st) {
  if (p->head_dim != TP || p->d_state != TN) return SQ_ERR_ARG;
  if (ldx % 16 || ldbc % 16 || ldz % 16 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(Bm) & 15) || (reinterpret_cast<uintptr_t>(Cm) & 15) ||
      (reinterpret_cast<uintptr_t>(z) & 15) || ldy % 4 || (reinterpret_cast<uintptr_t>(y) & 15))
    return SQ_ERR_ARG;
  static std::once_flag once[64];   // per device
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(ssd_chunk_tc_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSsdSmem::ALLOC);
  });
  ssd_chunk_tc_kernel<TN><<<dim3(p->n_heads, B), TC_SSD_THREADS, TcSsdSmem::ALLOC, st>>>(
      *p, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy);
  return check_launch("sq_ssd_scan_int8 (tcgen05 chunks)");
}

}  // namespace sq
