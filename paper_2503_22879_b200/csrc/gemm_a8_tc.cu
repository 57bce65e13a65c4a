// K1/K2 on the 5th-gen tensor cores: A8 projection GEMM with tcgen05.mma kind::i8,
// TMEM accumulators, TMA-fed activation tiles and (for W4A8) on-the-fly int4 -> int8
// weight expansion (LEDGER G11b: w8 = w4 * sg, exact int32 over K).
//
// Swap-AB formulation: the CTA's 128 weight rows are the MMA M side (one TMEM lane per
// output channel) and the token tile (16..256) is the MMA N side, so small-batch decode
// (M = 64 tokens) still issues full-height 128xN MMAs while the weights stream once.
//
//   warp 0      TMA producer: activation K-blocks [NTOK x 128 B] (SWIZZLE_128B) and, for
//               W8, the weight K-block [128 x 128 B]
//   warp 1      TMEM allocator + single-thread MMA issuer (4 x K=32 per stage)
//   warps 2..9  W4: converters — each thread owns one weight row, reads its packed
//               nibbles from the smem ring, expands them to UINT8 (v+8)*sg with one IMUL per
//               4 bytes and writes the A operand straight into TMEM (tcgen05.st; kind::i8
//               A-from-TMEM) or into a swizzled smem tile (WMODE 2);  all: epilogue
//   warp 10     W4: per-token group sums S[kb][t] of every activation tile (dp4a), used by
//               the epilogue to undo the +8 offset:  acc -= 8 * sum_kb sg[n,kb] * S[kb][t]
//   warp 11     W4: streams the contiguous 8 KB packed-weight tiles into a deep smem ring
//               with 1-D bulk TMA (cp.async.bulk), so HBM latency never stalls conversion
//
// Split-K (small N, e.g. out_proj N=4096): SPLITS CTAs of one output tile form a cluster;
// each reduces a token slice of the int32 partials through DSMEM in fixed rank order,
// so results are deterministic and bit-exact (integer sums).
//
// Epilogue per (n, t): y = f32(acc) * alpha[n] -> I32 | F32 | int8 requant | residual add.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace sq {
using namespace sm100;

constexpr int TC_BN = 128;
constexpr int TC_BK = 128;
constexpr int TC_ACOL = 256;      // first TMEM column of the A (weight) stages in TS mode
constexpr int TC_THREADS = 384;     // 12 warps: TMA, MMA, 8 converter/epilogue, group-sum, W4 stream
constexpr int TC_MAX_KB = 64;       // max K-blocks per split (K <= 8192)
constexpr int W4_TILE_BYTES = TC_BN * TC_BK / 2;  // 8 KB per (n-tile, k-block)
// packed-weight ring depth for small token tiles (8 KB slots).  Same-box A/B of the decode step
// with 2-k-block converter batches (scripts/ab_lib.sh): 6 / 8 / 10 / 12 / 14 / 16 slots ->
// 15.38k / 15.43k / 15.31k / 15.17k / 14.83k / 13.80k tok/s, so 64 KB in flight per SM wins.
#ifndef SQ_RAW64
#define SQ_RAW64 8
#endif
constexpr int g_raw64 = SQ_RAW64;

enum { WM_W8 = 0, WM_W4_TS = 1, WM_W4_SS = 2 };

struct TcArgs {
  const uint8_t* w4;
  const int8_t* sg;
  int group;
  const float* alpha;
  int M, N, K;
  int epi;
  void* out;
  int64_t ldo;
  const float* col_scale;
  const int32_t* gsum;   // optional precomputed activation sums per 128-K block [M x K/128]
  int64_t ldg;
  int dbg;   // profiling only (SQ_GEMM_DBG): 1 = skip the group-sum arithmetic, 2 = CTA timeline, 64 = time 512 back-to-back MMAs first
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// 4 signed nibbles (low 16 bits of x) -> 4 int8 = nibble * sg via byte LUTs
//   L0 = [0,1,2,3]*sg  L1 = [4..7]*sg  L2 = [-8..-5]*sg  L3 = [-4..-1]*sg
__device__ __forceinline__ uint32_t nib4_to_s8(uint32_t x, uint32_t L0, uint32_t L1, uint32_t L2, uint32_t L3) {
  const uint32_t sel = x & 0x7777u;
  const uint32_t p = prmt(L0, L1, sel);
  const uint32_t q = prmt(L2, L3, sel);
  const uint32_t msel = ((x >> 3) & 0x1111u) ^ 0x9999u;   // nibble bit3 ? 0x8 : 0x9
  const uint32_t mask = prmt(0x80u, 0u, msel);             // 0xFF where the nibble is negative
  return (p & ~mask) | (q & mask);
}

// Kernel nibble order inside every 32-bit word (set by sq_repack_w4): byte j holds
// element j (low nibble) and element j+4 (high nibble), so one AND / one SHF+AND split a
// word into elements 0-3 and 4-7 already in byte order.
__host__ __device__ __forceinline__ uint32_t spread4(uint32_t x) {   // nibbles 0..3 -> bytes 0..3
  x = (x | (x << 8)) & 0x00FF00FFu;
  return (x | (x << 4)) & 0x0F0F0F0Fu;
}
__host__ __device__ __forceinline__ uint32_t compact4(uint32_t x) {  // inverse of spread4
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return (x | (x >> 8)) & 0x0000FFFFu;
}
__host__ __device__ __forceinline__ uint32_t nib_permute(uint32_t std_word) {
  return spread4(std_word & 0xFFFFu) | (spread4(std_word >> 16) << 4);
}
__host__ __device__ __forceinline__ uint32_t nib_unpermute(uint32_t w) {
  return compact4(w & 0x0F0F0F0Fu) | (compact4((w >> 4) & 0x0F0F0F0Fu) << 16);
}

// Unsigned-offset expansion for the tensor core: (v + 8) * sg  in [0, 225] per byte.
// The A operand is fed as UINT8; the epilogue subtracts 8 * sum_g sg[n,g] * S[t,g].
__device__ __forceinline__ void nib8_to_u8(uint32_t w, uint32_t sg, uint32_t& lo, uint32_t& hi) {
  const uint32_t u = w ^ 0x88888888u;
  lo = (u & 0x0F0F0F0Fu) * sg;
  hi = ((u >> 4) & 0x0F0F0F0Fu) * sg;
}

__device__ __forceinline__ int4 ldg_stream(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void epi_store(const TcArgs& a, int m, int n, int v, float alpha, float cs, float ics) {
  const int64_t o = (int64_t)m * a.ldo + n;
  if (a.epi == SQ_EPI_I32) {
    reinterpret_cast<int32_t*>(a.out)[o] = v;
    return;
  }
  const float y = __fmul_rn((float)v, alpha);
  if (a.epi == SQ_EPI_F32)
    reinterpret_cast<float*>(a.out)[o] = y;
  else if (a.epi == SQ_EPI_QUANT)
    reinterpret_cast<int8_t*>(a.out)[o] = quant8_inv(y, cs, ics);
  else
    reinterpret_cast<float*>(a.out)[o] = __fadd_rn(reinterpret_cast<float*>(a.out)[o], y);
}

template <int NTOK, int WMODE, int SPLITS, int STAGES, int RAW>
struct TcCfg {
  static constexpr bool W4 = WMODE != WM_W8;
  // offset correction on the tensor core (extra accumulators need 3*NTOK <= TC_ACOL columns)
  static constexpr bool MMA_CORR = (WMODE == WM_W4_TS) && NTOK <= 64;
  static constexpr int ACT_BYTES = NTOK * TC_BK;
  static constexpr int W_BYTES = (WMODE == WM_W4_TS) ? 0 : TC_BN * TC_BK;
  static constexpr int STAGE_BYTES = ACT_BYTES + W_BYTES;
  static constexpr int RAW_BYTES = W4 ? RAW * W4_TILE_BYTES : 0;
  static constexpr int SUM_BYTES = W4 ? TC_MAX_KB * NTOK * 4 : 0;    // S[kb][t]
  static constexpr int SGS_BYTES = W4 ? TC_MAX_KB * TC_BN : 0;        // sg[kb][row]
  static constexpr int OFF_W = STAGES * ACT_BYTES;
  static constexpr int OFF_RAW = OFF_W + STAGES * W_BYTES;
  static constexpr int OFF_SUM = OFF_RAW + RAW_BYTES;
  static constexpr int OFF_SGS = OFF_SUM + SUM_BYTES;
  static constexpr int OFF_BAR = OFF_SGS + SGS_BYTES;
  static constexpr int NBAR = 2 * STAGES + 2 * RAW + 2;
  static constexpr int OFF_EPI = OFF_BAR + NBAR * 8 + 16;   // alpha[128], col_scale[128]
  static constexpr int SMEM0 = 1024 + OFF_EPI + 2 * TC_BN * 4;
  // W4: 1 CTA/SM (TMEM alloc of 512 cols: accumulators + A stages).  W8: accumulators only
  // (<= 256 cols), two CTAs per SM so one CTA's epilogue overlaps the other's main loop.
  static constexpr int TMEM_COLS = W4 ? 512 : 256;
  static constexpr int SMEM = (W4 && SMEM0 < 120 * 1024) ? 120 * 1024 : SMEM0;
};

template <int NTOK, int WMODE, int SPLITS, int STAGES, int RAW>
__global__ void __launch_bounds__(TC_THREADS, WMODE == WM_W8 ? 2 : 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w, TcArgs args) {
  using Cfg = TcCfg<NTOK, WMODE, SPLITS, STAGES, RAW>;
  // converter batch: D k-blocks per raw-ring barrier and per TMEM-stage wait (D < STAGES, no self-wait)
#ifndef SQ_CONV_D
#define SQ_CONV_D 2
#endif
  constexpr int D = STAGES >= 8 ? SQ_CONV_D : (STAGES >= 4 ? 2 : 1);
  constexpr int RB = RAW / D;   // raw-ring batch slots
  static_assert(WMODE == WM_W8 || RAW % D == 0, "raw ring must hold whole converter batches");
  constexpr bool W4 = Cfg::W4;
  // byte offsets from the extern array keep every access in the shared space (LDS/STS)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // SW128 atoms need 1 KB
  uint8_t* act = smem;
  uint8_t* wsm = smem + Cfg::OFF_W;
  uint8_t* raw = smem + Cfg::OFF_RAW;
  int32_t* gsum = reinterpret_cast<int32_t*>(smem + Cfg::OFF_SUM);
  int8_t* sgs = reinterpret_cast<int8_t*>(smem + Cfg::OFF_SGS);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* rfull = empty + STAGES;
  uint64_t* rempty = rfull + RAW;
  uint64_t* accf = rempty + RAW;
  uint64_t* corr_ready = accf + 1;     // MMA_CORR: H/L tiles + TMEM sg column written
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(corr_ready + 1);
  uint8_t* bh = smem + Cfg::OFF_SUM;                 // MMA_CORR: S>>7 as [2 ksteps][NTOK x 32 B] no-swizzle
  uint8_t* bl = bh + 2 * NTOK * 32;                  //           S&127

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, split = blockIdx.y, m_tile = blockIdx.z;
  const bool tl = (args.dbg & 2) && lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && split == 0;
  const uint64_t t_entry = tl ? gtimer() : 0;
  uint64_t t_raw0 = 0, t_rawl = 0, t_conv_done = 0, t_acc = 0, t_epi0 = 0, t_epi1 = 0, t_ld0 = 0, t_loop = 0;
  long long c_raw = 0, c_emp = 0, c_stw = 0, c_full = 0;   // timeline: SM cycles spent waiting
  long long c_b0 = 0, c_b1 = 0, c_b2 = 0;                  // timeline: convert / store / signal phases
  uint64_t t_mloop = 0, t_mcorr = 0;                       // timeline: MMA warp issue progress
  const int nkb_total = args.K / TC_BK;
  const int kb_begin = split * nkb_total / SPLITS;
  const int nkb = (split + 1) * nkb_total / SPLITS - kb_begin;

  pdl_trigger();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], W4 ? 1 + 8 : 1);      // TMA (+ 8 converter warps)
      mbar_init(&empty[s], (W4 && !args.gsum) ? 2 : 1);   // MMA commit (+ group-sum warp)
    }
    for (int r = 0; r < RB; ++r) {
      mbar_init(&rfull[r], 1);
      mbar_init(&rempty[r], 8);
    }
    mbar_init(accf, 1);
    mbar_init(corr_ready, 1 + 4);        // group-sum warp + the 4 sg-staging converter warps
    fence_barrier_init();
    tma_prefetch(&tm_act);
    if (!W4) tma_prefetch(&tm_w);
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- activation (and W8 weight) TMA producer
    pdl_wait();   // activations come from the previous grid
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait_lazy(&empty[s], ((i / STAGES) & 1) ^ 1);   // polling would steal converter issue slots
        mbar_arrive_expect_tx(&full[s], Cfg::ACT_BYTES + (W4 ? 0 : Cfg::W_BYTES));
        tma_load_2d(act + s * Cfg::ACT_BYTES, &tm_act, &full[s], (kb_begin + i) * TC_BK, m_tile * NTOK);
        if (!W4) tma_load_2d(wsm + s * Cfg::W_BYTES, &tm_w, &full[s], (kb_begin + i) * TC_BK, n_tile * TC_BN);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- single-thread MMA issuer
    if (lane == 0) {
      // W4: A = (v+8)*sg as UINT8 (corrected in the epilogue); W8: signed x signed
      constexpr uint32_t idesc = W4 ? (idesc_i8(TC_BN, NTOK) & ~(7u << 7)) : idesc_i8(TC_BN, NTOK);
      if ((args.dbg & 64) && blockIdx.x == 0 && split == 0) {
        // profiling (scripts/mma_rate.sh): issue rate of back-to-back MMAs on garbage operands
        // (the main loop's first MMA overwrites the accumulator, so results stay correct)
        const long long c0 = clock64();
        for (int r = 0; r < 512; ++r) {
          const int s = (r / 4) % STAGES, ks = r % 4;
          if (WMODE == WM_W4_TS)
            mma_i8_ts(tmem, tmem + TC_ACOL + s * 32 + ks * 8, desc_sw128(act + s * Cfg::ACT_BYTES) + 2 * ks, idesc, 1u);
          else
            mma_i8_ss(tmem, desc_sw128(wsm + s * Cfg::W_BYTES) + 2 * ks, desc_sw128(act + s * Cfg::ACT_BYTES) + 2 * ks,
                      idesc, 1u);
        }
        printf("gemm mma-rate N=%d NTOK=%d mode=%d: %.1f cycles per MMA issue (512 MMAs)\n", args.N, NTOK, WMODE,
               (clock64() - c0) / 512.0);
      }
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const long long c0 = tl ? clock64() : 0;
        mbar_wait(&full[s], (i / STAGES) & 1);
        if (tl) c_full += clock64() - c0;
        tc_fence_after();
        const uint64_t bdesc = desc_sw128(act + s * Cfg::ACT_BYTES);
#pragma unroll
        for (int ks = 0; ks < TC_BK / 32; ++ks) {
          const uint32_t acc = (i > 0 || ks > 0) ? 1u : 0u;
          if (args.dbg & 32) continue;   // profiling: no main-loop MMAs (commit only)
          if (WMODE == WM_W4_TS) {
            mma_i8_ts(tmem, tmem + TC_ACOL + s * 32 + ks * 8, bdesc + 2 * ks, idesc, acc);
          } else {
            const uint64_t adesc = desc_sw128(wsm + s * Cfg::W_BYTES);
            mma_i8_ss(tmem, adesc + 2 * ks, bdesc + 2 * ks, idesc, acc);
          }
        }
        mma_commit(&empty[s]);
      }
      t_mloop = tl ? gtimer() : 0;
      if (Cfg::MMA_CORR) {
        // dH = sum_kb sg[n,kb] * (S[kb][t] >> 7), dL = sum_kb sg[n,kb] * (S[kb][t] & 127)
        mbar_wait(corr_ready, 0);
        tc_fence_after();
        constexpr uint32_t id_h = (idesc_i8(TC_BN, NTOK) & ~(7u << 7));                  // u8 x s8
        constexpr uint32_t id_l = (idesc_i8(TC_BN, NTOK) & ~(7u << 7)) & ~(7u << 10);    // u8 x u8
        const int ksteps = (nkb + 31) / 32;
        for (int ks = 0; ks < ksteps; ++ks) {
          mma_i8_ts(tmem + 64, tmem + 192 + ks * 8, desc_noswz(bh + ks * NTOK * 32, 128, 256), id_h, ks > 0);
          mma_i8_ts(tmem + 128, tmem + 192 + ks * 8, desc_noswz(bl + ks * NTOK * 32, 128, 256), id_l, ks > 0);
        }
      }
      mma_commit(accf);
      t_mcorr = tl ? gtimer() : 0;
    }
    __syncwarp();
  } else if (warp == 10) {
    // ---------------- group sums S[kb][t] of every activation tile (W4 only)
    if (W4) {
      if (Cfg::MMA_CORR) {   // zero the (padded) K range of both B tiles
        for (int o = lane * 16; o < 4 * NTOK * 32; o += 32 * 16) *reinterpret_cast<int4*>(bh + o) = make_int4(0, 0, 0, 0);
        __syncwarp();
      }
      pdl_wait();
      if (args.gsum) {
        // sums precomputed by the producer of the activations: just stage them
        for (int idx = lane; idx < NTOK * nkb; idx += 32) {
          const int t = idx / nkb, i = idx % nkb;
          const int m = m_tile * NTOK + t;
          const int acc = m < args.M ? args.gsum[(int64_t)m * args.ldg + kb_begin + i] : 0;
          if (Cfg::MMA_CORR) {
            const int o = (i >> 5) * NTOK * 32 + (t >> 3) * 256 + ((i >> 4) & 1) * 128 + (t & 7) * 16 + (i & 15);
            bh[o] = (uint8_t)(acc >> 7);
            bl[o] = (uint8_t)(acc & 127);
          } else {
            gsum[i * NTOK + t] = acc;
          }
        }
        __syncwarp();
      }
      for (int i = 0; i < nkb && !args.gsum; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        const uint8_t* tile = act + s * Cfg::ACT_BYTES;
        for (int t = lane; t < NTOK && !(args.dbg & 1); t += 32) {
          int acc = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {   // any chunk order sums the row; rotate per lane -> no bank conflicts
            const int4 v = *reinterpret_cast<const int4*>(tile + t * TC_BK + ((c ^ (t & 7)) * 16));
            acc = __dp4a(v.x, 0x01010101, acc);
            acc = __dp4a(v.y, 0x01010101, acc);
            acc = __dp4a(v.z, 0x01010101, acc);
            acc = __dp4a(v.w, 0x01010101, acc);
          }
          if (Cfg::MMA_CORR) {
            // element (t, kb) of a no-swizzle K-major [NTOK x 32 B] tile per 32-kb step
            const int o = (i >> 5) * NTOK * 32 + (t >> 3) * 256 + ((i >> 4) & 1) * 128 + (t & 7) * 16 + (i & 15);
            bh[o] = (uint8_t)(acc >> 7);
            bl[o] = (uint8_t)(acc & 127);
          } else {
            gsum[i * NTOK + t] = acc;
          }
        }
        fence_proxy_async_smem();   // generic reads of the stage precede the next TMA write into it
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (Cfg::MMA_CORR) {
        fence_proxy_async_smem();          // generic smem writes -> tensor-core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(corr_ready);
      }
      named_bar(1, 288);   // sums complete -> epilogue warps
    }
  } else if (warp == 11) {
    // ---------------- packed W4 tiles: contiguous 8 KB per (n-tile, k-block) -> smem ring
    if (W4 && lane == 0) {
      const uint8_t* src = args.w4 + ((size_t)n_tile * nkb_total + kb_begin) * W4_TILE_BYTES;
      for (int bi = 0; bi * D < nkb; ++bi) {   // one barrier per converter batch of D tiles
        const int r = bi % RB;
        mbar_wait_lazy(&rempty[r], ((bi / RB) & 1) ^ 1);
        const int n = min(D, nkb - bi * D);
        mbar_arrive_expect_tx(&rfull[r], n * W4_TILE_BYTES);
        for (int t = 0; t < n; ++t)
          bulk_load(raw + (r * D + t) * W4_TILE_BYTES, src + (size_t)(bi * D + t) * W4_TILE_BYTES, W4_TILE_BYTES,
                    &rfull[r]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;              // TMEM lane quadrant this warp may touch
    const int half = (warp - 2) >> 2;    // which half of the K-block / of the token columns
    const int row = q * 32 + lane;
    const int n = n_tile * TC_BN + row;
    const bool valid_n = n < args.N;
    // epilogue scales fetched now, so their latency hides behind the main loop
    float* s_alpha = reinterpret_cast<float*>(smem + Cfg::OFF_EPI);
    float* s_cs = s_alpha + TC_BN;
    if (half == 0) {
      s_alpha[row] = (valid_n && args.epi != SQ_EPI_I32) ? args.alpha[n] : 0.f;
      s_cs[row] = (valid_n && args.epi == SQ_EPI_QUANT) ? args.col_scale[n] : 1.f;
    }
    if (W4) {
      const int8_t* sgr = args.sg + (size_t)(valid_n ? n : 0) * (args.K / args.group);
      if (half == 0) {
        // all of this row's group scales (<= 64 bytes, zero beyond nkb) in registers
        const int8_t* p = sgr + kb_begin * TC_BK / args.group;
        int4 v[TC_MAX_KB / 16];
        if (args.group == TC_BK && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (nkb & 15) == 0) {
#pragma unroll
          for (int c = 0; c < TC_MAX_KB / 16; ++c)
            v[c] = (valid_n && c * 16 < nkb) ? *reinterpret_cast<const int4*>(p + c * 16) : make_int4(0, 0, 0, 0);
        } else {
          uint32_t wds[TC_MAX_KB / 4];
#pragma unroll
          for (int w = 0; w < TC_MAX_KB / 4; ++w) wds[w] = 0;
#pragma unroll
          for (int i = 0; i < TC_MAX_KB; ++i)
            if (valid_n && i < nkb) wds[i / 4] |= (uint32_t)(uint8_t)sgr[(kb_begin + i) * TC_BK / args.group] << (8 * (i % 4));
#pragma unroll
          for (int c = 0; c < TC_MAX_KB / 16; ++c) v[c] = make_int4(wds[c * 4], wds[c * 4 + 1], wds[c * 4 + 2], wds[c * 4 + 3]);
        }
#pragma unroll
        for (int c = 0; c < TC_MAX_KB / 16; ++c)
          if (c * 16 < nkb) {
            const uint32_t wq[4] = {(uint32_t)v[c].x, (uint32_t)v[c].y, (uint32_t)v[c].z, (uint32_t)v[c].w};
#pragma unroll
            for (int e = 0; e < 16; ++e) sgs[(c * 16 + e) * TC_BN + row] = (int8_t)(wq[e / 4] >> (8 * (e % 4)));
          }
        if (Cfg::MMA_CORR) {   // A operand of the correction MMAs: sg[row][kb] in TMEM cols 192..207
          uint32_t cw[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            cw[c * 4] = v[c].x; cw[c * 4 + 1] = v[c].y; cw[c * 4 + 2] = v[c].z; cw[c * 4 + 3] = v[c].w;
          }
          tmem_st_x16(tmem + ((uint32_t)(q * 32) << 16) + 192, cw);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(corr_ready);
        }
      }
      named_bar(2, 256);                 // converter warps: sg staged
      for (int i0 = 0; i0 < nkb; i0 += D) {
        const int rb = (i0 / D) % RB, nb = min(D, nkb - i0);
        const long long cb0 = tl ? clock64() : 0;
        // (1) the batch's tiles landed; (2) every smem read of the batch issued together; (3)
        // the expansion of D tiles interleaved — no barrier wait sits between a load and the
        // next tile's load, so the LDS / IMUL latencies overlap across the batch.
        uint32_t wv[D][16];
        {
          const long long c0 = tl ? clock64() : 0;
          mbar_wait(&rfull[rb], ((i0 / D) / RB) & 1);
          if (tl) c_raw += clock64() - c0;
          if (tl && warp == 2 && i0 == 0) t_raw0 = gtimer();
          if (tl && warp == 2 && i0 + D >= nkb) t_rawl = gtimer();
        }
        uint4 p0[D], p1[D];
        uint32_t sgv[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const int i = min(i0 + j, nkb - 1);
          const uint8_t* rp = raw + (rb * D + (i - i0)) * W4_TILE_BYTES + half * 2 * 2048 + row * 16;
          p0[j] = *reinterpret_cast<const uint4*>(rp);
          p1[j] = *reinterpret_cast<const uint4*>(rp + 2048);
          sgv[j] = (uint32_t)(uint8_t)sgs[i * TC_BN + row];
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          nib8_to_u8(p0[j].x, sgv[j], wv[j][0], wv[j][1]);
          nib8_to_u8(p0[j].y, sgv[j], wv[j][2], wv[j][3]);
          nib8_to_u8(p0[j].z, sgv[j], wv[j][4], wv[j][5]);
          nib8_to_u8(p0[j].w, sgv[j], wv[j][6], wv[j][7]);
          nib8_to_u8(p1[j].x, sgv[j], wv[j][8], wv[j][9]);
          nib8_to_u8(p1[j].y, sgv[j], wv[j][10], wv[j][11]);
          nib8_to_u8(p1[j].z, sgv[j], wv[j][12], wv[j][13]);
          nib8_to_u8(p1[j].w, sgv[j], wv[j][14], wv[j][15]);
        }
        // generic-proxy reads of the raw slot are ordered before the bulk copy (async proxy)
        // that will refill it
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&rempty[rb]);
        }
        const long long cb1 = tl ? clock64() : 0;
        {
          // the batch's stages are free once the MMA read their previous contents; MMAs and
          // their commits complete in issue order, so the batch's last stage implies the rest
          // (the barriers are never more than one phase ahead: the MMA waits on our arrivals)
          const int il = i0 + nb - 1;
          const long long c0 = tl ? clock64() : 0;
          mbar_wait(&empty[il % STAGES], ((il / STAGES) & 1) ^ 1);
          if (tl) c_emp += clock64() - c0;
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const int i = i0 + j;
          if (i < nkb) {
            const int s = i % STAGES;
            if (WMODE == WM_W4_TS) {
              if (!(args.dbg & 4)) tmem_st_x16(tmem + ((uint32_t)(q * 32) << 16) + TC_ACOL + s * 32 + half * 16, wv[j]);
              // publish each stage as soon as it is in TMEM, so the MMA issuer starts on the
              // batch's first k-block while the later ones are still being stored (shorter MMA
              // tail after the last batch); the wait covers only this warp's stores
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&full[s]);
            } else {
              // swizzled SW128 K-major tile: row r, 16-byte chunk c at ((c ^ (r&7)) * 16)
              uint8_t* base = wsm + s * Cfg::W_BYTES + (row >> 3) * 1024 + (row & 7) * 128;
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int c16 = half * 4 + c;
                *reinterpret_cast<uint4*>(base + ((c16 ^ (row & 7)) * 16)) =
                    make_uint4(wv[j][c * 4], wv[j][c * 4 + 1], wv[j][c * 4 + 2], wv[j][c * 4 + 3]);
              }
            }
          }
        }
        const long long cb2 = tl ? clock64() : 0;
        if (WMODE != WM_W4_TS) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < D; ++j)
              if (i0 + j < nkb) mbar_arrive(&full[(i0 + j) % STAGES]);
          }
        }
        if (tl) {
          const long long cb3 = clock64();
          c_b0 += cb1 - cb0;
          c_b1 += cb2 - cb1;
          c_b2 += cb3 - cb2;
        }
      }
    }
    // ---------------- epilogue: TMEM -> registers -> (offset correction) -> HBM / DSMEM
    if (tl && warp == 2) t_conv_done = gtimer();
    mbar_wait(accf, 0);
    tc_fence_after();
    if (tl && warp == 2) t_acc = gtimer();
    if (W4) named_bar(1, 288);           // group sums ready
    if (tl && warp == 2) t_epi0 = gtimer();
    pdl_wait();                          // outputs / residual belong to earlier grids too
    named_bar(3, 256);                   // s_alpha / s_cs (stored at kernel start) visible
    const float alpha = s_alpha[row], cs = s_cs[row];
    const float ics = __frcp_rn(cs);
    constexpr int CH = NTOK / 2;
    int32_t* red = reinterpret_cast<int32_t*>(act);     // split-K: [NTOK][128], aliases the act stages
    // staging the whole fp32 tile can exceed the stage area when two CTAs share an SM (W8):
    // then the token halves are staged and stored one after the other
    const int esz = args.epi == SQ_EPI_QUANT ? 1 : 4;
    const int npass = (SPLITS == 1 && NTOK * TC_BN * esz > Cfg::OFF_SUM) ? 2 : 1;
    static_assert(SPLITS > 1 || NTOK * TC_BN * 2 <= Cfg::OFF_SUM, "half a fp32 tile must fit the stage area");
    // (W4 tiles wider than 128 tokens run without split-K: gemm_a8_tc dispatch)
    static_assert(SPLITS == 1 || (W4 && NTOK > 128) || NTOK * TC_BN * 4 <= Cfg::OFF_SUM,
                  "split-K reduction tile must fit the stage area");
    for (int pass = 0; pass < npass; ++pass) {
    const int tbase = npass == 2 ? pass * CH : 0;        // first token of this pass's staging buffer
    const int tcount = npass == 2 ? CH : NTOK;
#pragma unroll 1
    for (int c0 = half * CH; c0 < (half + 1) * CH && (npass == 1 || half == pass); c0 += 8) {
      uint32_t v[8];
      tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
      tmem_wait_ld();
      if (tl && warp == 2 && c0 == half * CH) t_ld0 = gtimer();
      int val[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) val[j] = (int)v[j];
      if (Cfg::MMA_CORR) {
        uint32_t vh[8], vl[8];
        tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + 64 + c0, vh);
        tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + 128 + c0, vl);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) val[j] -= 1024 * (int)vh[j] + 8 * (int)vl[j];
      } else if (W4) {
        // undo the +8 offset of the unsigned weight operand: acc -= 8 * sum_kb sg[n,kb] * S[kb][t]
        int corr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 4
        for (int i = 0; i < nkb; ++i) {
          const int sgv = sgs[i * TC_BN + row];
          const int4 g0 = *reinterpret_cast<const int4*>(&gsum[i * NTOK + c0]);
          const int4 g1 = *reinterpret_cast<const int4*>(&gsum[i * NTOK + c0 + 4]);
          corr[0] += sgv * g0.x; corr[1] += sgv * g0.y; corr[2] += sgv * g0.z; corr[3] += sgv * g0.w;
          corr[4] += sgv * g1.x; corr[5] += sgv * g1.y; corr[6] += sgv * g1.z; corr[7] += sgv * g1.w;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) val[j] -= 8 * corr[j];
      }
      if (SPLITS == 1) {
        // stage [NTOK][TC_BN] in smem (aliases the activation stages: every MMA has completed)
        if (args.epi == SQ_EPI_QUANT && (args.dbg & 16)) {
#pragma unroll
          for (int j = 0; j < 8; ++j) act[(c0 + j - tbase) * TC_BN + row] = (uint8_t)val[j];
        } else if (args.epi == SQ_EPI_QUANT) {
          float yv[8];
          int8_t qv[8];
          bool tie = false;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            yv[j] = __fmul_rn((float)val[j], alpha);
            qv[j] = quant8_fast(yv[j], ics, tie);
          }
          if (tie) {   // rare: a value within 1e-4 of a rounding tie -> exact division
#pragma unroll
            for (int j = 0; j < 8; ++j) qv[j] = quant8(yv[j], cs);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) act[(c0 + j - tbase) * TC_BN + row] = (uint8_t)qv[j];
        } else {
          uint32_t* st32 = reinterpret_cast<uint32_t*>(act);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            st32[(c0 + j - tbase) * TC_BN + row] =
                args.epi == SQ_EPI_I32 ? (uint32_t)val[j] : __float_as_uint(__fmul_rn((float)val[j], alpha));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) red[(c0 + j) * TC_BN + row] = val[j];
      }
    }
    if (tl && warp == 2) t_loop = gtimer();
    if (SPLITS == 1) {
      // coalesced 16-B stores of the staged tile (residual epilogue: 16-B read-add-write)
      named_bar(3, 256);
      const int et = threadIdx.x - 64;
      const int per16 = 16 / esz;
      const int chunks = TC_BN / per16;
      // residual epilogue: the read-add-write is done in batches of RU items whose residual
      // loads are all issued before any add/store (a store may alias a later load as far as
      // the compiler knows, so an item-at-a-time loop pays one HBM latency per item)
      constexpr int RU = 4;
      int idx0 = et;
      if (args.epi == SQ_EPI_RESID) {
        for (; idx0 + 256 * (RU - 1) < tcount * chunks; idx0 += 256 * RU) {
          float4 o[RU];
          float* d[RU];
          bool fast[RU];
#pragma unroll
          for (int u = 0; u < RU; ++u) {
            const int idx = idx0 + 256 * u;
            const int ts = idx / chunks, c = idx % chunks;
            const int m = m_tile * NTOK + tbase + ts;
            const int n0 = n_tile * TC_BN + c * per16;
            d[u] = reinterpret_cast<float*>(args.out) + (int64_t)m * args.ldo + n0;
            fast[u] = m < args.M && n0 + per16 <= args.N && (reinterpret_cast<uintptr_t>(d[u]) & 15) == 0;
            o[u] = fast[u] ? *reinterpret_cast<const float4*>(d[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < RU; ++u) {
            const int idx = idx0 + 256 * u;
            const int ts = idx / chunks, c = idx % chunks;
            const float* src = reinterpret_cast<const float*>(act) + ts * TC_BN + c * per16;
            if (fast[u]) {
              const float4 v = *reinterpret_cast<const float4*>(src);
              *reinterpret_cast<float4*>(d[u]) = make_float4(__fadd_rn(o[u].x, v.x), __fadd_rn(o[u].y, v.y),
                                                             __fadd_rn(o[u].z, v.z), __fadd_rn(o[u].w, v.w));
            } else {
              const int m = m_tile * NTOK + tbase + ts;
              const int n0 = n_tile * TC_BN + c * per16;
              if (m >= args.M || n0 >= args.N) continue;
              for (int e = 0; e < min(per16, args.N - n0); ++e) d[u][e] = __fadd_rn(d[u][e], src[e]);
            }
          }
        }
      }
      for (int idx = idx0; idx < tcount * chunks; idx += 256) {
        const int ts = idx / chunks, c = idx % chunks;
        const int t = tbase + ts;
        const int m = m_tile * NTOK + t;
        const int n0 = n_tile * TC_BN + c * per16;
        if (m >= args.M || n0 >= args.N) continue;
        const uint8_t* src = act + (ts * TC_BN + c * per16) * esz;
        uint8_t* dst = reinterpret_cast<uint8_t*>(args.out) + ((int64_t)m * args.ldo + n0) * esz;
        const int nv = min(per16, args.N - n0);
        if (nv == per16 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          uint4 v = *reinterpret_cast<const uint4*>(src);
          if (args.epi == SQ_EPI_RESID) {
            const float4 o = *reinterpret_cast<const float4*>(dst);
            v.x = __float_as_uint(__fadd_rn(o.x, __uint_as_float(v.x)));
            v.y = __float_as_uint(__fadd_rn(o.y, __uint_as_float(v.y)));
            v.z = __float_as_uint(__fadd_rn(o.z, __uint_as_float(v.z)));
            v.w = __float_as_uint(__fadd_rn(o.w, __uint_as_float(v.w)));
          }
          *reinterpret_cast<uint4*>(dst) = v;
        } else {
          for (int e = 0; e < nv; ++e) {
            if (esz == 1) {
              dst[e] = src[e];
            } else {
              const uint32_t v = reinterpret_cast<const uint32_t*>(src)[e];
              float* d = reinterpret_cast<float*>(dst) + e;
              if (args.epi == SQ_EPI_RESID) *d = __fadd_rn(*d, __uint_as_float(v));
              else *reinterpret_cast<uint32_t*>(d) = v;
            }
          }
        }
      }
    }
      if (npass == 2 && pass == 0) named_bar(3, 256);   // staging buffer reused by the next pass
    }
  }

  if (tl && warp == 2) t_epi1 = gtimer();
  if (SPLITS > 1) {
    pdl_wait();
    __syncwarp();
    cluster_sync();
    const uint32_t rank = cluster_rank();
    constexpr int TPR = NTOK / SPLITS;   // tokens reduced by this CTA
    int32_t* red = reinterpret_cast<int32_t*>(act);
    const uint32_t red_addr = smem_u32(red);
    // 4 consecutive output channels per thread: one 16-B DSMEM load per peer, all in flight
    for (int idx = threadIdx.x; idx < TPR * (TC_BN / 4); idx += TC_THREADS) {
      const int t = rank * TPR + idx / (TC_BN / 4);
      const int r = (idx % (TC_BN / 4)) * 4;
      int4 part[SPLITS];
#pragma unroll
      for (int j = 0; j < SPLITS; ++j) part[j] = ld_dsmem_v4s32(map_peer(red_addr + (t * TC_BN + r) * 4, j));
      int sum[4] = {0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < SPLITS; ++j) {   // fixed rank order: deterministic (and exact: int32)
        sum[0] += part[j].x; sum[1] += part[j].y; sum[2] += part[j].z; sum[3] += part[j].w;
      }
      const int m = m_tile * NTOK + t;
      if (m >= args.M) continue;
      const float* s_alpha = reinterpret_cast<const float*>(smem + Cfg::OFF_EPI);
      const int n0 = n_tile * TC_BN + r;
      const int64_t o = (int64_t)m * args.ldo + n0;
      if ((args.epi == SQ_EPI_F32 || args.epi == SQ_EPI_RESID) && n0 + 3 < args.N &&
          (reinterpret_cast<uintptr_t>(reinterpret_cast<float*>(args.out) + o) & 15) == 0) {
        // four contiguous channels: one 16-B store (16-B read-add-write for the residual)
        const float4 al = *reinterpret_cast<const float4*>(s_alpha + r);
        float4 yv = make_float4(__fmul_rn((float)sum[0], al.x), __fmul_rn((float)sum[1], al.y),
                                __fmul_rn((float)sum[2], al.z), __fmul_rn((float)sum[3], al.w));
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(args.out) + o);
        if (args.epi == SQ_EPI_RESID) {
          const float4 h = *dst;
          yv = make_float4(__fadd_rn(h.x, yv.x), __fadd_rn(h.y, yv.y), __fadd_rn(h.z, yv.z), __fadd_rn(h.w, yv.w));
        }
        *dst = yv;
        continue;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int nn = n0 + e;
        if (nn < args.N) {
          const float cs = s_alpha[TC_BN + r + e];
          epi_store(args, m, nn, sum[e], s_alpha[r + e], cs, __frcp_rn(cs));
        }
      }
    }
    cluster_sync();
  }
  tc_fence_before();
  __syncthreads();
  if (tl && warp == 2)
    printf("gemm cta %d N=%d K=%d: raw0 %.2f rawlast %.2f conv_done %.2f acc %.2f epi0 %.2f epi1 %.2f end %.2f us\n",
           blockIdx.x, args.N, args.K, (t_raw0 - t_entry) * 1e-3, (t_rawl - t_entry) * 1e-3,
           (t_conv_done - t_entry) * 1e-3, (t_acc - t_entry) * 1e-3, (t_epi0 - t_entry) * 1e-3,
           (t_epi1 - t_entry) * 1e-3, (gtimer() - t_entry) * 1e-3);
  if (tl && warp == 2)
    printf("gemm cta %d: first tmem ld %.2f  loop end %.2f us\n", blockIdx.x, (t_ld0 - t_entry) * 1e-3,
           (t_loop - t_entry) * 1e-3);
  if (tl && warp == 2 && lane == 0)
    printf("gemm cta %d waits (cycles): converter rfull %lld empty %lld wait_st %lld | phases convert %lld store %lld "
           "signal %lld\n", blockIdx.x, c_raw, c_emp, c_stw, c_b0, c_b1, c_b2);
  if (tl && warp == 1 && lane == 0)
    printf("gemm cta %d waits (cycles): mma full %lld | main-loop MMAs issued %.2f us, correction issued %.2f us\n",
           blockIdx.x, c_full, (t_mloop - t_entry) * 1e-3, (t_mcorr - t_entry) * 1e-3);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem);
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encoder() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode != nullptr;
}

static int make_map_2d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                       uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int NTOK, int WMODE, int SPLITS>
static int launch_tc(const int8_t* a, int64_t lda, const uint8_t* w, const TcArgs& args, cudaStream_t st) {
  constexpr int RAW = WMODE == WM_W8 ? 1 : (NTOK <= 64 ? g_raw64 : (NTOK == 128 ? 8 : 6));
  using C1 = TcCfg<NTOK, WMODE, SPLITS, 1, RAW>;
  // W8 targets two CTAs per SM (~105 KB each); W4 one CTA with the raw ring
  // (split-K keeps the one-CTA budget: its int32 reduction tile [NTOK][128] needs the room)
  // (W8 split-K with small token tiles: the [NTOK][128] int32 reduction tile is small, so it
  //  keeps the two-CTA budget and small-batch projections spread over twice the CTAs)
  constexpr int BUDGET = (WMODE == WM_W8 && (SPLITS == 1 || NTOK <= 32)) ? 104 * 1024 : 210 * 1024;
  constexpr int ST0 = (BUDGET - C1::RAW_BYTES - C1::SUM_BYTES - C1::SGS_BYTES) / C1::STAGE_BYTES;
  constexpr int STAGES = ST0 > 8 ? 8 : (ST0 < 2 ? 2 : ST0);
  using Cfg = TcCfg<NTOK, WMODE, SPLITS, STAGES, RAW>;
  static_assert(Cfg::SMEM <= 227 * 1024, "smem budget");
  auto kern = gemm_tc_kernel<NTOK, WMODE, SPLITS, STAGES, RAW>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (SPLITS > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  CUtensorMap tm_act, tm_w;
  if (!make_map_2d(&tm_act, a, (uint64_t)args.K, (uint64_t)args.M, (uint64_t)lda, TC_BK, NTOK)) {
    set_error("gemm_tc: activation tensor map encode failed");
    return SQ_ERR_CUDA;
  }
  if (WMODE == WM_W8) {
    if (!make_map_2d(&tm_w, w, (uint64_t)args.K, (uint64_t)args.N, (uint64_t)args.K, TC_BK, TC_BN)) {
      set_error("gemm_tc: weight tensor map encode failed");
      return SQ_ERR_CUDA;
    }
  } else {
    tm_w = tm_act;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((args.N + TC_BN - 1) / TC_BN, SPLITS, (args.M + NTOK - 1) / NTOK);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (SPLITS > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1;
    at[na].val.clusterDim.y = SPLITS;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled(PDL_GEMM)) {   // weights stream in while the previous grid drains (see common.cuh)
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm_act, tm_w, args);
  if (e != cudaSuccess) {
    set_error("gemm_tc launch: %s", cudaGetErrorString(e));
    return SQ_ERR_CUDA;
  }
  return check_launch("gemm_tc");
}

template <int WMODE, int SPLITS>
static int dispatch_ntok(int ntok, const int8_t* a, int64_t lda, const uint8_t* w, const TcArgs& args,
                         cudaStream_t st) {
  switch (ntok) {
    case 16: return launch_tc<16, WMODE, SPLITS>(a, lda, w, args, st);
    case 32: return launch_tc<32, WMODE, SPLITS>(a, lda, w, args, st);
    case 64: return launch_tc<64, WMODE, SPLITS>(a, lda, w, args, st);
    case 128: return launch_tc<128, WMODE, SPLITS>(a, lda, w, args, st);
    default: return launch_tc<256, WMODE, SPLITS>(a, lda, w, args, st);
  }
}

template <int WMODE>
static int dispatch_split(int splits, int ntok, const int8_t* a, int64_t lda, const uint8_t* w, const TcArgs& args,
                          cudaStream_t st) {
  switch (splits) {
    case 1: return dispatch_ntok<WMODE, 1>(ntok, a, lda, w, args, st);
    case 2: return dispatch_ntok<WMODE, 2>(ntok, a, lda, w, args, st);
    case 4: return dispatch_ntok<WMODE, 4>(ntok, a, lda, w, args, st);
    default: return dispatch_ntok<WMODE, 8>(ntok, a, lda, w, args, st);
  }
}

int g_tc_w4_mode = WM_W4_TS;   // sq_set_gemm_mode() switches TS/SS for A/B measurements

// Returns SQ_ERR_ARG when the shape is not eligible (caller falls back to mma.sync).
int gemm_a8_tc(const int8_t* a, int64_t lda, const uint8_t* w, const int8_t* sg, int group, bool w4,
               const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
               const int32_t* a_gsum, int64_t ld_gsum, cudaStream_t st) {
  if (K % TC_BK != 0 || (w4 && group % TC_BK != 0) || lda % 16 != 0 || (reinterpret_cast<uintptr_t>(a) & 15) ||
      (!w4 && (reinterpret_cast<uintptr_t>(w) & 15)))
    return SQ_ERR_ARG;
  if (!get_encoder()) return SQ_ERR_ARG;
  static const int ntok_force = [] {   // profiling: SQ_GEMM_NTOK forces the token tile
    const char* e = getenv("SQ_GEMM_NTOK");
    return e ? atoi(e) : 0;
  }();
  int ntok = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
  if (ntok_force) ntok = ntok_force;
  const int tiles = ((N + TC_BN - 1) / TC_BN) * ((M + ntok - 1) / ntok);
  const int nkb = K / TC_BK;
  int splits = 1;
  const int slots = (!w4 && ntok <= 32) ? 2 * 148 : 148;   // resident CTAs (see launch_tc BUDGET)
  while (splits < 8 && tiles * splits * 2 <= slots && nkb / (splits * 2) >= 4 && ntok % (splits * 2) == 0) splits *= 2;
  if (w4 && (nkb + splits - 1) / splits > TC_MAX_KB) return SQ_ERR_ARG;
  static const int dbg = [] {
    const char* e = getenv("SQ_GEMM_DBG");
    return e ? atoi(e) : 0;
  }();
  TcArgs args{w, sg, group, alpha, M, N, K, epi, out, ldo, col_scale, w4 ? a_gsum : nullptr, ld_gsum, dbg};
  if (!w4) return dispatch_split<WM_W8>(splits, ntok, a, lda, w, args, st);
  // A-from-TMEM is used up to 128-token tiles (the 256-column accumulator leaves too few
  // TMEM columns for the A stages); larger tiles stage the expanded weights in smem.
  // SS (weights expanded into smem) is used without split-K only.
  if (ntok > 128) return dispatch_split<WM_W4_SS>(1, ntok, a, lda, w, args, st);
  if (g_tc_w4_mode == WM_W4_SS && splits == 1) return dispatch_split<WM_W4_SS>(1, ntok, a, lda, w, args, st);
  return dispatch_split<WM_W4_TS>(splits, ntok, a, lda, w, args, st);
}

// W4 kernel layout: [n_tile][k_block][chunk 0..3][row 0..127][16 B]; rows >= N zero.
__global__ void repack_w4_kernel(const uint8_t* __restrict__ src, int N, int K, uint8_t* __restrict__ dst) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one 16-B piece
  const int nkb = K / TC_BK;
  const int64_t pieces = (int64_t)((N + TC_BN - 1) / TC_BN) * nkb * 4 * TC_BN;
  if (idx >= pieces) return;
  const int row = idx % TC_BN;
  const int chunk = (idx / TC_BN) % 4;
  const int kb = (idx / (TC_BN * 4)) % nkb;
  const int tile = idx / ((int64_t)TC_BN * 4 * nkb);
  const int n = tile * TC_BN + row;
  int4 v = make_int4(0, 0, 0, 0);
  if (n < N) v = *reinterpret_cast<const int4*>(src + (int64_t)n * (K / 2) + kb * 64 + chunk * 16);
  v.x = (int)nib_permute((uint32_t)v.x);
  v.y = (int)nib_permute((uint32_t)v.y);
  v.z = (int)nib_permute((uint32_t)v.z);
  v.w = (int)nib_permute((uint32_t)v.w);
  *reinterpret_cast<int4*>(dst + idx * 16) = v;
}

__global__ void unpack_w4_kernel(const uint8_t* __restrict__ src, int N, int K, uint8_t* __restrict__ dst) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nkb = K / TC_BK;
  const int64_t pieces = (int64_t)N * nkb * 4;
  if (idx >= pieces) return;
  const int n = idx / (nkb * 4);
  const int kb = (idx / 4) % nkb;
  const int chunk = idx % 4;
  const int tile = n / TC_BN, row = n % TC_BN;
  const int64_t s = ((((int64_t)tile * nkb + kb) * 4 + chunk) * TC_BN + row) * 16;
  int4 v = *reinterpret_cast<const int4*>(src + s);
  v.x = (int)nib_unpermute((uint32_t)v.x);
  v.y = (int)nib_unpermute((uint32_t)v.y);
  v.z = (int)nib_unpermute((uint32_t)v.z);
  v.w = (int)nib_unpermute((uint32_t)v.w);
  *reinterpret_cast<int4*>(dst + (int64_t)n * (K / 2) + kb * 64 + chunk * 16) = v;
}

int64_t w4_layout_bytes(int N, int K) {
  if (K % TC_BK == 0) return (int64_t)((N + TC_BN - 1) / TC_BN) * TC_BN * K / 2;
  return (int64_t)N * K / 2;
}

int repack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st) {
  if (K % TC_BK != 0) {
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)N * K / 2, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SQ_OK : SQ_ERR_CUDA;
  }
  const int64_t pieces = (int64_t)((N + TC_BN - 1) / TC_BN) * (K / TC_BK) * 4 * TC_BN;
  repack_w4_kernel<<<(unsigned)((pieces + 255) / 256), 256, 0, st>>>(src, N, K, dst);
  return check_launch("sq_repack_w4");
}

int unpack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st) {
  if (K % TC_BK != 0) {
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)N * K / 2, cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? SQ_OK : SQ_ERR_CUDA;
  }
  const int64_t pieces = (int64_t)N * (K / TC_BK) * 4;
  unpack_w4_kernel<<<(unsigned)((pieces + 255) / 256), 256, 0, st>>>(src, N, K, dst);
  return check_launch("sq_unpack_w4");
}

}  // namespace sq
