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
//   warps 2..9  W4: converters — each thread owns one weight row, streams its packed
//               nibbles with coalesced 16-B loads (repacked tile layout, sq_repack_w4),
//               expands them with a per-(row, group) byte LUT (v*sg) and writes the int8
//               A operand straight into TMEM (tcgen05.st; kind::i8 A-from-TMEM) or into a
//               swizzled smem tile (WMODE 2);  all: epilogue (TMEM -> regs -> HBM)
//
// Split-K (small N, e.g. out_proj N=4096): SPLITS CTAs of one output tile form a cluster;
// each reduces a token slice of the int32 partials through DSMEM in fixed rank order,
// so results are deterministic and bit-exact (integer sums).
//
// Epilogue per (n, t): y = f32(acc) * alpha[n] -> I32 | F32 | int8 requant | residual add.
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace sq {
using namespace sm100;

constexpr int TC_BN = 128;
constexpr int TC_BK = 128;
constexpr int TC_ACOL = 256;      // first TMEM column of the A (weight) stages in TS mode
constexpr int TC_THREADS = 320;
constexpr int W4_TILE_BYTES = TC_BN * TC_BK / 2;  // 8 KB per (n-tile, k-block)

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

__device__ __forceinline__ int4 ldg_stream(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void epi_store(const TcArgs& a, int m, int n, int v, float alpha, float cs) {
  const int64_t o = (int64_t)m * a.ldo + n;
  if (a.epi == SQ_EPI_I32) {
    reinterpret_cast<int32_t*>(a.out)[o] = v;
    return;
  }
  const float y = __fmul_rn((float)v, alpha);
  if (a.epi == SQ_EPI_F32)
    reinterpret_cast<float*>(a.out)[o] = y;
  else if (a.epi == SQ_EPI_QUANT)
    reinterpret_cast<int8_t*>(a.out)[o] = quant8(y, cs);
  else
    reinterpret_cast<float*>(a.out)[o] = __fadd_rn(reinterpret_cast<float*>(a.out)[o], y);
}

template <int NTOK, int WMODE, int SPLITS, int STAGES>
struct TcCfg {
  static constexpr int ACT_BYTES = NTOK * TC_BK;
  static constexpr int W_BYTES = (WMODE == WM_W4_TS) ? 0 : TC_BN * TC_BK;
  static constexpr int STAGE_BYTES = ACT_BYTES + W_BYTES;
  static constexpr int SMEM0 = 1024 + STAGES * STAGE_BYTES + 2 * STAGES * 8 + 64;
  static constexpr int SMEM = SMEM0 < 120 * 1024 ? 120 * 1024 : SMEM0;   // 1 CTA/SM: TMEM alloc of 512 cols
};

template <int NTOK, int WMODE, int SPLITS, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w, TcArgs args) {
  using Cfg = TcCfg<NTOK, WMODE, SPLITS, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act = smem;
  uint8_t* wsm = smem + STAGES * Cfg::ACT_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, split = blockIdx.y, m_tile = blockIdx.z;
  const int nkb_total = args.K / TC_BK;
  const int kb_begin = split * nkb_total / SPLITS;
  const int nkb = (split + 1) * nkb_total / SPLITS - kb_begin;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], WMODE == WM_W8 ? 1 : 1 + 8);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
    tma_prefetch(&tm_act);
    if (WMODE == WM_W8) tma_prefetch(&tm_w);
  }
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::ACT_BYTES + (WMODE == WM_W8 ? Cfg::W_BYTES : 0));
        tma_load_2d(act + s * Cfg::ACT_BYTES, &tm_act, &full[s], (kb_begin + i) * TC_BK, m_tile * NTOK);
        if (WMODE == WM_W8)
          tma_load_2d(wsm + s * Cfg::W_BYTES, &tm_w, &full[s], (kb_begin + i) * TC_BK, n_tile * TC_BN);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(TC_BN, NTOK);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        tc_fence_after();
        const uint64_t bdesc = desc_sw128(act + s * Cfg::ACT_BYTES);
#pragma unroll
        for (int ks = 0; ks < TC_BK / 32; ++ks) {
          const uint32_t acc = (i > 0 || ks > 0) ? 1u : 0u;
          if (WMODE == WM_W4_TS) {
            mma_i8_ts(tmem, tmem + TC_ACOL + s * 32 + ks * 8, bdesc + 2 * ks, idesc, acc);
          } else {
            const uint64_t adesc = desc_sw128(wsm + s * Cfg::W_BYTES);
            mma_i8_ss(tmem, adesc + 2 * ks, bdesc + 2 * ks, idesc, acc);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;              // TMEM lane quadrant this warp may touch
    const int half = (warp - 2) >> 2;    // which half of the K-block / of the token columns
    const int row = q * 32 + lane;
    const int n = n_tile * TC_BN + row;
    const bool valid_n = n < args.N;
    if (WMODE != WM_W8) {
      // Batched converter: D K-blocks are converted, stored (TMEM or smem) and released
      // together, so the tcgen05.st / proxy-fence latency is paid once per batch while
      // the next batch's weight loads are already in flight.
      constexpr int D = 4;
      const uint8_t* wsrc = args.w4 + (size_t)n_tile * nkb_total * W4_TILE_BYTES + row * 16 + half * 2 * 2048;
      const int ng = args.K / args.group;
      const int8_t* sgrow = args.sg + (size_t)(valid_n ? n : 0) * ng;
      int4 buf[D][2];
      int sgb[D];
      auto fetch = [&](int i, int j) {
        if (i < nkb && valid_n) {
          const uint8_t* p = wsrc + (size_t)(kb_begin + i) * W4_TILE_BYTES;
          buf[j][0] = ldg_stream(p);
          buf[j][1] = ldg_stream(p + 2048);
          sgb[j] = sgrow[(kb_begin + i) * TC_BK / args.group];
        } else {
          buf[j][0] = buf[j][1] = make_int4(0, 0, 0, 0);
          sgb[j] = 0;
        }
      };
#pragma unroll
      for (int j = 0; j < D; ++j) fetch(j, j);
      for (int i0 = 0; i0 < nkb; i0 += D) {
        uint32_t wv[D][16];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const uint32_t sg = (uint32_t)sgb[j];
          const uint32_t L0 = sg * 0x03020100u, L1 = sg * 0x07060504u;
          const uint32_t L2 = ~(sg * 0x05060708u) + 0x01010101u, L3 = ~(sg * 0x01020304u) + 0x01010101u;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(&buf[j][c]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              wv[j][c * 8 + e * 2] = nib4_to_s8(pw[e], L0, L1, L2, L3);
              wv[j][c * 8 + e * 2 + 1] = nib4_to_s8(pw[e] >> 16, L0, L1, L2, L3);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < D; ++j) fetch(i0 + D + j, j);   // next batch in flight
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const int i = i0 + j;
          if (i < nkb) {
            const int s = i % STAGES;
            mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
            if (WMODE == WM_W4_TS) {
              tmem_st_x16(tmem + ((uint32_t)(q * 32) << 16) + TC_ACOL + s * 32 + half * 16, wv[j]);
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
        if (WMODE == WM_W4_TS) {
          tmem_wait_st();
          tc_fence_before();
        } else {
          fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < D; ++j)
            if (i0 + j < nkb) mbar_arrive(&full[(i0 + j) % STAGES]);
        }
      }
    }
    // ---------------- epilogue
    mbar_wait(accf, 0);
    tc_fence_after();
    const float alpha = (valid_n && args.epi != SQ_EPI_I32) ? args.alpha[n] : 0.f;
    const float cs = (valid_n && args.epi == SQ_EPI_QUANT) ? args.col_scale[n] : 1.f;
    constexpr int CH = NTOK / 2;
    constexpr int CW = CH < 8 ? CH : 8;
    if (SPLITS == 1) {
#pragma unroll 1
      for (int c0 = half * CH; c0 < (half + 1) * CH; c0 += 8) {
        uint32_t v[8];
        tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int m = m_tile * NTOK + c0 + j;
          if (valid_n && m < args.M) epi_store(args, m, n, (int)v[j], alpha, cs);
        }
      }
    } else {
      int32_t* red = reinterpret_cast<int32_t*>(act);     // [NTOK][128], aliases the act stages
#pragma unroll 1
      for (int c0 = half * CH; c0 < (half + 1) * CH; c0 += 8) {
        uint32_t v[8];
        tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) red[(c0 + j) * TC_BN + row] = (int)v[j];
      }
      (void)CW;
    }
  }

  if (SPLITS > 1) {
    __syncwarp();
    cluster_sync();
    const uint32_t rank = cluster_rank();
    constexpr int TPR = NTOK / SPLITS;   // tokens reduced by this CTA
    int32_t* red = reinterpret_cast<int32_t*>(act);
    const uint32_t red_addr = smem_u32(red);
    for (int idx = threadIdx.x; idx < TPR * TC_BN; idx += TC_THREADS) {
      const int t = rank * TPR + idx / TC_BN;
      const int r = idx % TC_BN;
      const int nn = n_tile * TC_BN + r;
      const int m = m_tile * NTOK + t;
      int sum = 0;
#pragma unroll
      for (int j = 0; j < SPLITS; ++j) sum += ld_dsmem_s32(map_peer(red_addr + (t * TC_BN + r) * 4, j));
      if (nn < args.N && m < args.M) {
        const float al = args.epi != SQ_EPI_I32 ? args.alpha[nn] : 0.f;
        const float cs = args.epi == SQ_EPI_QUANT ? args.col_scale[nn] : 1.f;
        epi_store(args, m, nn, sum, al, cs);
      }
    }
    cluster_sync();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
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
  constexpr int STAGE_BYTES = TcCfg<NTOK, WMODE, SPLITS, 1>::STAGE_BYTES;
  constexpr int ST0 = (200 * 1024) / STAGE_BYTES;
  constexpr int STAGES = ST0 > 8 ? 8 : (ST0 < 2 ? 2 : ST0);
  using Cfg = TcCfg<NTOK, WMODE, SPLITS, STAGES>;
  auto kern = gemm_tc_kernel<NTOK, WMODE, SPLITS, STAGES>;
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
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = SPLITS;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = SPLITS > 1 ? 1 : 0;
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
               cudaStream_t st) {
  if (K % TC_BK != 0 || (w4 && group % TC_BK != 0) || lda % 16 != 0 || (reinterpret_cast<uintptr_t>(a) & 15) ||
      (!w4 && (reinterpret_cast<uintptr_t>(w) & 15)))
    return SQ_ERR_ARG;
  if (!get_encoder()) return SQ_ERR_ARG;
  const int ntok = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
  const int tiles = ((N + TC_BN - 1) / TC_BN) * ((M + ntok - 1) / ntok);
  const int nkb = K / TC_BK;
  int splits = 1;
  while (splits < 8 && tiles * splits * 2 <= 148 && nkb / (splits * 2) >= 4 && ntok % (splits * 2) == 0) splits *= 2;
  TcArgs args{w, sg, group, alpha, M, N, K, epi, out, ldo, col_scale};
  if (!w4) return dispatch_split<WM_W8>(splits, ntok, a, lda, w, args, st);
  if (g_tc_w4_mode == WM_W4_SS) return dispatch_split<WM_W4_SS>(splits, ntok, a, lda, w, args, st);
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
  *reinterpret_cast<int4*>(dst + (int64_t)n * (K / 2) + kb * 64 + chunk * 16) = *reinterpret_cast<const int4*>(src + s);
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
