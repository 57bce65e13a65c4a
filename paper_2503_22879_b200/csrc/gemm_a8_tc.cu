// K1 on the 5th-gen tensor cores: W8A8 projection GEMM with tcgen05.mma kind::i8, TMEM
// accumulators and TMA-fed operand tiles.  W8A8 weights are
// per-output-channel (SPEC PerChannel, LEDGER G11), so the int32 accumulator spans all of K and
// the epilogue applies alpha[n] = f32(s_w[n] * s_a) (quantizer.fuse_scales).
// (W4A8 has per-group scales and its own kernel, gemm_w4a8.cu.)
//
// Swap-AB formulation: the CTA's 128 weight rows are the MMA M side (one TMEM lane per output
// channel) and the token tile (16..256) is the MMA N side, so small-batch projections still
// issue full-height 128xN MMAs while the weights stream once.
//
//   warp 0      TMA producer: activation K-block [NTOK x 128 B] and weight K-block [128 x 128 B]
//               (both SWIZZLE_128B) into a STAGES-deep ring
//   warp 1      TMEM allocator + single-thread MMA issuer (4 x K=32 per stage)
//   warps 2..9  epilogue: TMEM -> registers -> staged tile -> coalesced 16-B stores
//
// Split-K (small N): SPLITS CTAs of one output tile form a cluster; each reduces a token slice
// of the int32 partials through DSMEM in fixed rank order (integer sums: exact).
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
constexpr int TC_THREADS = 320;     // 10 warps: TMA, MMA, 8 epilogue

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


template <int NTOK, int SPLITS, int STAGES>
struct TcCfg {
  static constexpr int ACT_BYTES = NTOK * TC_BK;
  static constexpr int W_BYTES = TC_BN * TC_BK;
  static constexpr int STAGE_BYTES = ACT_BYTES + W_BYTES;
  static constexpr int OFF_W = STAGES * ACT_BYTES;
  static constexpr int OFF_BAR = OFF_W + STAGES * W_BYTES;
  static constexpr int NBAR = 2 * STAGES + 1;
  static constexpr int OFF_EPI = (OFF_BAR + NBAR * 8 + 16 + 15) & ~15;   // alpha[128], col_scale[128] (16-B aligned)
  static constexpr int SMEM = 1024 + OFF_EPI + 2 * TC_BN * 4;
  static constexpr int TMEM_COLS = NTOK <= 32 ? 32 : NTOK;   // power of two >= 32
};

struct TcArgs {
  const float* alpha;
  int M, N, K;
  int epi;
  void* out;
  int64_t ldo;
  const float* col_scale;
};

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

template <int NTOK, int SPLITS, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_act, const __grid_constant__ CUtensorMap tm_w, TcArgs args) {
  using Cfg = TcCfg<NTOK, SPLITS, STAGES>;
  // byte offsets from the extern array keep every access in the shared space (LDS/STS)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // SW128 atoms need 1 KB
  uint8_t* act = smem;
  uint8_t* wsm = smem + Cfg::OFF_W;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(accf + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, split = blockIdx.y, m_tile = blockIdx.z;
  const int nkb_total = (args.K + TC_BK - 1) / TC_BK;   // a partial last K-block is zero-filled by TMA
  const int kb_begin = split * nkb_total / SPLITS;
  const int nkb = (split + 1) * nkb_total / SPLITS - kb_begin;

  pdl_trigger();
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
    tma_prefetch(&tm_act);
    tma_prefetch(&tm_w);
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- activation + weight TMA producer
    pdl_wait();   // activations come from the previous grid
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait_lazy(&empty[s], ((i / STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        tma_load_2d(act + s * Cfg::ACT_BYTES, &tm_act, &full[s], (kb_begin + i) * TC_BK, m_tile * NTOK);
        tma_load_2d(wsm + s * Cfg::W_BYTES, &tm_w, &full[s], (kb_begin + i) * TC_BK, n_tile * TC_BN);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- single-thread MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(TC_BN, NTOK);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(&full[s], (i / STAGES) & 1);
        tc_fence_after();
        const uint64_t adesc = desc_sw128(wsm + s * Cfg::W_BYTES);
        const uint64_t bdesc = desc_sw128(act + s * Cfg::ACT_BYTES);
#pragma unroll
        for (int ks = 0; ks < TC_BK / 32; ++ks)
          mma_i8_ss(tmem, adesc + 2 * ks, bdesc + 2 * ks, idesc, (i > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&empty[s]);
      }
      mma_commit(accf);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: TMEM -> registers -> staged tile / DSMEM -> HBM
    const int q = warp & 3;              // TMEM lane quadrant this warp may touch
    const int half = (warp - 2) >> 2;    // which half of the token columns
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
    mbar_wait(accf, 0);
    tc_fence_after();
    pdl_wait();                          // outputs / residual belong to earlier grids too
    named_bar(3, 256);                   // s_alpha / s_cs visible
    const float alpha = s_alpha[row], cs = s_cs[row];
    const float ics = __frcp_rn(cs);
    constexpr int CH = NTOK / 2;
    int32_t* red = reinterpret_cast<int32_t*>(act);     // split-K: [NTOK][128], aliases the stages
    // staging the whole fp32 tile can exceed the stage area when two CTAs share an SM: then the
    // token halves are staged and stored one after the other
    const int esz = args.epi == SQ_EPI_QUANT ? 1 : 4;
    const int npass = (SPLITS == 1 && NTOK * TC_BN * esz > Cfg::OFF_BAR) ? 2 : 1;
    static_assert(SPLITS > 1 || NTOK * TC_BN * 2 <= Cfg::OFF_BAR, "half a fp32 tile must fit the stage area");
    static_assert(SPLITS == 1 || NTOK * TC_BN * 4 <= Cfg::OFF_BAR, "split-K reduction tile must fit the stage area");
    for (int pass = 0; pass < npass; ++pass) {
      const int tbase = npass == 2 ? pass * CH : 0;        // first token of this pass's staging buffer
      const int tcount = npass == 2 ? CH : NTOK;
#pragma unroll 1
      for (int c0 = half * CH; c0 < (half + 1) * CH && (npass == 1 || half == pass); c0 += 8) {
        uint32_t v[8];
        tmem_ld_x8(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
        tmem_wait_ld();
        int val[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) val[j] = (int)v[j];
        if (SPLITS == 1) {
          // stage [NTOK][TC_BN] in smem (aliases the stages: every MMA has completed)
          if (args.epi == SQ_EPI_QUANT) {
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

  if (SPLITS > 1) {
    pdl_wait();
    __syncwarp();
    cluster_sync();
    const uint32_t rank = cluster_rank();
    constexpr int TPR = NTOK / SPLITS;   // tokens reduced by this CTA
    int32_t* red = reinterpret_cast<int32_t*>(act);
    const uint32_t red_addr = smem_u32(red);
    const float* s_alpha = reinterpret_cast<const float*>(smem + Cfg::OFF_EPI);
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

template <int NTOK, int SPLITS>
static int launch_tc(const int8_t* a, int64_t lda, const uint8_t* w, const TcArgs& args, cudaStream_t st) {
  // two CTAs per SM (~105 KB each) so one CTA's epilogue overlaps the other's main loop; split-K
  // with wide token tiles keeps the one-CTA budget (its int32 reduction tile needs the room)
  using C1 = TcCfg<NTOK, SPLITS, 1>;
  constexpr int BUDGET = (SPLITS == 1 || NTOK <= 32) ? 104 * 1024 : 210 * 1024;
  constexpr int ST0 = BUDGET / C1::STAGE_BYTES;
  constexpr int STAGES = ST0 > 8 ? 8 : (ST0 < 2 ? 2 : ST0);
  using Cfg = TcCfg<NTOK, SPLITS, STAGES>;
  static_assert(Cfg::SMEM <= 227 * 1024, "smem budget");
  auto kern = gemm_tc_kernel<NTOK, SPLITS, STAGES>;
  static std::once_flag once[64];   // per device: a process may drive several GPUs
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (SPLITS > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
  CUtensorMap tm_act, tm_w;
  if (!make_map_2d(&tm_act, a, (uint64_t)args.K, (uint64_t)args.M, (uint64_t)lda, TC_BK, NTOK) ||
      !make_map_2d(&tm_w, w, (uint64_t)args.K, (uint64_t)args.N, (uint64_t)args.K, TC_BK, TC_BN)) {
    set_error("gemm_tc: tensor map encode failed");
    return SQ_ERR_CUDA;
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
  if (pdl_enabled(PDL_GEMM)) {   // the next grid's prologue overlaps this one's tail (common.cuh)
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

template <int SPLITS>
static int dispatch_ntok(int ntok, const int8_t* a, int64_t lda, const uint8_t* w, const TcArgs& args,
                         cudaStream_t st) {
  switch (ntok) {
    case 16: return launch_tc<16, SPLITS>(a, lda, w, args, st);
    case 32: return launch_tc<32, SPLITS>(a, lda, w, args, st);
    case 64: return launch_tc<64, SPLITS>(a, lda, w, args, st);
    case 128: return launch_tc<128, SPLITS>(a, lda, w, args, st);
    default: return launch_tc<256, SPLITS>(a, lda, w, args, st);
  }
}

// Returns SQ_ERR_ARG when the shape is not eligible (caller falls back to mma.sync).
int gemm_a8_tc(const int8_t* a, int64_t lda, const uint8_t* w, const float* alpha, int M, int N, int K, int epi,
               void* out, int64_t ldo, const float* col_scale, cudaStream_t st) {
  // K need not be a multiple of 128 (e.g. Mamba1 dt_proj, K = dt_rank = 160): the TMA boxes past K
  // are zero-filled for both operands, so the padded products add nothing; rows must be 16-B aligned
  if (K % 16 != 0 || lda % 16 != 0 || (reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(w) & 15))
    return SQ_ERR_ARG;
  if (!get_encoder()) return SQ_ERR_ARG;
  int ntok = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
  const int nkb = (K + TC_BK - 1) / TC_BK;
  auto pick_splits = [&](int nt) {
    const int tiles = ((N + TC_BN - 1) / TC_BN) * ((M + nt - 1) / nt);
    const int slots = nt <= 32 ? 2 * 148 : 148;   // resident CTAs (see launch_tc BUDGET)
    int s = 1;
    while (s < 8 && tiles * s * 2 <= slots && nkb / (s * 2) >= 4 && nt % (s * 2) == 0) s *= 2;
    return s;
  };
  int splits = pick_splits(ntok);
  // mid-size M with few 256-token tiles (e.g. the 2.8B out_proj at 1024 tokens: 80 tiles, 37 us)
  // fills more SMs with 128-token tiles (160 tiles, 22.5 us; scripts/probe_tc.py)
  if (ntok == 256 && splits == 1 && ((N + TC_BN - 1) / TC_BN) * ((M + 255) / 256) < 148) {
    ntok = 128;
    splits = pick_splits(ntok);
  }
  TcArgs args{alpha, M, N, K, epi, out, ldo, col_scale};
  switch (splits) {
    case 1: return dispatch_ntok<1>(ntok, a, lda, w, args, st);
    case 2: return dispatch_ntok<2>(ntok, a, lda, w, args, st);
    case 4: return dispatch_ntok<4>(ntok, a, lda, w, args, st);
    default: return dispatch_ntok<8>(ntok, a, lda, w, args, st);
  }
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
