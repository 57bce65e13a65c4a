// C-ABI entry points for the A8 projections (K1/K2) and the int4 weight layout.
#include "common.cuh"

namespace sq {
extern int g_tc_w4_mode;
static int g_gemm_mode = 1;   // 0: mma.sync only, 1: tcgen05 (TS for W4), 2: tcgen05 (SS for W4)
int gemm_a8_tc(const int8_t* a, int64_t lda, const uint8_t* w, const int8_t* sg, int group, bool w4,
               const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
               const int32_t* a_gsum, int64_t ld_gsum, cudaStream_t st);
int64_t w4_layout_bytes(int N, int K);
int repack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st);
int unpack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st);
int gemm_a8_mma(const int8_t* a, int64_t lda, const uint8_t* w, const int8_t* sg, int group, bool w4,
                const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
                cudaStream_t st);

static int check_gemm(const char* name, const void* a, int64_t lda, int M, int N, int K, int epi, int64_t ldo,
                      const float* col_scale) {
  SQ_REQUIRE(M >= 0 && N > 0 && K > 0, SQ_ERR_SHAPE, "%s: bad M/N/K (%d,%d,%d)", name, M, N, K);
  SQ_REQUIRE(K % 32 == 0, SQ_ERR_SHAPE, "%s: K (%d) must be a multiple of 32", name, K);
  SQ_REQUIRE(lda % 16 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0, SQ_ERR_LAYOUT,
             "%s: activation rows must be 16-byte aligned", name);
  SQ_REQUIRE(epi >= SQ_EPI_I32 && epi <= SQ_EPI_RESID, SQ_ERR_ARG, "%s: bad epilogue %d", name, epi);
  SQ_REQUIRE(epi != SQ_EPI_QUANT || col_scale != nullptr, SQ_ERR_ARG, "%s: QUANT epilogue needs col_scale", name);
  SQ_REQUIRE(ldo >= N, SQ_ERR_SHAPE, "%s: ldo < N", name);
  return SQ_OK;
}
}  // namespace sq

using namespace sq;

extern "C" int64_t sq_w4_bytes(int N, int K) { return w4_layout_bytes(N, K); }

// Kernel layout (K % 128 == 0): [n_tile][k_block][chunk][row][16 B] so a warp's 32 weight
// rows load 512 contiguous bytes per instruction; otherwise row-major u4packed.
// sq_unpack_w4 inverts it (bit-exact round trip, tested).
extern "C" int sq_repack_w4(const uint8_t* u4packed, int N, int K, uint8_t* dst, void* stream) {
  SQ_REQUIRE(N > 0 && K > 0 && K % 32 == 0, SQ_ERR_SHAPE, "sq_repack_w4: K must be a multiple of 32");
  return repack_w4(u4packed, N, K, dst, as_stream(stream));
}

extern "C" int sq_unpack_w4(const uint8_t* src, int N, int K, uint8_t* u4packed, void* stream) {
  SQ_REQUIRE(N > 0 && K > 0 && K % 32 == 0, SQ_ERR_SHAPE, "sq_unpack_w4: K must be a multiple of 32");
  return unpack_w4(src, N, K, u4packed, as_stream(stream));
}

extern "C" int sq_set_gemm_mode(int mode) {
  SQ_REQUIRE(mode >= 0 && mode <= 2, SQ_ERR_ARG, "sq_set_gemm_mode: mode must be 0, 1 or 2");
  g_gemm_mode = mode;
  g_tc_w4_mode = mode == 2 ? 2 : 1;
  return SQ_OK;
}

extern "C" int sq_gemm_w8a8(const int8_t* a, int64_t lda, const int8_t* w, const float* alpha, int M, int N, int K,
                            int epi, void* out, int64_t ldo, const float* col_scale, void* stream) {
  int rc = check_gemm("sq_gemm_w8a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  if (M == 0) return SQ_OK;
  if (g_gemm_mode != 0) {
    rc = gemm_a8_tc(a, lda, reinterpret_cast<const uint8_t*>(w), nullptr, K, false, alpha, M, N, K, epi, out, ldo,
                    col_scale, nullptr, 0, as_stream(stream));
    if (rc != SQ_ERR_ARG) return rc;
  }
  return gemm_a8_mma(a, lda, reinterpret_cast<const uint8_t*>(w), nullptr, K, false, alpha, M, N, K, epi, out, ldo,
                     col_scale, as_stream(stream));
}

extern "C" int sq_gemm_w4a8(const int8_t* a, int64_t lda, const uint8_t* w4, const int8_t* sg, int group,
                            const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo,
                            const float* col_scale, const int32_t* a_gsum, int64_t ld_gsum, void* stream) {
  int rc = check_gemm("sq_gemm_w4a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  SQ_REQUIRE(group % 32 == 0 && K % group == 0 && sg != nullptr, SQ_ERR_LAYOUT,
             "sq_gemm_w4a8: group (%d) must be a multiple of 32 dividing K", group);
  if (M == 0) return SQ_OK;
  if (g_gemm_mode != 0) {
    SQ_REQUIRE(!a_gsum || ld_gsum >= K / 128, SQ_ERR_LAYOUT, "sq_gemm_w4a8: ld_gsum < K/128");
    rc = gemm_a8_tc(a, lda, w4, sg, group, true, alpha, M, N, K, epi, out, ldo, col_scale, a_gsum, ld_gsum,
                    as_stream(stream));
    if (rc != SQ_ERR_ARG) return rc;
  }
  return gemm_a8_mma(a, lda, w4, sg, group, true, alpha, M, N, K, epi, out, ldo, col_scale, as_stream(stream));
}
