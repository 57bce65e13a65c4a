// C-ABI entry points for the A8 projections (K1/K2) and the int4 weight layout.
#include "common.cuh"

namespace sq {
int gemm_a8_tc(const int8_t* a, int64_t lda, const uint8_t* w, const float* alpha, int M, int N, int K, int epi,
               void* out, int64_t ldo, const float* col_scale, cudaStream_t st);
int gemm_w4a8_tc(const int8_t* a, int64_t lda, const uint8_t* w4, const float* ws, float s_a, int M, int N, int K,
                 int epi, void* out, int64_t ldo, const float* col_scale, cudaStream_t st);
int w4a8_splits(int M, int N, int K);
int tile_scales(const float* s, int N, int G, float* dst, cudaStream_t st);
int64_t w4_layout_bytes(int N, int K);
int repack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st);
int unpack_w4(const uint8_t* src, int N, int K, uint8_t* dst, cudaStream_t st);
int gemm_a8_mma(const int8_t* a, int64_t lda, const uint8_t* w, const float* ws, int group, float s_a, bool w4,
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

extern "C" int64_t sq_group_scale_elems(int N, int G) { return (int64_t)((N + 127) / 128) * 128 * G; }

extern "C" int sq_tile_group_scales(const float* s_group, int N, int G, float* dst, void* stream) {
  SQ_REQUIRE(N > 0 && G > 0, SQ_ERR_SHAPE, "sq_tile_group_scales: bad N/G (%d,%d)", N, G);
  return tile_scales(s_group, N, G, dst, as_stream(stream));
}

extern "C" int sq_gemm_w4a8_splits(int M, int N, int K) { return w4a8_splits(M, N, K); }

extern "C" int sq_gemm_w8a8(const int8_t* a, int64_t lda, const int8_t* w, const float* alpha, int M, int N, int K,
                            int epi, void* out, int64_t ldo, const float* col_scale, void* stream) {
  int rc = check_gemm("sq_gemm_w8a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  if (M == 0) return SQ_OK;
  rc = gemm_a8_tc(a, lda, reinterpret_cast<const uint8_t*>(w), alpha, M, N, K, epi, out, ldo, col_scale,
                  as_stream(stream));
  if (rc != SQ_ERR_ARG) return rc;
  return gemm_a8_mma(a, lda, reinterpret_cast<const uint8_t*>(w), nullptr, K, 1.f, false, alpha, M, N, K, epi, out,
                     ldo, col_scale, as_stream(stream));
}

extern "C" int sq_gemm_w4a8(const int8_t* a, int64_t lda, const uint8_t* w4, const float* w_scale, int group,
                            float s_a, int M, int N, int K, int epi, void* out, int64_t ldo, const float* col_scale,
                            void* stream) {
  int rc = check_gemm("sq_gemm_w4a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  SQ_REQUIRE(epi != SQ_EPI_I32, SQ_ERR_ARG, "sq_gemm_w4a8: per-group scales have no single int32 accumulator");
  SQ_REQUIRE(group % 32 == 0 && K % group == 0 && w_scale != nullptr, SQ_ERR_LAYOUT,
             "sq_gemm_w4a8: group (%d) must be a multiple of 32 dividing K", group);
  SQ_REQUIRE(s_a > 0.f, SQ_ERR_ARG, "sq_gemm_w4a8: s_a must be > 0");
  if (M == 0) return SQ_OK;
  if (group == 128) {
    rc = gemm_w4a8_tc(a, lda, w4, w_scale, s_a, M, N, K, epi, out, ldo, col_scale, as_stream(stream));
    if (rc != SQ_ERR_ARG) return rc;
  }
  return gemm_a8_mma(a, lda, w4, w_scale, group, s_a, true, nullptr, M, N, K, epi, out, ldo, col_scale,
                     as_stream(stream));
}
