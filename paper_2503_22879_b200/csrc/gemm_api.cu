// C-ABI entry points for the A8 projections (K1/K2) and the int4 weight layout.
#include "common.cuh"

namespace sq {
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

extern "C" int64_t sq_w4_bytes(int N, int K) { return (int64_t)N * K / 2; }

// Layout v1: row-major u4packed (identity).  Kept behind the repack API so the kernel
// layout can change without touching callers; sq_unpack_w4 proves the round trip.
extern "C" int sq_repack_w4(const uint8_t* u4packed, int N, int K, uint8_t* dst, void* stream) {
  SQ_REQUIRE(N > 0 && K > 0 && K % 32 == 0, SQ_ERR_SHAPE, "sq_repack_w4: K must be a multiple of 32");
  cudaError_t e = cudaMemcpyAsync(dst, u4packed, (size_t)N * K / 2, cudaMemcpyDeviceToDevice, as_stream(stream));
  SQ_REQUIRE(e == cudaSuccess, SQ_ERR_CUDA, "sq_repack_w4: %s", cudaGetErrorString(e));
  return SQ_OK;
}

extern "C" int sq_unpack_w4(const uint8_t* src, int N, int K, uint8_t* u4packed, void* stream) {
  SQ_REQUIRE(N > 0 && K > 0 && K % 32 == 0, SQ_ERR_SHAPE, "sq_unpack_w4: K must be a multiple of 32");
  cudaError_t e = cudaMemcpyAsync(u4packed, src, (size_t)N * K / 2, cudaMemcpyDeviceToDevice, as_stream(stream));
  SQ_REQUIRE(e == cudaSuccess, SQ_ERR_CUDA, "sq_unpack_w4: %s", cudaGetErrorString(e));
  return SQ_OK;
}

extern "C" int sq_gemm_w8a8(const int8_t* a, int64_t lda, const int8_t* w, const float* alpha, int M, int N, int K,
                            int epi, void* out, int64_t ldo, const float* col_scale, void* stream) {
  int rc = check_gemm("sq_gemm_w8a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  if (M == 0) return SQ_OK;
  return gemm_a8_mma(a, lda, reinterpret_cast<const uint8_t*>(w), nullptr, K, false, alpha, M, N, K, epi, out, ldo,
                     col_scale, as_stream(stream));
}

extern "C" int sq_gemm_w4a8(const int8_t* a, int64_t lda, const uint8_t* w4, const int8_t* sg, int group,
                            const float* alpha, int M, int N, int K, int epi, void* out, int64_t ldo,
                            const float* col_scale, void* stream) {
  int rc = check_gemm("sq_gemm_w4a8", a, lda, M, N, K, epi, ldo, col_scale);
  if (rc) return rc;
  SQ_REQUIRE(group % 32 == 0 && K % group == 0 && sg != nullptr, SQ_ERR_LAYOUT,
             "sq_gemm_w4a8: group (%d) must be a multiple of 32 dividing K", group);
  if (M == 0) return SQ_OK;
  return gemm_a8_mma(a, lda, w4, sg, group, true, alpha, M, N, K, epi, out, ldo, col_scale, as_stream(stream));
}
