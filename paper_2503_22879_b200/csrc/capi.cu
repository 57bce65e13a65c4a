// C-ABI plumbing: version, thread-local last error, device check.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace sq {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SQ_ERR_CUDA;
  }
  return SQ_OK;
}

// Kernel classes launched with programmatic dependent launch: a build-time choice
// (-DSQ_PDL_MASK=m for A/B builds); default GEMMs, decode prep, state ring, the b=1 f32 chain and
// the b=1 int8 chain (the latter since its kernels load their parameters before the dependency
// wait: Mamba1-2.8B decode 431 -> 443 tok/s same-box, where it had been slower without that).
#ifndef SQ_PDL_MASK
#define SQ_PDL_MASK 118
#endif
bool pdl_enabled(int cls) { return (SQ_PDL_MASK & cls) != 0; }

}  // namespace sq

extern "C" int sq_abi_version(void) { return SQ_ABI_VERSION; }

extern "C" const char* sq_last_error(void) { return sq::g_err; }

extern "C" int sq_device_supported(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
  return p.major == 10 && p.minor == 0;
}
