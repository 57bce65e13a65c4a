// Row kernels: model pre-norm + quant, gated-norm + Hadamard + quant (K6), embedding,
// argmax.  HBM-bound: one CTA per token row, the row staged once in shared memory.
//
// Parity (oracle/ssm_block.py rmsnorm, oracle/hadamard.py): the sum of squares is
// accumulated in f64 (the oracle's np.mean over f64) and every later op is the same
// IEEE f32 op in the same order, so codes match the oracle bit-for-bit except when the
// f64 sum order moves the f32 mean across a rounding boundary (≤1 step, rare).
// The FWHT runs the oracle's butterfly stages h = 1, 2, 4, … with identical f32
// a+b / a-b, so the transform itself is bit-identical.
#include <cstdlib>

#include "common.cuh"

namespace sq {

template <int NT>
__device__ __forceinline__ double block_sum_d(double v, double* red) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = (l < NT / 32) ? red[l] : 0.0;
    t = warp_sum_d(t);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ float rms_factor(double ss, int D, float eps) {
  float ms = (float)(ss / (double)D);
  return __fdiv_rn(1.0f, sqrtf(__fadd_rn(ms, eps)));
}

template <int NT, bool QUANT>
__global__ void __launch_bounds__(NT) rmsnorm_kernel(const float* x, int64_t ldx,
                                                     const float* __restrict__ gamma, float eps, float s,
                                                     int D, void* __restrict__ out, int64_t ldo) {
  __shared__ double red[NT / 32];
  pdl_trigger();
  pdl_wait();
  const float* xr = x + (int64_t)blockIdx.x * ldx;
  double ss = 0.0;
  for (int i = threadIdx.x; i < D; i += NT) {
    float v = xr[i];
    ss += (double)v * (double)v;
  }
  ss = block_sum_d<NT>(ss, red);
  const float r = rms_factor(ss, D, eps);
  for (int i = threadIdx.x; i < D; i += NT) {
    float v = __fmul_rn(__fmul_rn(xr[i], r), gamma[i]);
    if (QUANT)
      reinterpret_cast<int8_t*>(out)[(int64_t)blockIdx.x * ldo + i] = quant8(v, s);
    else
      reinterpret_cast<float*>(out)[(int64_t)blockIdx.x * ldo + i] = v;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) gate_norm_had_quant_kernel(const float* __restrict__ y, int64_t ldy,
                                                                 const float* __restrict__ gamma, float eps,
                                                                 float s_y, int had_block, int D,
                                                                 int8_t* __restrict__ out, int64_t ldo) {
  extern __shared__ float buf[];
  __shared__ double red[NT / 32];
  const float* yr = y + (int64_t)blockIdx.x * ldy;
  double ss = 0.0;
  for (int i = threadIdx.x * 4; i < D; i += NT * 4) {
    float4 v = *reinterpret_cast<const float4*>(yr + i);
    *reinterpret_cast<float4*>(buf + i) = v;
    ss += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
  ss = block_sum_d<NT>(ss, red);
  const float r = rms_factor(ss, D, eps);
  for (int i = threadIdx.x; i < D; i += NT) buf[i] = __fmul_rn(__fmul_rn(buf[i], r), gamma[i]);
  __syncthreads();
  // Sylvester butterflies within each power-of-two block (LEDGER G9).
  for (int h = 1; h < had_block; h <<= 1) {
    for (int idx = threadIdx.x; idx < D / 2; idx += NT) {
      const int i = (idx / h) * 2 * h + (idx % h);
      const float a = buf[i], b = buf[i + h];
      buf[i] = __fadd_rn(a, b);
      buf[i + h] = __fsub_rn(a, b);
    }
    __syncthreads();
  }
  int8_t* o = out + (int64_t)blockIdx.x * ldo;
  for (int i = threadIdx.x * 4; i < D; i += NT * 4) {
    char4 q;
    q.x = quant8(buf[i], s_y);
    q.y = quant8(buf[i + 1], s_y);
    q.z = quant8(buf[i + 2], s_y);
    q.w = quant8(buf[i + 3], s_y);
    *reinterpret_cast<char4*>(o + i) = q;
  }
}

// ---- register-resident variants: one thread per 16 contiguous elements (D/16 threads) ----
// Block sum with one barrier: every thread adds the per-warp partials in warp order (a fixed,
// deterministic order).  Callers alternate `red` between two buffers on consecutive rows.
__device__ __forceinline__ double block_sum_dyn(double v, double* red) {
  v = warp_sum_d(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

__device__ __forceinline__ void load16(const float* p, float (&v)[16]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float4 f = *reinterpret_cast<const float4*>(p + e * 4);
    v[e * 4] = f.x; v[e * 4 + 1] = f.y; v[e * 4 + 2] = f.z; v[e * 4 + 3] = f.w;
  }
}

// 16 codes packed little-endian into 4 words: division-free quantizer, and the exact
// quant8 only when some value sits within 1e-4 of a rounding tie (bit-identical codes).
__device__ __forceinline__ void quant16(const float (&v)[16], float s, uint32_t (&w)[4]) {
  const float is = __frcp_rn(s);
  const float2 is2 = make_float2(is, is);
  bool tie = false;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    w[e] = quant8x4_fast(make_float2(v[e * 4], v[e * 4 + 1]), make_float2(v[e * 4 + 2], v[e * 4 + 3]), is2, is2, tie);
  if (tie) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      w[e] = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) w[e] |= (uint32_t)(uint8_t)quant8(v[e * 4 + k], s) << (8 * k);
    }
  }
}

__device__ __forceinline__ void store16_q(int8_t* p, const float (&v)[16], float s) {
  uint32_t w[4];
  quant16(v, s, w);
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

// Row loops: a CTA walks rows blockIdx.x, blockIdx.x + gridDim.x, … and loads the next row
// into registers before working on the current one, so HBM latency overlaps the reduction
// and transform; the reduction scratch alternates between two buffers per row.
template <bool QUANT>
__global__ void __launch_bounds__(512) rmsnorm16_kernel(const float* x, int64_t ldx,
                                                         const float* __restrict__ gamma, float eps, float s, int D,
                                                         int M, void* __restrict__ out, int64_t ldo,
                                                         int32_t* __restrict__ gsum, int64_t ldg) {
  __shared__ double red[2][32];
  const int base = threadIdx.x * 16;
  float v[16], g[16];
  pdl_trigger();
  load16(gamma + base, g);
  pdl_wait();
  int row = blockIdx.x;
  load16(x + (int64_t)row * ldx + base, v);
  for (int it = 0; row < M; row += gridDim.x, ++it) {
    float vn[16];
    const int nrow = row + gridDim.x;
    if (nrow < M) load16(x + (int64_t)nrow * ldx + base, vn);
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) ss += (double)v[i] * (double)v[i];
    ss = block_sum_dyn(ss, red[it & 1]);
    const float r = rms_factor(ss, D, eps);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __fmul_rn(__fmul_rn(v[i], r), g[i]);
    if (QUANT) {
      uint32_t w[4];
      quant16(v, s, w);
      *reinterpret_cast<uint4*>(reinterpret_cast<int8_t*>(out) + (int64_t)row * ldo + base) =
          make_uint4(w[0], w[1], w[2], w[3]);
      if (gsum) {   // sums of the codes over each 128-wide block (8 threads)
        int cs = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) cs = __dp4a((int)w[e], 0x01010101, cs);
        cs += __shfl_xor_sync(0xffffffffu, cs, 1);
        cs += __shfl_xor_sync(0xffffffffu, cs, 2);
        cs += __shfl_xor_sync(0xffffffffu, cs, 4);
        if ((threadIdx.x & 7) == 0) gsum[(int64_t)row * ldg + (base >> 7)] = cs;
      }
    } else {
      float* o = reinterpret_cast<float*>(out) + (int64_t)row * ldo + base;
#pragma unroll
      for (int e = 0; e < 4; ++e) *reinterpret_cast<float4*>(o + e * 4) = make_float4(v[e * 4], v[e * 4 + 1], v[e * 4 + 2], v[e * 4 + 3]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = vn[i];
  }
}

// Gated-norm + blocked Sylvester FWHT + quant with the row in registers: stages h < 16
// inside a thread, 16 <= h < 512 across lanes (shfl_xor), h >= 512 through smem.
// Every butterfly is the oracle's f32 a+b / a-b, in the oracle's stage order.
__global__ void __launch_bounds__(512) gate_norm_had_quant16_kernel(const float* __restrict__ y, int64_t ldy,
                                                                     const float* __restrict__ gamma, float eps,
                                                                     float s_y, int blk, int D, int M,
                                                                     int8_t* __restrict__ out, int64_t ldo) {
  extern __shared__ float buf[];
  __shared__ double red[2][32];
  const int base = threadIdx.x * 16;
  const int lane = threadIdx.x & 31;
  float v[16];
  int row = blockIdx.x;
  load16(y + (int64_t)row * ldy + base, v);
  int stage = 0;   // partner-stage counter: the exchange buffer alternates halves
  for (int it = 0; row < M; row += gridDim.x, ++it) {
    float vn[16];
    const int nrow = row + gridDim.x;
    if (nrow < M) load16(y + (int64_t)nrow * ldy + base, vn);
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) ss += (double)v[i] * (double)v[i];
    ss = block_sum_dyn(ss, red[it & 1]);
    const float r = rms_factor(ss, D, eps);
    {
      float g[16];
      load16(gamma + base, g);
      const float2 r2 = make_float2(r, r);
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 t = __fmul2_rn(__fmul2_rn(make_float2(v[i], v[i + 1]), r2), make_float2(g[i], g[i + 1]));
        v[i] = t.x;
        v[i + 1] = t.y;
      }
    }
    // in-thread stages: h = 1 scalar; h >= 2 as packed pairs (a - b as fma(b, -1, a))
    if (blk > 1) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float a = v[i], b = v[i + 1];
        v[i] = __fadd_rn(a, b);
        v[i + 1] = __fsub_rn(a, b);
      }
    }
#pragma unroll
    for (int h = 2; h < 16; h <<= 1) {
      if (h < blk) {
        const float2 M1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          if ((i & h) == 0) {
            const float2 a = make_float2(v[i], v[i + 1]), b = make_float2(v[i + h], v[i + h + 1]);
            const float2 sm = __fadd2_rn(a, b), df = __ffma2_rn(b, M1, a);
            v[i] = sm.x; v[i + 1] = sm.y; v[i + h] = df.x; v[i + h + 1] = df.y;
          }
        }
      }
    }
    // cross-thread stages: the lower element gets a + b, the upper b' - a' — one FMA with
    // sign ±1 (fma(-1, v, o) = RN(o - v), fma(1, v, o) = RN(v + o): the same rounding),
    // two elements per packed FMA
    for (int m = 1; m < 32 && 16 * m < blk; m <<= 1) {
      const float sg = (lane & m) ? -1.f : 1.f;
      const float2 sg2 = make_float2(sg, sg);
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v[i], m), __shfl_xor_sync(0xffffffffu, v[i + 1], m));
        const float2 t = __ffma2_rn(sg2, make_float2(v[i], v[i + 1]), o);
        v[i] = t.x;
        v[i + 1] = t.y;
      }
    }
    // stages h >= 512 pair thread t with thread t ^ (h / 16) through shared memory
    // (two exchange buffers: a stage's writes go to the half the previous stage did not read,
    //  whose readers all passed that stage's barrier, so one barrier per stage suffices)
    for (int m = 32; 16 * m < blk; m <<= 1, ++stage) {
      float* xb = buf + (stage & 1) * D;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        *reinterpret_cast<float4*>(xb + base + e * 4) = make_float4(v[e * 4], v[e * 4 + 1], v[e * 4 + 2], v[e * 4 + 3]);
      __syncthreads();
      const float sg = (threadIdx.x & m) ? -1.f : 1.f;
      const float2 sg2 = make_float2(sg, sg);
      const float* o = xb + (int)((threadIdx.x ^ m) * 16);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float4 f = *reinterpret_cast<const float4*>(o + e * 4);
        const float2 t0 = __ffma2_rn(sg2, make_float2(v[e * 4], v[e * 4 + 1]), make_float2(f.x, f.y));
        const float2 t1 = __ffma2_rn(sg2, make_float2(v[e * 4 + 2], v[e * 4 + 3]), make_float2(f.z, f.w));
        v[e * 4] = t0.x; v[e * 4 + 1] = t0.y; v[e * 4 + 2] = t1.x; v[e * 4 + 3] = t1.y;
      }
    }
    store16_q(out + (int64_t)row * ldo + base, v, s_y);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = vn[i];
  }
}

// Gated-norm + I_q ⊗ H_1024 + quant (D = q·1024: Mamba2-2.7B / Mamba1-2.8B d_inner 5120, G9).
// One warp per 1024-point Hadamard block, one CTA (D/1024 warps) per row in a row loop with
// the next row prefetched.  Global loads and stores are fully coalesced (lane l moves the
// 16 B at l·16 of every 512 B); a per-warp shared tile of 32 rows × 36 floats (conflict-free
// for both float4 row access and scalar column access) redistributes the block so that lane l
// first holds elements l·32 + i (stages h = 1..16 in registers), then elements i·32 + l (stages
// h = 32..512 in registers).  No shuffles; the only CTA barrier is the row's Σy².
// Same f32 butterflies in the oracle's stage order as gate_norm_had_quant16_kernel.
constexpr int N1K_LD = 36;                       // tile row stride (floats)
constexpr int N1K_WARP_FLOATS = 2 * 32 * N1K_LD + 256;   // data tile, γ tile, 1 KB of codes

__device__ __forceinline__ int n1k_off(int p) { return (p >> 5) * N1K_LD + (p & 31); }   // element p -> tile

// Sylvester stages h = 1..16 over 32 registers (element bits 0..4 = register index), the oracle's
// stage order: h = 1 scalar (its pairs are adjacent registers), h >= 2 on packed f32x2 pairs
// (v[i], v[i+1]) vs (v[i+h], v[i+h+1]); a - b as fma(b, -1, a) rounds like the subtraction.
__device__ __forceinline__ void had32_regs(float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    const float a = v[i], b = v[i + 1];
    v[i] = __fadd_rn(a, b);
    v[i + 1] = __fsub_rn(a, b);
  }
  const float2 M1 = make_float2(-1.f, -1.f);
#pragma unroll
  for (int h = 2; h < 32; h <<= 1) {
#pragma unroll
    for (int i = 0; i < 32; i += 2)
      if ((i & h) == 0) {
        const float2 a = make_float2(v[i], v[i + 1]), b = make_float2(v[i + h], v[i + h + 1]);
        const float2 sm = __fadd2_rn(a, b), df = __ffma2_rn(b, M1, a);
        v[i] = sm.x; v[i + 1] = sm.y; v[i + h] = df.x; v[i + h + 1] = df.y;
      }
  }
}

__global__ void __launch_bounds__(512) gate_norm_had1k_kernel(const float* y, int64_t ldy,
                                                               const float* __restrict__ gamma, float eps, float s_y,
                                                               int D, int M, int8_t* out, int64_t ldo) {
  extern __shared__ float tsm[];
  __shared__ double red[2][16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float* s = tsm + warp * N1K_WARP_FLOATS;
  float* gs = s + 32 * N1K_LD;
  uint8_t* qb = reinterpret_cast<uint8_t*>(gs + 32 * N1K_LD);
  const int blk0 = warp * 1024;
  pdl_trigger();
  // γ of this block, once, in the tile layout (a weight: read before the grid dependency wait)
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int p = e * 128 + lane * 4;
    *reinterpret_cast<float4*>(gs + n1k_off(p)) = __ldg(reinterpret_cast<const float4*>(gamma + blk0 + p));
  }
  pdl_wait();   // y comes from the previous grid (launched with PDL_SMALL)
  float4 cur[8];
  int row = blockIdx.x;
#pragma unroll
  for (int e = 0; e < 8; ++e) cur[e] = *reinterpret_cast<const float4*>(y + (int64_t)row * ldy + blk0 + e * 128 + lane * 4);
  for (int it = 0; row < M; row += gridDim.x, ++it) {
    // coalesced rows -> tile
#pragma unroll
    for (int e = 0; e < 8; ++e) *reinterpret_cast<float4*>(s + n1k_off(e * 128 + lane * 4)) = cur[e];
    const int nrow = row + gridDim.x;
    if (nrow < M) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        cur[e] = *reinterpret_cast<const float4*>(y + (int64_t)nrow * ldy + blk0 + e * 128 + lane * 4);
    }
    __syncwarp();
    float v[32];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 f = *reinterpret_cast<const float4*>(s + lane * N1K_LD + k * 4);
      v[k * 4] = f.x; v[k * 4 + 1] = f.y; v[k * 4 + 2] = f.z; v[k * 4 + 3] = f.w;
    }
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) ss += (double)v[i] * (double)v[i];
    ss = warp_sum_d(ss);
    if (lane == 0) red[it & 1][warp] = ss;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < nw; ++w) tot += red[it & 1][w];   // fixed warp order: deterministic
    const float r = rms_factor(tot, D, eps);
    const float2 r2 = make_float2(r, r);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 g = *reinterpret_cast<const float4*>(gs + lane * N1K_LD + k * 4);
      const float2 t0 = __fmul2_rn(__fmul2_rn(make_float2(v[k * 4], v[k * 4 + 1]), r2), make_float2(g.x, g.y));
      const float2 t1 = __fmul2_rn(__fmul2_rn(make_float2(v[k * 4 + 2], v[k * 4 + 3]), r2), make_float2(g.z, g.w));
      v[k * 4] = t0.x; v[k * 4 + 1] = t0.y; v[k * 4 + 2] = t1.x; v[k * 4 + 3] = t1.y;
    }
    // stages h = 1..16 (element bits 0..4 = register index)
    had32_regs(v);
    __syncwarp();   // every lane has read its row of the tile
#pragma unroll
    for (int k = 0; k < 8; ++k)
      *reinterpret_cast<float4*>(s + lane * N1K_LD + k * 4) = make_float4(v[k * 4], v[k * 4 + 1], v[k * 4 + 2], v[k * 4 + 3]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = s[i * N1K_LD + lane];   // lane l: elements i·32 + l
    // stages h = 32..512 (element bits 5..9 = register index)
    had32_regs(v);
    const float is = __frcp_rn(s_y);
    const float2 is2 = make_float2(is, is);
    bool tie = false;
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      w[e] = quant8x4_fast(make_float2(v[e * 4], v[e * 4 + 1]), make_float2(v[e * 4 + 2], v[e * 4 + 3]), is2, is2, tie);
    if (tie) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        w[e] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) w[e] |= (uint32_t)(uint8_t)quant8(v[e * 4 + k], s_y) << (8 * k);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) qb[i * 32 + lane] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
    __syncwarp();
    int8_t* o = out + (int64_t)row * ldo + blk0;
    *reinterpret_cast<uint4*>(o + lane * 16) = *reinterpret_cast<const uint4*>(qb + lane * 16);
    *reinterpret_cast<uint4*>(o + 512 + lane * 16) = *reinterpret_cast<const uint4*>(qb + 512 + lane * 16);
    // the next row's first tile write follows these reads in program order of every lane
    // only after the __syncwarp below
    __syncwarp();
  }
}

// CTAs for a row loop: every resident slot, but never more CTAs than rows.
template <typename K>
static int row_grid(K kern, int threads, size_t smem, int M) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  return max(1, min(M, sms * max(per_sm, 1)));
}

__global__ void quantize_kernel(const float* x, int64_t ldx, float s, int D, int8_t* __restrict__ out,
                                int64_t ldo) {
  pdl_trigger();
  pdl_wait();
  const float* r = x + (int64_t)blockIdx.x * ldx;
  int8_t* o = out + (int64_t)blockIdx.x * ldo;
  for (int i = threadIdx.x; i < D; i += blockDim.x) o[i] = quant8(r[i], s);
}

__global__ void embed_kernel(const int8_t* __restrict__ codes, const float* __restrict__ rs,
                             const int32_t* tok, int D, float* __restrict__ h) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int t = tok[m];
  const float s = rs[t];
  for (int i = threadIdx.x; i < D; i += blockDim.x)
    h[(int64_t)m * D + i] = __fmul_rn((float)codes[(int64_t)t * D + i], s);
}

// 4-bit embedding rows (head-to-toe quantization): u4packed [V x D/2] (low
// nibble = even index), h[m, d] = v(tok[m], d) * row_scale[tok[m]].
__global__ void embed_u4_kernel(const uint8_t* __restrict__ packed, const float* __restrict__ rs,
                                const int32_t* tok, int D, float* __restrict__ h) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int t = tok[m];
  const float s = rs[t];
  const uint8_t* row = packed + (int64_t)t * (D / 2);
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const uint32_t b = row[i];
    const int lo = ((int)(b << 28)) >> 28, hi = ((int)(b << 24)) >> 28;
    *reinterpret_cast<float2*>(h + (int64_t)m * D + 2 * i) = make_float2(__fmul_rn((float)lo, s), __fmul_rn((float)hi, s));
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) argmax_kernel(const float* lg, int64_t ld, int N,
                                                    int32_t* __restrict__ tok) {
  __shared__ float bv[NT / 32];
  __shared__ int bi[NT / 32];
  pdl_trigger();
  pdl_wait();
  const float* r = lg + (int64_t)blockIdx.x * ld;
  float best = -INFINITY;
  int bidx = 0x7fffffff;
  for (int i = threadIdx.x; i < N; i += NT) {
    float v = r[i];
    if (v > best) { best = v; bidx = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { bv[w] = best; bi[w] = bidx; }
  __syncthreads();
  if (w == 0) {
    best = l < NT / 32 ? bv[l] : -INFINITY;
    bidx = l < NT / 32 ? bi[l] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      float ov = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    if (l == 0) tok[blockIdx.x] = bidx;
  }
}

}  // namespace sq

using namespace sq;

namespace sq {
__global__ void group_sum_kernel(const int8_t* codes, int64_t ld, int K, int32_t* __restrict__ gsum,
                                 int64_t ldg) {
  // one warp per 128-wide block: 32 lanes x 4 codes
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.y;
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= K / 128) return;
  const int lane = threadIdx.x & 31;
  int acc = __dp4a(*reinterpret_cast<const int*>(codes + (int64_t)m * ld + g * 128 + lane * 4), 0x01010101, 0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) gsum[(int64_t)m * ldg + g] = acc;
}

int launch_group_sum(const int8_t* codes, int64_t ld, int M, int K, int32_t* gsum, int64_t ldg, cudaStream_t st) {
  SQ_REQUIRE(K % 128 == 0 && ld % 4 == 0, SQ_ERR_SHAPE, "group sums need K %% 128 == 0 and 4-byte aligned rows");
  if (M == 0) return SQ_OK;
  launch_k(PDL_ROW, group_sum_kernel, dim3((K / 128 + 7) / 8, M), dim3(256), 0, st, codes, ld, K, gsum, ldg);
  return check_launch("group_sum");
}
}  // namespace sq

extern "C" int sq_rmsnorm_quant(const float* x, int64_t ldx, const float* gamma, float eps, float s, int M,
                                int D, int8_t* out, int64_t ldo, int32_t* gsum, int64_t ldg, void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0 && s > 0.f, SQ_ERR_SHAPE, "sq_rmsnorm_quant: bad M/D/s");
  SQ_REQUIRE(!gsum || (D % 128 == 0 && ldg >= D / 128), SQ_ERR_SHAPE, "sq_rmsnorm_quant: gsum needs D %% 128 == 0");
  if (M == 0) return SQ_OK;
  if (D % 512 == 0 && D / 16 <= 512 && ldx % 4 == 0 && ldo % 16 == 0) {
    launch_k(PDL_ROW, rmsnorm16_kernel<true>, dim3(row_grid(rmsnorm16_kernel<true>, D / 16, 0, M)), dim3(D / 16), 0,
             as_stream(stream), x, ldx, gamma, eps, s, D, M, (void*)out, ldo, gsum, ldg);
  } else {
    launch_k(PDL_ROW, rmsnorm_kernel<256, true>, dim3(M), dim3(256), 0, as_stream(stream), x, ldx, gamma, eps, s, D,
             (void*)out, ldo);
    if (gsum) return launch_group_sum(out, ldo, M, D, gsum, ldg, as_stream(stream));
  }
  return check_launch("sq_rmsnorm_quant");
}

extern "C" int sq_rmsnorm_f32(const float* x, int64_t ldx, const float* gamma, float eps, int M, int D,
                              float* out, int64_t ldo, void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0, SQ_ERR_SHAPE, "sq_rmsnorm_f32: bad M/D");
  if (M == 0) return SQ_OK;
  if (D % 512 == 0 && D / 16 <= 512 && ldx % 4 == 0 && ldo % 4 == 0)
    launch_k(PDL_ROW, rmsnorm16_kernel<false>, dim3(row_grid(rmsnorm16_kernel<false>, D / 16, 0, M)), dim3(D / 16), 0,
             as_stream(stream), x, ldx, gamma, eps, 1.f, D, M, (void*)out, ldo, (int32_t*)nullptr, (int64_t)0);
  else
    launch_k(PDL_ROW, rmsnorm_kernel<256, false>, dim3(M), dim3(256), 0, as_stream(stream), x, ldx, gamma, eps, 1.f, D,
             (void*)out, ldo);
  return check_launch("sq_rmsnorm_f32");
}


extern "C" int sq_gate_norm_had_quant(const float* y, int64_t ldy, const float* gamma, float eps, float s_y,
                                      int hadamard, int M, int D, int8_t* out, int64_t ldo, void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0 && D % 4 == 0 && D <= 16384 && ldy % 4 == 0 && ldo % 4 == 0, SQ_ERR_SHAPE,
             "sq_gate_norm_had_quant: D must be a multiple of 4 and <= 16384 (D=%d)", D);
  SQ_REQUIRE(s_y > 0.f, SQ_ERR_ARG, "sq_gate_norm_had_quant: s_y must be > 0");
  if (M == 0) return SQ_OK;
  const int blk = hadamard ? (D & -D) : 1;
  const size_t smem = (size_t)D * sizeof(float);
  if (blk == 1024 && D / 1024 <= 16 && ldy % 4 == 0 && ldo % 16 == 0) {
    auto k1 = gate_norm_had1k_kernel;
    const int nthr = D / 32;
    const size_t sm1 = (size_t)(D / 1024) * N1K_WARP_FLOATS * sizeof(float);
    if (sm1 > 48 * 1024) cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    launch_k(PDL_SMALL8, k1, dim3(row_grid(k1, nthr, sm1, M)), dim3(nthr), sm1, as_stream(stream), y, ldy, gamma, eps, s_y,
             D, M, out, ldo);
    return check_launch("sq_gate_norm_had_quant");
  }
  if (D % 512 == 0 && D / 16 <= 512 && ldy % 4 == 0 && ldo % 16 == 0) {
    auto k16 = gate_norm_had_quant16_kernel;
    const size_t sm16 = blk > 512 ? 2 * smem : 0;
    if (sm16 > 48 * 1024) cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm16);
    k16<<<row_grid(k16, D / 16, sm16, M), D / 16, sm16, as_stream(stream)>>>(y, ldy, gamma, eps, s_y, blk, D, M, out,
                                                                             ldo);
    return check_launch("sq_gate_norm_had_quant");
  }
  auto k = gate_norm_had_quant_kernel<512>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<M, 512, smem, as_stream(stream)>>>(y, ldy, gamma, eps, s_y, blk, D, out, ldo);
  return check_launch("sq_gate_norm_had_quant");
}

extern "C" int sq_quantize_f32(const float* x, int64_t ldx, float s, int M, int D, int8_t* out, int64_t ldo,
                               void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0 && s > 0.f, SQ_ERR_SHAPE, "sq_quantize_f32: bad shape/scale");
  if (M == 0) return SQ_OK;
  launch_k(PDL_ROW, quantize_kernel, dim3(M), dim3(256), 0, as_stream(stream), x, ldx, s, D, out, ldo);
  return check_launch("sq_quantize_f32");
}

extern "C" int sq_embed_int8(const int8_t* codes, const float* row_scale, const int32_t* tok, int M, int D,
                             float* h, void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0, SQ_ERR_SHAPE, "sq_embed_int8: bad shape");
  if (M == 0) return SQ_OK;
  launch_k(PDL_ROW, embed_kernel, dim3(M), dim3(256), 0, as_stream(stream), codes, row_scale, tok, D, h);
  return check_launch("sq_embed_int8");
}

extern "C" int sq_embed_u4(const uint8_t* packed, const float* row_scale, const int32_t* tok, int M, int D,
                           float* h, void* stream) {
  SQ_REQUIRE(M >= 0 && D > 0 && D % 2 == 0, SQ_ERR_SHAPE, "sq_embed_u4: D must be even");
  SQ_REQUIRE((reinterpret_cast<uintptr_t>(h) & 7) == 0, SQ_ERR_LAYOUT, "sq_embed_u4: h must be 8-B aligned");
  if (M == 0) return SQ_OK;
  launch_k(PDL_ROW, embed_u4_kernel, dim3(M), dim3(256), 0, as_stream(stream), packed, row_scale, tok, D, h);
  return check_launch("sq_embed_u4");
}

extern "C" int sq_argmax_f32(const float* logits, int64_t ld, int M, int N, int32_t* tok, void* stream) {
  SQ_REQUIRE(M >= 0 && N > 0, SQ_ERR_SHAPE, "sq_argmax_f32: bad shape");
  if (M == 0) return SQ_OK;
  launch_k(PDL_ROW, argmax_kernel<1024>, dim3(M), dim3(1024), 0, as_stream(stream), logits, ld, N, tok);
  return check_launch("sq_argmax_f32");
}
