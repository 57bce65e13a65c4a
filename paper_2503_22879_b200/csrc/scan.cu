// K7/K8/K9 sequential-recurrence kernels (reference semantics: Eq. 2,
// SPEC.md:340-341 int8 cached state):
//   * sq_state_update_int8  — Mamba2 decode step (T=1); HBM-bound on the int8 state
//   * sq_ssd_scan_int8      — Mamba2 prefill, token-sequential over T (the fp32 state
//                             lives in registers for the whole sequence)
//   * sq_ssd_scan_f32       — W4A16 float path (fp32 state)
//   * sq_selective_scan_int8 — Mamba1 (state [d_inner x N], N=16)
//
// Mamba2 mapping: one CTA per (sequence, head); thread t owns state row p = t / TPR and a
// contiguous run of NPT = N / TPR state columns, so the int8 state row is read and written
// with 16-byte vector accesses, fully coalesced per warp (K9: "vectorised, coalesced").
// Per token:  Δ = softplus(f32(Δq)·sΔ + dt_bias[h]);  Ȧ = exp(Δ·A[h]);
//   h[p,n] = Ȧ·h[p,n] + (Δ·x̂[p])·B̂[n]   (unfused f32, oracle order)
//   y[p]   = Σ_n h[p,n]·Ĉ[n] + D[h]·x̂[p];  y ← y·silu(ẑ[p])
// The cached state is requantised once per call: q = rint(h / s_h[h,p]).
#include <cstdlib>

#include "common.cuh"

namespace sq {

template <typename TQ>
struct Deq;
template <>
struct Deq<int8_t> {
  __device__ static float f(int8_t q, float s) { return __fmul_rn((float)q, s); }
};
template <>
struct Deq<float> {
  __device__ static float f(float q, float) { return q; }
};

template <typename TQ, int NPT>
__device__ __forceinline__ void load_vec(const TQ* p, float s, float* out) {
  if constexpr (sizeof(TQ) == 1) {
#pragma unroll
    for (int i = 0; i < NPT; i += 16) {
      int4 v = *reinterpret_cast<const int4*>(p + i);
      const int8_t* b = reinterpret_cast<const int8_t*>(&v);
#pragma unroll
      for (int j = 0; j < 16; ++j) out[i + j] = __fmul_rn((float)b[j], s);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NPT; i += 4) {
      float4 v = *reinterpret_cast<const float4*>(p + i);
      out[i] = v.x; out[i + 1] = v.y; out[i + 2] = v.z; out[i + 3] = v.w;
    }
  }
}

template <typename TQ, int NPT>
__device__ __forceinline__ void store_state(TQ* p, float s, const float* h) {
  if constexpr (sizeof(TQ) == 1) {
#pragma unroll
    for (int i = 0; i < NPT; i += 16) {
      int4 v;
      int8_t* b = reinterpret_cast<int8_t*>(&v);
#pragma unroll
      for (int j = 0; j < 16; ++j) b[j] = quant8(h[i + j], s);
      *reinterpret_cast<int4*>(p + i) = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NPT; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
  }
}

template <typename TQ, int NPT>
__global__ void __launch_bounds__(256) mamba2_scan_kernel(sq_mamba2_params p, int T, const TQ* __restrict__ x,
                                                         int64_t ldx, const TQ* __restrict__ Bm,
                                                         const TQ* __restrict__ Cm, int64_t ldbc,
                                                         const TQ* __restrict__ dt, int64_t lddt,
                                                         const TQ* __restrict__ z, int64_t ldz, TQ* __restrict__ state,
                                                         int state_in, float* __restrict__ y, int64_t ldy) {
  constexpr bool Q = sizeof(TQ) == 1;
  const int h = blockIdx.x;
  const int b = blockIdx.y;
  const int P = p.head_dim, N = p.d_state;
  const int TPR = N / NPT;
  const int row = threadIdx.x / TPR;
  const int n0 = (threadIdx.x % TPR) * NPT;
  const int g = p.head_group[h];
  const int ch = h * P + row;
  const float sx = Q ? p.s_x[ch] : 1.f;
  const float sh = Q ? p.s_h[ch] : 1.f;
  const float sB = Q ? p.s_B[g] : 1.f;
  const float sC = Q ? p.s_C[g] : 1.f;
  const float A = p.A[h], Dh = p.D[h], dtb = p.dt_bias[h];
  TQ* st = state + (((int64_t)b * p.n_heads + h) * P + row) * N + n0;
  float hs[NPT];
  if (state_in) {
    load_vec<TQ, NPT>(st, sh, hs);
  } else {
#pragma unroll
    for (int i = 0; i < NPT; ++i) hs[i] = 0.f;
  }
  for (int t = 0; t < T; ++t) {
    const int64_t tok = (int64_t)b * T + t;
    const float draw = Q ? __fadd_rn(__fmul_rn((float)dt[tok * lddt + h], p.s_dt), dtb)
                         : __fadd_rn((float)dt[tok * lddt + h], dtb);
    const float delta = softplus_f(draw);
    const float dA = expf(__fmul_rn(delta, A));
    const float xh = Deq<TQ>::f(x[tok * ldx + ch], sx);
    const float dtx = __fmul_rn(delta, xh);
    float bv[NPT], cv[NPT];
    load_vec<TQ, NPT>(Bm + tok * ldbc + g * N + n0, sB, bv);
    load_vec<TQ, NPT>(Cm + tok * ldbc + g * N + n0, sC, cv);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      hs[i] = __fadd_rn(__fmul_rn(dA, hs[i]), __fmul_rn(dtx, bv[i]));
      acc = fmaf(hs[i], cv[i], acc);
    }
    for (int o = TPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x % TPR) == 0) {
      float yv = __fadd_rn(acc, __fmul_rn(Dh, xh));
      const float zv = Q ? __fmul_rn((float)z[tok * ldz + ch], p.s_z) : (float)z[tok * ldz + ch];
      y[tok * ldy + ch] = __fmul_rn(yv, silu_f(zv));
    }
  }
  store_state<TQ, NPT>(st, sh, hs);
}

// W4A16 float path, coalesced: CTA = (head, sequence, 32-row block), warp = 8 state rows,
// lane = CPL consecutive state columns, so every state load / store instruction of a warp
// moves one whole contiguous row (N·4 bytes) and B / C of the lane's columns sit in CPL
// registers for all rows.  The per-element update is mamba2_scan_kernel's (identical f32 ops,
// bit-identical state); only y's column sum runs in a different order (lane partials, then a
// warp butterfly).
// PRE: Ȧ and Δ are inputs (SPEC selective_scan(x, Ȧ, Δ, ...)) in dAp / dt, same
// layout; otherwise Δ = softplus(dt + dt_bias), Ȧ = exp(Δ·A) (discretize fused).  z may be null
// (ungated output).
template <int CPL, bool PRE>
__global__ void __launch_bounds__(128) mamba2_scan_f32_rows_kernel(sq_mamba2_params p, int T, const float* x,
                                                                   int64_t ldx, const float* Bm, const float* Cm,
                                                                   int64_t ldbc, const float* dt, const float* dAp,
                                                                   int64_t lddt, const float* z, int64_t ldz,
                                                                   float* state, int state_in, float* y, int64_t ldy) {
  pdl_trigger();
  const int h = blockIdx.x, b = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = p.head_dim, N = p.d_state;   // N == 32 * CPL
  const int r0 = blockIdx.z * 32 + warp * 8;
  if (r0 >= P) return;                        // P % 8 == 0; whole warps idle past the last row
  // parameters before the grid dependency wait (static); state and operands after it
  const int g = p.head_group[h];
  const float A = PRE ? 0.f : p.A[h], Dh = p.D[h], dtb = PRE ? 0.f : p.dt_bias[h];
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  float* st = state + (((int64_t)b * p.n_heads + h) * P + r0) * N + lane * CPL;
  float hs[8][CPL];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int i = 0; i < CPL; i += 2) {
      if (state_in) {
        const float2 v = *reinterpret_cast<const float2*>(st + r * N + i);
        hs[r][i] = v.x;
        hs[r][i + 1] = v.y;
      } else {
        hs[r][i] = hs[r][i + 1] = 0.f;
      }
    }
  for (int t = 0; t < T; ++t) {
    const int64_t tok = (int64_t)b * T + t;
    const float delta = PRE ? dt[tok * lddt + h] : softplus_f(__fadd_rn(dt[tok * lddt + h], dtb));
    const float dA = PRE ? dAp[tok * lddt + h] : expf(__fmul_rn(delta, A));
    float bv[CPL], cv[CPL], xr[8];
#pragma unroll
    for (int i = 0; i < CPL; i += 2) {
      const float2 b2 = *reinterpret_cast<const float2*>(Bm + tok * ldbc + g * N + lane * CPL + i);
      const float2 c2 = *reinterpret_cast<const float2*>(Cm + tok * ldbc + g * N + lane * CPL + i);
      bv[i] = b2.x; bv[i + 1] = b2.y;
      cv[i] = c2.x; cv[i + 1] = c2.y;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) xr[r] = x[tok * ldx + h * P + r0 + r];
    float acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const float dtx = __fmul_rn(delta, xr[r]);
      acc[r] = 0.f;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        hs[r][i] = __fadd_rn(__fmul_rn(dA, hs[r][i]), __fmul_rn(dtx, bv[i]));
        acc[r] = fmaf(hs[r][i], cv[i], acc[r]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int r = 0; r < 8; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    if (lane < 8) {
      float a = acc[0], xv = xr[0];
#pragma unroll
      for (int r = 1; r < 8; ++r)
        if (lane == r) {
          a = acc[r];
          xv = xr[r];
        }
      const float yv = __fadd_rn(a, __fmul_rn(Dh, xv));
      const int ch = h * P + r0 + lane;
      y[tok * ldy + ch] = z ? __fmul_rn(yv, silu_f(z[tok * ldz + ch])) : yv;
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int i = 0; i < CPL; i += 2)
      *reinterpret_cast<float2*>(st + r * N + i) = make_float2(hs[r][i], hs[r][i + 1]);
}

template <typename TQ>
static int launch_mamba2(const sq_mamba2_params* p, int B, int T, const TQ* x, int64_t ldx, const TQ* Bm,
                         const TQ* Cm, int64_t ldbc, const TQ* dt, int64_t lddt, const TQ* z, int64_t ldz,
                         TQ* state, int state_in, float* y, int64_t ldy, cudaStream_t st, const char* name) {
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "%s: bad args", name);
  const int P = p->head_dim, N = p->d_state;
  SQ_REQUIRE(N % 16 == 0 && N <= 256 && P >= 1, SQ_ERR_SHAPE, "%s: d_state must be a multiple of 16 <= 256", name);
  const int TPR = (N + 63) / 64;
  const int NPT = N / TPR;
  SQ_REQUIRE(P * TPR <= 256 && (TPR & (TPR - 1)) == 0 && (NPT == 16 || NPT == 32 || NPT == 64), SQ_ERR_SHAPE,
             "%s: unsupported head_dim/d_state (P=%d N=%d)", name, P, N);
  SQ_REQUIRE(p->n_groups >= 1, SQ_ERR_SHAPE, "%s: n_groups", name);   // heads map to groups via head_group
  if (B == 0 || T == 0) return SQ_OK;
  dim3 grid(p->n_heads, B), block(P * TPR);
#define SQ_M2(NPTV)                                                                                           \
  mamba2_scan_kernel<TQ, NPTV><<<grid, block, 0, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, \
                                                      state_in, y, ldy)
  if (NPT == 16) SQ_M2(16);
  else if (NPT == 32) SQ_M2(32);
  else SQ_M2(64);
#undef SQ_M2
  return check_launch(name);
}

// Mamba1: one thread per (sequence, channel); N state columns in registers.
template <int N>
__global__ void __launch_bounds__(128) mamba1_scan_kernel(sq_mamba1_params p, int B, int T, const int8_t* x,
                                                         int64_t ldx, const int8_t* dt, int64_t lddt,
                                                         const int8_t* BC, int64_t ldbc, const int8_t* z,
                                                         int64_t ldz, int8_t* state, int state_in, float* y,
                                                         int64_t ldy) {
  pdl_trigger();
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (c >= p.d_inner) return;
  const float sx = p.s_x[c], sh = p.s_h[c], Dc = p.D[c], dtb = p.dt_bias[c];
  float A[N], hs[N];
#pragma unroll
  for (int n = 0; n < N; ++n) A[n] = p.A[c * N + n];
  int8_t* st = state + ((int64_t)b * p.d_inner + c) * N;
  if (state_in) {
#pragma unroll
    for (int n = 0; n < N; ++n) hs[n] = __fmul_rn((float)st[n], sh);
  } else {
#pragma unroll
    for (int n = 0; n < N; ++n) hs[n] = 0.f;
  }
  for (int t = 0; t < T; ++t) {
    const int64_t tok = (int64_t)b * T + t;
    const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dt[tok * lddt + c], p.s_dt), dtb));
    const float xh = __fmul_rn((float)x[tok * ldx + c], sx);
    const float dtx = __fmul_rn(delta, xh);
    const int8_t* bc = BC + tok * ldbc;
    float acc = 0.f;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float dA = expf(__fmul_rn(delta, A[n]));
      const float bn = __fmul_rn((float)bc[n], p.s_B);
      const float cn = __fmul_rn((float)bc[N + n], p.s_C);
      hs[n] = __fadd_rn(__fmul_rn(dA, hs[n]), __fmul_rn(dtx, bn));
      acc = fmaf(hs[n], cn, acc);
    }
    const float yv = __fadd_rn(acc, __fmul_rn(Dc, xh));
    const float zv = __fmul_rn((float)z[tok * ldz + c], p.s_z);
    y[tok * ldy + c] = __fmul_rn(yv, silu_f(zv));
  }
#pragma unroll
  for (int n = 0; n < N; ++n) st[n] = quant8(hs[n], sh);
}

// Mamba1 int8 decode step (T = 1): thread = (sequence, channel, state), 16 threads per channel,
// so d_inner 5120 runs on 320 CTAs instead of 40 one-channel-per-thread CTAs.  Per state the
// update is mamba1_scan_kernel's (h = Ȧ·h + (Δx̂)·B̂, unfused f32, requantised with s_h); the
// channel's C·h is reduced over its 16 threads with shuffles (a different f32 summation order
// than the sequential kernel: tolerance-compared).  Parameters are read before the grid
// dependency wait.
__global__ void __launch_bounds__(256) mamba1_step_kernel(sq_mamba1_params p, int B, const int8_t* x, int64_t ldx,
                                                          const int8_t* dt, int64_t lddt, const int8_t* BC,
                                                          int64_t ldbc, const int8_t* z, int64_t ldz, int8_t* state,
                                                          int state_in, float* y, int64_t ldy) {
  constexpr int N = 16;
  pdl_trigger();
  const int n = threadIdx.x & (N - 1);
  const int c = blockIdx.x * (256 / N) + (threadIdx.x >> 4);
  const int b = blockIdx.y;
  const bool live = c < p.d_inner;
  const int cc = live ? c : 0;
  const float An = p.A[(int64_t)cc * N + n], dtb = p.dt_bias[cc], sx = p.s_x[cc], sh = p.s_h[cc], Dc = p.D[cc];
  pdl_wait();   // codes and the cached state come from earlier grids
  if (!live) return;
  const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dt[(int64_t)b * lddt + c], p.s_dt), dtb));
  const float xh = __fmul_rn((float)x[(int64_t)b * ldx + c], sx);
  const float dtx = __fmul_rn(delta, xh);
  const int8_t* bc = BC + (int64_t)b * ldbc;
  const float bn = __fmul_rn((float)bc[n], p.s_B), cn = __fmul_rn((float)bc[N + n], p.s_C);
  int8_t* st = state + ((int64_t)b * p.d_inner + c) * N + n;
  const float h0 = state_in ? __fmul_rn((float)*st, sh) : 0.f;
  const float h = __fadd_rn(__fmul_rn(expf(__fmul_rn(delta, An)), h0), __fmul_rn(dtx, bn));
  float acc = __fmul_rn(h, cn);
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  *st = quant8(h, sh);
  if (n == 0) {
    const float yv = __fadd_rn(acc, __fmul_rn(Dc, xh));
    y[(int64_t)b * ldy + c] = __fmul_rn(yv, silu_f(__fmul_rn((float)z[(int64_t)b * ldz + c], p.s_z)));
  }
}

// Mamba1 int8 selective scan (K8): thread = one channel with
// all 16 states in registers, CTA = CH channels (128 at the 2.8B shape: 40 channel blocks x 16 time
// chunks = 640 CTAs).  Time is walked in chunks of M1_TC tokens whose int8 codes are staged into
// shared memory by cp.async one chunk ahead; B̂ | Ĉ are dequantised once per chunk into f32 for the
// whole CTA.  Per token a thread forms Δ = softplus(Δ̂ + dt_bias), x̂, SiLU(ẑ) and its 16
// Ȧ = 2^(Δ·A·log2 e) (SFU, off the recurrence chain), then updates the 16 states with packed
// f32x2 arithmetic (h = Ȧ·h + (Δx̂)·B̂, unfused like the oracle).  The states sit in the
// permuted order m1_perm so each f32x2 pair holds the same position of two 4-state quarters, and
// C·h is two packed FMA chains whose lanes are exactly the four quarter sums of the
// one-quarter-per-thread form, added as (q0 + q1) + (q2 + q3).  Codes are widened with the
// 1.5·2^23 magic add (integer + FMA pipes) instead of I2F, which shares the SFU's issue port.
// The final state is requantised once.
constexpr int M1_TC = 16;
#ifndef SQ_M1_UNROLL
#define SQ_M1_UNROLL 4
#endif
constexpr int M1_UNROLL = SQ_M1_UNROLL;   // tokens per unrolled recurrence step
__host__ __device__ constexpr int m1_perm(int p) { return (p >> 3) * 8 + ((p >> 1) & 3) + 4 * (p & 1); }
__device__ __forceinline__ float s8f(int v) { return __fsub_rn(__int_as_float(0x4B400000 + v), 12582912.0f); }
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NW>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NW) : "memory"); }

// Time-chunked parallel form (MODE 1 / 2, gridDim.z = time chunks): the recurrence h_t = Ȧ_t h_{t-1}
// + b_t is linear, so pass 1 (MODE 1) runs every chunk but the last from h = 0 (chunk 0 from the
// real initial state) and keeps its end state and its decay product Π Ȧ; pass 2 (MODE 2) starts
// chunk j from the folded carry h = Π_j ⊙ h + h_end_j of the chunks before it and re-runs the
// chunk with the y output; the last chunk requantises the final state.  MODE 0 is the single pass.
// The carried start state is the sequential one up to f32 rounding (tolerance-compared, like the
// oracle's chunked SSD).
template <int MODE, int CH, int TPC>
__global__ void __launch_bounds__(CH * TPC) mamba1_scan_chunk_kernel(sq_mamba1_params p, int B, int T, const int8_t* x,
                                                                     int64_t ldx, const int8_t* dt, int64_t lddt,
                                                                     const int8_t* BC, int64_t ldbc, const int8_t* z,
                                                                     int64_t ldz, int8_t* state, int state_in, float* y,
                                                                     int64_t ldy, float* ws, int tchunk) {
  constexpr int N = 16;
  constexpr int NT = CH * TPC;    // threads: TPC per channel
  constexpr int KP = 8 / TPC;     // f32x2 state pairs per thread (pairs hf*KP .. hf*KP+KP-1)
  __shared__ __align__(16) int8_t raw[2][M1_TC][3 * CH + 32];
  __shared__ __align__(16) float bcf[2][M1_TC][32];   // B̂ | Ĉ (f32, m1_perm order)
  const int tid = threadIdx.x;
  const int cl = tid / TPC, hf = tid % TPC;   // channel within the CTA, state half
  const int c0 = blockIdx.x * CH, c = c0 + cl;
  const int b = blockIdx.y;
  const int tc = blockIdx.z, nz = gridDim.z;
  pdl_trigger();
  if (MODE == 1 && tc == nz - 1) return;   // the last chunk's summary is never read
  float2 A2[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k)
    A2[k] = make_float2(p.A[(int64_t)c * N + m1_perm(2 * (hf * KP + k))] * 1.4426950408889634f,
                        p.A[(int64_t)c * N + m1_perm(2 * (hf * KP + k) + 1)] * 1.4426950408889634f);
  const float sh = p.s_h[c], Dc = p.D[c], sx = p.s_x[c], dtb = p.dt_bias[c];
  const float s_dt = p.s_dt, s_z = p.s_z, s_B = p.s_B, s_C = p.s_C;
  pdl_wait();   // inputs come from the previous grid
  int8_t* st = state + ((int64_t)b * p.d_inner + c) * N;
  const int t0 = tc * tchunk, t1 = min(T, t0 + tchunk);   // this CTA's time range
  // per-chunk summaries [2][nz][B][d_inner][N] (natural state order): end state (from 0; chunk 0
  // from the initial state) and decay product.  The thread's pairs hold states hf*16/TPC .. +16/TPC.
  constexpr int SPT = N / TPC;    // states per thread (a contiguous natural range)
  const int64_t cell = ((int64_t)b * p.d_inner + c) * N, zst = (int64_t)B * p.d_inner * N;
  const int sb = hf * SPT;        // first natural state of this thread
  float2 H[KP], P2[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int kg = hf * KP + k;
    P2[k] = make_float2(1.f, 1.f);
    H[k] = (state_in && (MODE == 0 || tc == 0))
               ? make_float2(__fmul_rn((float)st[m1_perm(2 * kg)], sh), __fmul_rn((float)st[m1_perm(2 * kg + 1)], sh))
               : make_float2(0.f, 0.f);
  }
  if (MODE == 2 && tc > 0) {   // carry: fold the chunks before this one (16-B loads, 4 chunks in flight)
    float e[SPT];
    auto ld = [&](const float* src, float (&d)[SPT]) {
#pragma unroll
      for (int i = 0; i < SPT / 4; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(src + sb + 4 * i);
        d[4 * i] = v.x; d[4 * i + 1] = v.y; d[4 * i + 2] = v.z; d[4 * i + 3] = v.w;
      }
    };
    ld(ws + cell, e);
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int kg = hf * KP + k;
      H[k] = make_float2(e[m1_perm(2 * kg) - sb], e[m1_perm(2 * kg + 1) - sb]);
    }
#pragma unroll 4
    for (int j = 1; j < tc; ++j) {
      float q[SPT];
      ld(ws + j * zst + cell, e);
      ld(ws + (nz + j) * zst + cell, q);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int kg = hf * KP + k;
        H[k] = __fadd2_rn(__fmul2_rn(make_float2(q[m1_perm(2 * kg) - sb], q[m1_perm(2 * kg + 1) - sb]), H[k]),
                          make_float2(e[m1_perm(2 * kg) - sb], e[m1_perm(2 * kg + 1) - sb]));
      }
    }
  }
  const int nch = (t1 - t0 + M1_TC - 1) / M1_TC;
  auto issue = [&](int ch) {   // x | dt | z codes (CH bytes per token row each) and the B̂Ĉ row, 16-B pieces
    constexpr int PPR = CH / 16;   // pieces per token row and kind
    for (int i = tid; i < 3 * M1_TC * PPR; i += NT) {
      const int kind = i / (M1_TC * PPR), j = i % (M1_TC * PPR);
      const int row = j / PPR, off = (j % PPR) * 16;
      const int t = t0 + ch * M1_TC + row;
      if (t < t1) {
        const int64_t tok = (int64_t)b * T + t;
        const int8_t* src = kind == 0 ? x + tok * ldx : kind == 1 ? dt + tok * lddt : z + tok * ldz;
        cp_async16(&raw[ch & 1][row][kind * CH + off], src + c0 + off);
      }
    }
    if (tid < 2 * M1_TC) {
      const int rb = tid >> 1, hb = (tid & 1) * 16;
      const int tb = t0 + ch * M1_TC + rb;
      if (tb < t1) cp_async16(&raw[ch & 1][rb][3 * CH + hb], BC + ((int64_t)b * T + tb) * ldbc + hb);
    }
    cp_async_commit();
  };
  static_assert(2 * M1_TC <= NT && CH % 16 == 0, "B|C pieces: one per thread of the first 32");
  issue(0);
  for (int ch = 0; ch < nch; ++ch) {
    const int tn = min(M1_TC, t1 - t0 - ch * M1_TC);
    cp_async_wait<0>();
    __syncthreads();   // raw[ch & 1] landed; every thread is done with chunk ch - 1 (raw and bcf)
    if (ch + 1 < nch) issue(ch + 1);
    const int8_t(*r)[3 * CH + 32] = raw[ch & 1];
    float(*bf)[32] = bcf[ch & 1];
    for (int i = tid; i < tn * 32; i += NT) {
      const int row = i >> 5, q = i & 31;
      const int src = q < N ? m1_perm(q) : N + m1_perm(q - N);
      bf[row][q] = __fmul_rn(s8f(r[row][3 * CH + src]), q < N ? s_B : s_C);
    }
    __syncthreads();
    float* yrow = y + ((int64_t)b * T + t0 + ch * M1_TC) * ldy + c;
#pragma unroll M1_UNROLL
    for (int tt = 0; tt < tn; ++tt) {
      const float delta = softplus_approx(__fadd_rn(__fmul_rn(s8f(r[tt][CH + cl]), s_dt), dtb));
      const float xv = __fmul_rn(s8f(r[tt][cl]), sx);
      const float dx = __fmul_rn(delta, xv);
      const float2 dl2 = make_float2(delta, delta), dx2 = make_float2(dx, dx);
      const float4* b4 = reinterpret_cast<const float4*>(bf[tt]);
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int kg = hf * KP + k;
        const float2 t = __fmul2_rn(dl2, A2[k]);
        const float2 av = make_float2(ex2_approx(t.x), ex2_approx(t.y));
        const float4 bq = b4[kg >> 1];
        const float2 bv = (kg & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
        H[k] = __fadd2_rn(__fmul2_rn(av, H[k]), __fmul2_rn(dx2, bv));
        if constexpr (MODE == 1) P2[k] = __fmul2_rn(P2[k], av);
      }
      if constexpr (MODE != 1) {
        // quarter sums: pairs 4m .. 4m+3 form the f32x2 chain of quarters (2m, 2m+1)
        float part[2 / TPC];
#pragma unroll
        for (int m = 0; m < 2 / TPC; ++m) {
          const int kg0 = hf * KP + 4 * m;
          const float4 cqa = b4[4 + (kg0 >> 1)], cqb = b4[5 + (kg0 >> 1)];
          float2 aq = __fmul2_rn(H[4 * m], make_float2(cqa.x, cqa.y));
          aq = __ffma2_rn(H[4 * m + 1], make_float2(cqa.z, cqa.w), aq);
          aq = __ffma2_rn(H[4 * m + 2], make_float2(cqb.x, cqb.y), aq);
          aq = __ffma2_rn(H[4 * m + 3], make_float2(cqb.z, cqb.w), aq);
          part[m] = __fadd_rn(aq.x, aq.y);
        }
        float acc;
        if constexpr (TPC == 1) {
          acc = __fadd_rn(part[0], part[1]);
        } else {   // (q0 + q1) from the even lane, (q2 + q3) from the odd lane, added in that order
          const float other = __shfl_xor_sync(0xffffffffu, part[0], 1);
          acc = __fadd_rn(hf == 0 ? part[0] : other, hf == 0 ? other : part[0]);
        }
        if (hf == 0) {
          const float gz = silu_approx(__fmul_rn(s8f(r[tt][2 * CH + cl]), s_z));
          yrow[(int64_t)tt * ldy] = __fmul_rn(__fadd_rn(acc, __fmul_rn(Dc, xv)), gz);
        }
      }
    }
  }
  if constexpr (MODE == 1) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int kg = hf * KP + k;
      ws[tc * zst + cell + m1_perm(2 * kg)] = H[k].x;
      ws[tc * zst + cell + m1_perm(2 * kg + 1)] = H[k].y;
      ws[(nz + tc) * zst + cell + m1_perm(2 * kg)] = P2[k].x;
      ws[(nz + tc) * zst + cell + m1_perm(2 * kg + 1)] = P2[k].y;
    }
  } else if (MODE == 0 || tc == nz - 1) {
#pragma unroll
    for (int k = 0; k < KP; ++k) {
      const int kg = hf * KP + k;
      st[m1_perm(2 * kg)] = quant8(H[k].x, sh);
      st[m1_perm(2 * kg + 1)] = quant8(H[k].y, sh);
    }
  }
}

// time chunks of the two-pass form: up to 16, chunks >= 32 tokens
#ifndef SQ_M1_TPC
#define SQ_M1_TPC 1
#endif
constexpr int M1_TPC = SQ_M1_TPC;   // threads per channel of the chunked scan
static int m1_ch(int d_inner) {
#ifdef SQ_M1_PROBE_CH   // profiling builds only
  if (d_inner % SQ_M1_PROBE_CH == 0) return SQ_M1_PROBE_CH;
#endif
  if (M1_TPC == 2) return d_inner % 64 == 0 ? 64 : 32;
  return d_inner % 128 == 0 ? 128 : d_inner % 64 == 0 ? 64 : 32;
}
static int m1_time_chunks(int d_inner, int B, int T) {
#ifdef SQ_M1_PROBE_NZ   // profiling builds only: fixed chunk count
  if (T / SQ_M1_PROBE_NZ >= M1_TC) return SQ_M1_PROBE_NZ;
#endif
  const int ctas = (d_inner / m1_ch(d_inner)) * B;
  int nz = 1;
  while (nz < 16 && ctas * nz < 16 * 148 && T / (nz * 2) >= 32) nz *= 2;
  return nz;
}

// Mamba1 W4A16 (float) scan: the same recurrence on f32 operands and an f32 state
// (oracle/ssm_block.py selective_scan, Mamba1 branch).  dt is the raw
// dt_proj output; B|C come from the x_proj output row (C at +N).
// PRE: Ȧ [B*T x d_inner x N] and Δ are inputs (SPEC selective_scan); z may be null.
template <int N, bool PRE>
__global__ void __launch_bounds__(128) mamba1_scan_f32_kernel(sq_mamba1_params p, int B, int T, const float* x,
                                                             int64_t ldx, const float* dt, const float* dAp,
                                                             int64_t lddt, const float* Bm, const float* Cm,
                                                             int64_t ldbc, const float* z, int64_t ldz, float* state,
                                                             int state_in, float* y, int64_t ldy) {
  pdl_trigger();
  pdl_wait();   // inputs come from the previous grid (launched with PDL_SMALL)
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (c >= p.d_inner) return;
  const float Dc = p.D[c], dtb = PRE ? 0.f : p.dt_bias[c];
  float A[N], hs[N];
#pragma unroll
  for (int n = 0; n < N; ++n) A[n] = PRE ? 0.f : p.A[c * N + n];
  float* st = state + ((int64_t)b * p.d_inner + c) * N;
#pragma unroll
  for (int n = 0; n < N; ++n) hs[n] = state_in ? st[n] : 0.f;
  for (int t = 0; t < T; ++t) {
    const int64_t tok = (int64_t)b * T + t;
    const float delta = PRE ? dt[tok * lddt + c] : softplus_f(__fadd_rn(dt[tok * lddt + c], dtb));
    const float xv = x[tok * ldx + c];
    const float dtx = __fmul_rn(delta, xv);
    const float* bp = Bm + tok * ldbc;
    const float* cp = Cm + tok * ldbc;
    const float* dap = PRE ? dAp + (tok * p.d_inner + c) * N : nullptr;
    float acc = 0.f;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float dA = PRE ? dap[n] : expf(__fmul_rn(delta, A[n]));
      hs[n] = __fadd_rn(__fmul_rn(dA, hs[n]), __fmul_rn(dtx, bp[n]));
      acc = fmaf(hs[n], cp[n], acc);
    }
    const float yv = __fadd_rn(acc, __fmul_rn(Dc, xv));
    y[tok * ldy + c] = z ? __fmul_rn(yv, silu_f(z[tok * ldz + c])) : yv;
  }
#pragma unroll
  for (int n = 0; n < N; ++n) st[n] = hs[n];
}

// ---------------------------------------------------------------------------------
// K9 decode: Mamba2 int8 state update, HBM-streaming version.
// CTA = (sequence, 4 consecutive heads), 256 threads; thread t owns the 16-column
// chunk (t % 8) of rows {t/8, t/8+32} of each head -> 8 x 16-B loads in flight per
// thread, a warp touches 512 contiguous bytes.  B̂/Ĉ are dequantised once per CTA
// into smem; Δ, Ȧ once per head.  Per element: byte->f32 via PRMT+FADD magic,
// h' = (Ȧ·s_h)·q + (Δ·x̂)·B̂ (two FMA-pipe ops), y += h'·Ĉ, requant with 1/s_h and a
// magic-number round-to-nearest-even (≤1-ulp differences from the oracle's
// unfused f32 ops, i.e. a ≤1-step code difference at rounding ties, tested).
constexpr int SU_HPC = 4;
constexpr int SU_THREADS = 256;

__device__ __forceinline__ float s8byte_to_f(uint32_t u_xor80, int i) {
  // u_xor80 = word ^ 0x80808080 (unsigned b+128); returns (float)(signed byte i)
  uint32_t bits;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bits) : "r"(u_xor80), "r"(0x4B000000u), "r"(0x7440u | (uint32_t)i));
  return __int_as_float(bits) - 8388736.0f;
}

__device__ __forceinline__ float s8byte_to_f_raw(uint32_t u_xor80, int i) {
  // 2^23 + 128 + (signed byte i); subtract 8388736 to get the value
  uint32_t bits;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(bits) : "r"(u_xor80), "r"(0x4B000000u), "r"(0x7440u | (uint32_t)i));
  return __int_as_float(bits);
}

__device__ __forceinline__ uint32_t f_to_s8bits(float v) {
  v = fminf(fmaxf(v, -128.f), 127.f);
  return __float_as_uint(v + 12582912.0f);   // low byte = rint(v) (two's complement)
}

__global__ void __launch_bounds__(SU_THREADS) mamba2_state_update_kernel(
    sq_mamba2_params p, const int8_t* __restrict__ x, int64_t ldx, const int8_t* __restrict__ Bm,
    const int8_t* __restrict__ Cm, int64_t ldbc, const int8_t* __restrict__ dt, int64_t lddt,
    const int8_t* __restrict__ z, int64_t ldz, int8_t* __restrict__ state, float* __restrict__ y, int64_t ldy) {
  constexpr int P = 64, N = 128;   // dispatcher guarantees
  __shared__ __align__(16) float sB[SU_HPC][N];
  __shared__ __align__(16) float sC[SU_HPC][N];
  __shared__ float s_dA[SU_HPC], s_dt[SU_HPC];
  const int b = blockIdx.y;
  const int h0 = blockIdx.x * SU_HPC;
  const int tid = threadIdx.x;
  const int chunk = tid & 7;
  const int r0 = tid >> 3;               // rows r0 and r0 + 32 of each head
  // 1) every global load this thread needs, issued up front (state: 8 x 16 B)
  int4 raw[SU_HPC][2];
  int8_t xq[SU_HPC][2], zq[SU_HPC][2];
  float sxr[SU_HPC][2], shr[SU_HPC][2], Dh[SU_HPC];
#pragma unroll
  for (int hh = 0; hh < SU_HPC; ++hh) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int row = r0 + 32 * k;
      const int ch = (h0 + hh) * P + row;
      raw[hh][k] = *reinterpret_cast<const int4*>(state + (((int64_t)b * p.n_heads + h0 + hh) * P + row) * N + chunk * 16);
      xq[hh][k] = x[(int64_t)b * ldx + ch];
      zq[hh][k] = z[(int64_t)b * ldz + ch];
      sxr[hh][k] = p.s_x[ch];
      shr[hh][k] = p.s_h[ch];
    }
    Dh[hh] = p.D[h0 + hh];
  }
  // 2) B̂/Ĉ of each head's group and the per-head scalars, staged once per CTA
  for (int i = tid; i < SU_HPC * N; i += SU_THREADS) {
    const int hh = i / N, n = i % N;
    const int g = p.head_group[h0 + hh];
    sB[hh][n] = __fmul_rn((float)Bm[(int64_t)b * ldbc + g * N + n], p.s_B[g]);
    sC[hh][n] = __fmul_rn((float)Cm[(int64_t)b * ldbc + g * N + n], p.s_C[g]);
  }
  if (tid < SU_HPC) {
    const int h = h0 + tid;
    const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dt[(int64_t)b * lddt + h], p.s_dt), p.dt_bias[h]));
    s_dt[tid] = delta;
    s_dA[tid] = expf(__fmul_rn(delta, p.A[h]));
  }
  __syncthreads();
#pragma unroll
  for (int hh = 0; hh < SU_HPC; ++hh) {
    const int h = h0 + hh;
    const float dA = s_dA[hh], delta = s_dt[hh];
    float bv[16], cvv[16];    // this thread's 16 state columns of B̂ / Ĉ (smem broadcast)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 b4 = *reinterpret_cast<const float4*>(&sB[hh][chunk * 16 + e * 4]);
      const float4 c4 = *reinterpret_cast<const float4*>(&sC[hh][chunk * 16 + e * 4]);
      bv[e * 4] = b4.x; bv[e * 4 + 1] = b4.y; bv[e * 4 + 2] = b4.z; bv[e * 4 + 3] = b4.w;
      cvv[e * 4] = c4.x; cvv[e * 4 + 1] = c4.y; cvv[e * 4 + 2] = c4.z; cvv[e * 4 + 3] = c4.w;
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int row = r0 + 32 * k;
      const int ch = h * P + row;
      const float sh = shr[hh][k];
      const float xh = __fmul_rn((float)xq[hh][k], sxr[hh][k]);
      const float dtx = __fmul_rn(delta, xh);
      // scaled units t = h'/s_h = Ȧ·q + (Δx̂/s_h)·B̂: the requant is rint(t), and
      // y = s_h·Σ t·Ĉ.  Pairs of state columns go through packed FFMA2/FMUL2/FADD2.
      const float rs = __fdiv_rn(dtx, sh);
      const float2 dA2 = make_float2(dA, dA), rs2 = make_float2(rs, rs);
      const float2 mg = make_float2(-8388736.0f, -8388736.0f);
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw[hh][k]);
      uint32_t outw[4];
      float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t u = w[e] ^ 0x80808080u;
        uint32_t q[4];
#pragma unroll
        for (int i = 0; i < 4; i += 2) {
          const int n = e * 4 + i;
          float2 hq = make_float2(s8byte_to_f_raw(u, i), s8byte_to_f_raw(u, i + 1));
          hq = __fadd2_rn(hq, mg);
          const float2 t = __ffma2_rn(dA2, hq, __fmul2_rn(rs2, make_float2(bv[n], bv[n + 1])));
          acc2 = __ffma2_rn(t, make_float2(cvv[n], cvv[n + 1]), acc2);
          const float2 cl = make_float2(fminf(fmaxf(t.x, -128.f), 127.f), fminf(fmaxf(t.y, -128.f), 127.f));
          const float2 rq = __fadd2_rn(cl, make_float2(12582912.0f, 12582912.0f));   // low byte = rint
          q[i] = __float_as_uint(rq.x);
          q[i + 1] = __float_as_uint(rq.y);
        }
        outw[e] = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
      }
      float acc = __fmul_rn(sh, __fadd_rn(acc2.x, acc2.y));
      const int64_t off = (((int64_t)b * p.n_heads + h) * P + row) * N + chunk * 16;
      *reinterpret_cast<int4*>(state + off) = make_int4(outw[0], outw[1], outw[2], outw[3]);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (chunk == 0) {
        const float yv = __fadd_rn(acc, __fmul_rn(Dh[hh], xh));
        const float zv = __fmul_rn((float)zq[hh][k], p.s_z);
        y[(int64_t)b * ldy + ch] = __fmul_rn(yv, silu_f(zv));
      }
    }
  }
}

// Barrier-free variant: CTA = (sequence, 2 heads) x 256 threads; thread t owns head
// t >> 7, state columns [16*(t&7), +16) of rows ((t&127)>>3) + 16k, k = 0..3.  Every
// thread issues all of its loads (4 x 16-B state pieces, its 16 B̂ / Ĉ codes, per-row and
// per-head scalars) up front and computes its head's Δ / Ȧ itself — no smem, no
// __syncthreads, ~64 registers, so 4 CTAs (32 warps) per SM keep HBM busy.
__global__ void __launch_bounds__(256, 3) mamba2_state_update2_kernel(
    sq_mamba2_params p, const int8_t* __restrict__ x, int64_t ldx, const int8_t* __restrict__ Bm,
    const int8_t* __restrict__ Cm, int64_t ldbc, const int8_t* __restrict__ dt, int64_t lddt,
    const int8_t* __restrict__ z, int64_t ldz, int8_t* __restrict__ state, float* __restrict__ y, int64_t ldy) {
  constexpr int P = 64, N = 128;
  const int b = blockIdx.y;
  const int h = blockIdx.x * 2 + (threadIdx.x >> 7);
  const int t = threadIdx.x & 127;
  const int chunk = t & 7;
  const int r0 = t >> 3;
  const int g = p.head_group[h];
  int8_t* st_base = state + (((int64_t)b * p.n_heads + h) * P) * N + chunk * 16;
  int4 raw[4];
  int8_t xq[4], zq[4];
  float sxr[4], shr[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int row = r0 + 16 * k;
    raw[k] = *reinterpret_cast<const int4*>(st_base + (int64_t)row * N);
    const int ch = h * P + row;
    xq[k] = x[(int64_t)b * ldx + ch];
    zq[k] = z[(int64_t)b * ldz + ch];
    sxr[k] = p.s_x[ch];
    shr[k] = p.s_h[ch];
  }
  const int4 bq = *reinterpret_cast<const int4*>(Bm + (int64_t)b * ldbc + g * N + chunk * 16);
  const int4 cq = *reinterpret_cast<const int4*>(Cm + (int64_t)b * ldbc + g * N + chunk * 16);
  const float sB = p.s_B[g], sC = p.s_C[g];
  const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dt[(int64_t)b * lddt + h], p.s_dt), p.dt_bias[h]));
  const float dA = expf(__fmul_rn(delta, p.A[h]));
  const float Dh = p.D[h];
  // B̂ / Ĉ for this thread's 16 columns (exact: f32(code) * scale)
  float2 bv[8], cv[8];
  {
    const uint32_t* bw = reinterpret_cast<const uint32_t*>(&bq);
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(&cq);
    const float2 mg = make_float2(-8388736.0f, -8388736.0f);
    const float2 sB2 = make_float2(sB, sB), sC2 = make_float2(sC, sC);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t ub = bw[e] ^ 0x80808080u, uc = cw[e] ^ 0x80808080u;
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        bv[e * 2 + i / 2] = __fmul2_rn(__fadd2_rn(make_float2(s8byte_to_f_raw(ub, i), s8byte_to_f_raw(ub, i + 1)), mg), sB2);
        cv[e * 2 + i / 2] = __fmul2_rn(__fadd2_rn(make_float2(s8byte_to_f_raw(uc, i), s8byte_to_f_raw(uc, i + 1)), mg), sC2);
      }
    }
  }
  const float2 dA2 = make_float2(dA, dA);
  const float2 mg = make_float2(-8388736.0f, -8388736.0f);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int row = r0 + 16 * k;
    const float sh = shr[k];
    const float xh = __fmul_rn((float)xq[k], sxr[k]);
    const float rs = __fdiv_rn(__fmul_rn(delta, xh), sh);   // t = h'/s_h = Ȧ·q + (Δx̂/s_h)·B̂
    const float2 rs2 = make_float2(rs, rs);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&raw[k]);
    uint32_t outw[4];
    float2 acc2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t u = w[e] ^ 0x80808080u;
      uint32_t q[4];
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        const int n2 = e * 2 + i / 2;
        const float2 hq = __fadd2_rn(make_float2(s8byte_to_f_raw(u, i), s8byte_to_f_raw(u, i + 1)), mg);
        const float2 tt = __ffma2_rn(dA2, hq, __fmul2_rn(rs2, bv[n2]));
        acc2 = __ffma2_rn(tt, cv[n2], acc2);
        const float2 cl = make_float2(fminf(fmaxf(tt.x, -128.f), 127.f), fminf(fmaxf(tt.y, -128.f), 127.f));
        const float2 rq = __fadd2_rn(cl, make_float2(12582912.0f, 12582912.0f));   // low byte = rint
        q[i] = __float_as_uint(rq.x);
        q[i + 1] = __float_as_uint(rq.y);
      }
      outw[e] = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
    }
    *reinterpret_cast<int4*>(st_base + (int64_t)row * N) = make_int4(outw[0], outw[1], outw[2], outw[3]);
    float acc = __fmul_rn(sh, __fadd_rn(acc2.x, acc2.y));
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    if (chunk == 0) {
      const int ch = h * P + row;
      const float yv = __fadd_rn(acc, __fmul_rn(Dh, xh));
      const float zv = __fmul_rn((float)zq[k], p.s_z);
      y[(int64_t)b * ldy + ch] = __fmul_rn(yv, silu_f(zv));
    }
  }
}

}  // namespace sq

using namespace sq;

extern "C" int sq_ssd_scan_int8(const sq_mamba2_params* p, int B, int T, const int8_t* x, int64_t ldx,
                                const int8_t* Bm, const int8_t* Cm, int64_t ldbc, const int8_t* dt, int64_t lddt,
                                const int8_t* z, int64_t ldz, int8_t* state, int state_in, float* y, int64_t ldy,
                                int chunk, void* stream) {
  // chunk selects the engine per call: 128 = tcgen05 (128-token chunks, ssd_chunk_tc.cu), anything else
  // = mma.sync (64-token chunks, ssd_chunk.cu).  Results agree to the SPEC chunk tolerance.
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "sq_ssd_scan_int8: bad args");
  if (B == 0 || T == 0) return SQ_OK;
  if (T > 1) {   // chunked SSD on the tensor cores (ssd_chunk_tc.cu tcgen05, ssd_chunk.cu mma.sync);
                  // other shapes: sequential scan
    if (chunk == 128) {
      const int rc = launch_ssd_chunk_tc(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy,
                                         as_stream(stream));
      if (rc != SQ_ERR_ARG) return rc;
    }
    const int rc = launch_ssd_chunk(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy,
                                    as_stream(stream));
    if (rc != SQ_ERR_ARG) return rc;
  }
  return launch_mamba2<int8_t>(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy,
                               as_stream(stream), "sq_ssd_scan_int8");
}

extern "C" int sq_state_update_int8(const sq_mamba2_params* p, int B, const int8_t* x, int64_t ldx,
                                    const int8_t* Bm, const int8_t* Cm, int64_t ldbc, const int8_t* dt,
                                    int64_t lddt, const int8_t* z, int64_t ldz, int8_t* state, float* y,
                                    int64_t ldy, void* stream) {
  if (p && p->head_dim == 64 && p->d_state == 128 && p->n_heads % SU_HPC == 0 && ldbc % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(state) & 15) == 0) {
    if (B == 0) return SQ_OK;
    mamba2_state_update2_kernel<<<dim3(p->n_heads / 2, B), 256, 0, as_stream(stream)>>>(
        *p, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, y, ldy);
    return check_launch("sq_state_update_int8");
  }
  return launch_mamba2<int8_t>(p, B, 1, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, 1, y, ldy,
                               as_stream(stream), "sq_state_update_int8");
}

extern "C" int sq_ssd_scan_f32(const sq_mamba2_params* p, int B, int T, const float* x, int64_t ldx,
                               const float* Bm, const float* Cm, int64_t ldbc, const float* dt, int64_t lddt,
                               const float* z, int64_t ldz, float* state, int state_in, float* y, int64_t ldy,
                               void* stream) {
  if (p && B > 0 && T > 0 && p->head_dim % 32 == 0 && (p->d_state == 64 || p->d_state == 128 || p->d_state == 256) &&
      p->n_groups >= 1 && ldbc % 2 == 0 && (reinterpret_cast<uintptr_t>(Bm) & 7) == 0 &&
      (reinterpret_cast<uintptr_t>(Cm) & 7) == 0 && (reinterpret_cast<uintptr_t>(state) & 7) == 0) {
    const dim3 grid(p->n_heads, B, p->head_dim / 32);
    cudaStream_t st = as_stream(stream);
    if (p->d_state == 64)
      launch_k(PDL_SMALL, mamba2_scan_f32_rows_kernel<2, false>, grid, dim3(128), 0, st, *p, T, x, ldx, Bm, Cm, ldbc, dt, (const float*)nullptr, lddt, z, ldz, state, state_in, y, ldy);
    else if (p->d_state == 128)
      launch_k(PDL_SMALL, mamba2_scan_f32_rows_kernel<4, false>, grid, dim3(128), 0, st, *p, T, x, ldx, Bm, Cm, ldbc, dt, (const float*)nullptr, lddt, z, ldz, state, state_in, y, ldy);
    else
      launch_k(PDL_SMALL, mamba2_scan_f32_rows_kernel<8, false>, grid, dim3(128), 0, st, *p, T, x, ldx, Bm, Cm, ldbc, dt, (const float*)nullptr, lddt, z, ldz, state, state_in, y, ldy);
    return check_launch("sq_ssd_scan_f32");
  }
  return launch_mamba2<float>(p, B, T, x, ldx, Bm, Cm, ldbc, dt, lddt, z, ldz, state, state_in, y, ldy,
                              as_stream(stream), "sq_ssd_scan_f32");
}

extern "C" int64_t sq_selective_scan_int8_ws_bytes(const sq_mamba1_params* p, int B, int T) {
  if (!p || B < 0 || T < 0) return -1;
  const int nz = m1_time_chunks(p->d_inner, B, T);
  return nz > 1 ? (int64_t)2 * nz * B * p->d_inner * p->d_state * 4 : 0;
}

extern "C" int sq_selective_scan_int8(const sq_mamba1_params* p, int B, int T, const int8_t* x, int64_t ldx,
                                      const int8_t* dt, int64_t lddt, const int8_t* BC, int64_t ldbc,
                                      const int8_t* z, int64_t ldz, int8_t* state, int state_in, float* y,
                                      int64_t ldy, void* ws, void* stream) {
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "sq_selective_scan_int8: bad args");
  SQ_REQUIRE(p->d_state == 16, SQ_ERR_SHAPE, "sq_selective_scan_int8: d_state must be 16 (got %d)", p->d_state);
  if (B == 0 || T == 0) return SQ_OK;
  if (T > 1 && p->d_inner % 32 == 0 && ldx % 16 == 0 && lddt % 16 == 0 && ldz % 16 == 0 && ldbc % 16 == 0 &&
      !((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dt) | reinterpret_cast<uintptr_t>(z) |
         reinterpret_cast<uintptr_t>(BC)) & 15)) {
    cudaStream_t st = as_stream(stream);
    const int nz = ws ? m1_time_chunks(p->d_inner, B, T) : 1;
    const int tchunk = ((T + nz - 1) / nz + M1_TC - 1) / M1_TC * M1_TC;
    const int chn = m1_ch(p->d_inner);
    const dim3 grid(p->d_inner / chn, B, (T + tchunk - 1) / tchunk);
    float* wsf = reinterpret_cast<float*>(ws);
    SQ_REQUIRE(grid.z == 1 || (reinterpret_cast<uintptr_t>(ws) & 15) == 0, SQ_ERR_LAYOUT,
               "sq_selective_scan_int8: ws alignment");
#define SQ_M1_LAUNCH(MODE, C)                                                                                     \
  launch_k(PDL_SMALL8, mamba1_scan_chunk_kernel<MODE, C, M1_TPC>, grid, dim3(C * M1_TPC), 0, st, *p, B, T, x, ldx, dt, \
           lddt, BC, ldbc, \
           z, ldz, state, state_in, y, ldy, wsf, tchunk)
#define SQ_M1_PASSES(C)            \
  if (grid.z == 1) {               \
    SQ_M1_LAUNCH(0, C);            \
  } else {                         \
    SQ_M1_LAUNCH(1, C);            \
    SQ_M1_LAUNCH(2, C);            \
  }
    if (chn == 128) {
      SQ_M1_PASSES(128)
    } else if (chn == 64) {
      SQ_M1_PASSES(64)
    } else {
      SQ_M1_PASSES(32)
    }
#undef SQ_M1_PASSES
#undef SQ_M1_LAUNCH
    return check_launch("sq_selective_scan_int8");
  }
  if (T == 1) {   // decode step: 16 threads per channel
    launch_k(PDL_SMALL8, mamba1_step_kernel, dim3((p->d_inner + 15) / 16, B), dim3(256), 0, as_stream(stream), *p, B, x,
             ldx, dt, lddt, BC, ldbc, z, ldz, state, state_in, y, ldy);
    return check_launch("sq_selective_scan_int8");
  }
  dim3 grid((p->d_inner + 127) / 128, B);
  launch_k(PDL_SMALL8, mamba1_scan_kernel<16>, grid, dim3(128), 0, as_stream(stream), *p, B, T, x, ldx, dt, lddt, BC, ldbc, z, ldz, state,
                                                              state_in, y, ldy);
  return check_launch("sq_selective_scan_int8");
}

extern "C" int sq_selective_scan_f32(const sq_mamba1_params* p, int B, int T, const float* x, int64_t ldx,
                                     const float* dt, int64_t lddt, const float* BC, int64_t ldbc, const float* z,
                                     int64_t ldz, float* state, int state_in, float* y, int64_t ldy, void* stream) {
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "sq_selective_scan_f32: bad args");
  SQ_REQUIRE(p->d_state == 16, SQ_ERR_SHAPE, "sq_selective_scan_f32: d_state must be 16 (got %d)", p->d_state);
  if (B == 0 || T == 0) return SQ_OK;
  dim3 grid((p->d_inner + 127) / 128, B);
  launch_k(PDL_SMALL, mamba1_scan_f32_kernel<16, false>, grid, dim3(128), 0, as_stream(stream), *p, B, T, x, ldx, dt,
           (const float*)nullptr, lddt, BC, BC + 16, ldbc, z, ldz, state, state_in, y, ldy);
  return check_launch("sq_selective_scan_f32");
}

// ---- SPEC float ops (ssm_block.discretize / selective_scan / ssd_chunked on the GPU) ------
__global__ void discretize_kernel(const float* dt_raw, int64_t ld, const float* __restrict__ dt_bias,
                                  const float* __restrict__ A, int M, int H, int N, float* dA, float* delta) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * H) return;
  const int m = i / H, h = i % H;
  const float d = softplus_f(__fadd_rn(dt_raw[(int64_t)m * ld + h], dt_bias[h]));
  delta[i] = d;
  for (int n = 0; n < N; ++n) dA[i * N + n] = expf(__fmul_rn(d, A[(int64_t)h * N + n]));
}

extern "C" int sq_discretize_f32(const float* dt_raw, int64_t ld, const float* dt_bias, const float* A, int M, int H,
                                 int N, float* dA, float* delta, void* stream) {
  SQ_REQUIRE(M >= 0 && H > 0 && N >= 1 && ld >= H, SQ_ERR_SHAPE, "sq_discretize_f32: bad shape");
  if (M == 0) return SQ_OK;
  const int64_t n = (int64_t)M * H;
  discretize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(dt_raw, ld, dt_bias, A, M, H, N, dA,
                                                                                 delta);
  return check_launch("sq_discretize_f32");
}

// Mamba2 recurrence on precomputed Ȧ / Δ for small d_state (16 / 32, e.g. the SPEC toy dims):
// one thread per (sequence, head, row), the state row in registers.
template <int N>
__global__ void __launch_bounds__(128) scan2_pre_small_kernel(sq_mamba2_params p, int B, int T, const float* x,
                                                              int64_t ldx, const float* dAp, const float* dt,
                                                              int64_t lddt, const float* Bm, const float* Cm,
                                                              int64_t ldbc, const float* z, int64_t ldz, float* state,
                                                              int state_in, float* y, int64_t ldy) {
  const int P = p.head_dim;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)B * p.n_heads * P) return;
  const int r = idx % P, h = (idx / P) % p.n_heads, b = idx / ((int64_t)P * p.n_heads);
  const int g = p.head_group[h];
  float* st = state + idx * N;
  float hs[N];
#pragma unroll
  for (int n = 0; n < N; ++n) hs[n] = state_in ? st[n] : 0.f;
  const float Dh = p.D[h];
  for (int t = 0; t < T; ++t) {
    const int64_t tok = (int64_t)b * T + t;
    const float delta = dt[tok * lddt + h], dA = dAp[tok * lddt + h];
    const float xv = x[tok * ldx + h * P + r];
    const float dtx = __fmul_rn(delta, xv);
    const float* bp = Bm + tok * ldbc + g * N;
    const float* cp = Cm + tok * ldbc + g * N;
    float acc = 0.f;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      hs[n] = __fadd_rn(__fmul_rn(dA, hs[n]), __fmul_rn(dtx, bp[n]));
      acc = fmaf(hs[n], cp[n], acc);
    }
    const float yv = __fadd_rn(acc, __fmul_rn(Dh, xv));
    const int ch = h * P + r;
    y[tok * ldy + ch] = z ? __fmul_rn(yv, silu_f(z[tok * ldz + ch])) : yv;
  }
#pragma unroll
  for (int n = 0; n < N; ++n) st[n] = hs[n];
}

extern "C" int sq_selective_scan2_pre_f32(const sq_mamba2_params* p, int B, int T, const float* x, int64_t ldx,
                                          const float* dA, const float* delta, int64_t lddt, const float* Bm,
                                          const float* Cm, int64_t ldbc, const float* z, int64_t ldz, float* state,
                                          int state_in, float* y, int64_t ldy, void* stream) {
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "sq_selective_scan2_pre_f32: bad args");
  const int N = p ? p->d_state : 0;
  SQ_REQUIRE(p->n_groups >= 1 && (N == 16 || N == 32 || ((N == 64 || N == 128 || N == 256) &&
                                                                      p->head_dim % 8 == 0 && ldbc % 2 == 0)),
             SQ_ERR_SHAPE, "sq_selective_scan2_pre_f32: d_state in {16,32,64,128,256} (P=%d N=%d)", p->head_dim, N);
  if (B == 0 || T == 0) return SQ_OK;
  cudaStream_t st = as_stream(stream);
  if (N <= 32) {
    const int64_t rows = (int64_t)B * p->n_heads * p->head_dim;
    const unsigned nb = (unsigned)((rows + 127) / 128);
    if (N == 16)
      scan2_pre_small_kernel<16><<<nb, 128, 0, st>>>(*p, B, T, x, ldx, dA, delta, lddt, Bm, Cm, ldbc, z, ldz, state,
                                                     state_in, y, ldy);
    else
      scan2_pre_small_kernel<32><<<nb, 128, 0, st>>>(*p, B, T, x, ldx, dA, delta, lddt, Bm, Cm, ldbc, z, ldz, state,
                                                     state_in, y, ldy);
    return check_launch("sq_selective_scan2_pre_f32");
  }
  const dim3 grid(p->n_heads, B, (p->head_dim + 31) / 32);
  if (p->d_state == 64)
    mamba2_scan_f32_rows_kernel<2, true><<<grid, 128, 0, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, delta, dA, lddt, z, ldz,
                                                               state, state_in, y, ldy);
  else if (p->d_state == 128)
    mamba2_scan_f32_rows_kernel<4, true><<<grid, 128, 0, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, delta, dA, lddt, z, ldz,
                                                               state, state_in, y, ldy);
  else
    mamba2_scan_f32_rows_kernel<8, true><<<grid, 128, 0, st>>>(*p, T, x, ldx, Bm, Cm, ldbc, delta, dA, lddt, z, ldz,
                                                               state, state_in, y, ldy);
  return check_launch("sq_selective_scan2_pre_f32");
}

extern "C" int sq_selective_scan1_pre_f32(const sq_mamba1_params* p, int B, int T, const float* x, int64_t ldx,
                                          const float* dA, const float* delta, int64_t lddt, const float* Bm,
                                          const float* Cm, int64_t ldbc, const float* z, int64_t ldz, float* state,
                                          int state_in, float* y, int64_t ldy, void* stream) {
  SQ_REQUIRE(p && B >= 0 && T >= 0, SQ_ERR_ARG, "sq_selective_scan1_pre_f32: bad args");
  SQ_REQUIRE(p->d_state == 16, SQ_ERR_SHAPE, "sq_selective_scan1_pre_f32: d_state must be 16 (got %d)", p->d_state);
  if (B == 0 || T == 0) return SQ_OK;
  dim3 grid((p->d_inner + 127) / 128, B);
  mamba1_scan_f32_kernel<16, true><<<grid, 128, 0, as_stream(stream)>>>(*p, B, T, x, ldx, delta, dA, lddt, Bm, Cm, ldbc,
                                                                         z, ldz, state, state_in, y, ldy);
  return check_launch("sq_selective_scan1_pre_f32");
}
