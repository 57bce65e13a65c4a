// Mamba1 int8 decode, SSM half of a block in ONE launch (b <= 8; configs[4] decode is b = 1):
//   conv update (+ cache shift) -> x_proj (W8A8, requant) -> dt_proj (W8A8, requant)
//   -> selective-scan step (int8 state) -> gated RMSNorm + FWHT + quant (yq for out_proj).
// At b = 1 every stage is a few microseconds of latency and almost no work (x_proj 1 MB,
// dt_proj 0.8 MB of weights), so the five-launch chain (profiles/r02_launches_m1decode.txt:
// 4.6-7.7 us per launch cold) is replaced by one persistent grid (one CTA per SM) whose phases
// are separated by grid-wide barriers (a self-resetting sense counter in the caller's zeroed
// workspace).
//
// Arithmetic is the unfused chain's, op for op:
//   conv:     conv1d_update_kernel (conv1d.cu) -- exact f32 order, SiLU, quant8
//   x_proj / dt_proj: exact int32 dot products (dp4a), then quant8(f32(acc) * alpha[n], cs[n]),
//             the tcgen05 GEMM's EPI_QUANT epilogue (gemm_a8_tc.cu)
//   scan:     mamba1_step_kernel (scan.cu) -- 16 threads per channel, the same shuffle order
//   norm:     (y * r) * gamma, r = rms_factor(Σy² in f64), Sylvester stages h = 1, 2, ... in f32,
//             quant8 with s_y (gate_norm_had1k_kernel; Σy² is summed in another fixed order)
// PDL: parameters before the dependency wait; the dependents are released only after the last
// grid barrier (all CTAs resident), so an early-launched out_proj cannot starve the grid.
#include <mutex>

#include "common.cuh"

namespace sq {

constexpr int M1D_THREADS = 512;
constexpr int M1D_MAXB = 8;
constexpr int M1D_MAXBLK = 4096;   // Hadamard block (D & -D) staged in shared memory
constexpr int M1D_MAXRW = 16;      // dt_proj row words per thread (dt_rank <= 8 * 4 * 16)

__device__ __forceinline__ void cp_async16_m1(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

#ifdef SQ_M1D_TRACE   // profiling builds only: per-phase timestamps of CTA 0 / the last CTA in ws[64..]
__device__ __forceinline__ void m1d_mark(uint8_t* ws, int k) {
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    reinterpret_cast<unsigned long long*>(ws + 64)[k + (blockIdx.x == 0 ? 0 : 10)] = t;
  }
}
#define M1D_MARK(k) m1d_mark(a.ws, k)
#else
#define M1D_MARK(k)
#endif

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid-wide barrier on one word of zero-initialised workspace: CTA 0 adds 2^31 - (G - 1), every
// other CTA adds 1, so the word's top bit flips exactly when the last CTA arrives (one atomic
// per CTA, no separate release step) and its low bits return to their value: self-resetting.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned inc = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
    __threadfence();
    const unsigned old = atomicAdd(bar, inc);
    while (((ld_acquire_u32(bar) ^ old) & 0x80000000u) == 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float rms_factor_m1(double ss, int D, float eps) {   // rownorm.cu rms_factor
  const float ms = (float)(ss / (double)D);
  return __fdiv_rn(1.0f, sqrtf(__fadd_rn(ms, eps)));
}

struct M1DecodeArgs {
  sq_mamba1_decode_params p;
  int B;
  const int8_t* zx;
  int64_t ldzx;
  int8_t* cache;
  int8_t* state;
  uint8_t* ws;
  int8_t* yq;
  int64_t ldyq;
  // whole-layer mode (sq_mamba1_decode_layer_int8): pre-norm + in_proj before, out_proj after
  int layer;
  sq_mamba1_layer_params lp;
  float* h;
  int64_t ldh;
};

// workspace: [0, 256) barrier words | xc int8 [B x di] | xd int8 [B x NX] | y f32 [B x di] |
// zx int8 [B x 2 di] | yq int8 [B x di] (the last two in whole-layer mode)
struct M1Ws {
  int64_t xc, xd, y, zx, yq, total;
  __host__ __device__ M1Ws(int B, int di, int nx) {
    auto up = [](int64_t v) { return (v + 255) & ~(int64_t)255; };
    xc = 256;
    xd = xc + up((int64_t)B * di);
    y = xd + up((int64_t)B * nx);
    zx = y + up((int64_t)B * di * 4);
    yq = zx + up((int64_t)B * 2 * di);
    total = yq + up((int64_t)B * di);
  }
};
constexpr int M1D_MAXK16 = 16;   // 16-B weight pieces per lane and row of out_proj (K = d_inner <= 8192)
constexpr int M1D_MAXKIN = 8;    // ... of in_proj (K = d_model <= 4096; double-buffered)

__global__ void __launch_bounds__(M1D_THREADS, 1) mamba1_decode_fused_kernel(M1DecodeArgs a) {
  const sq_mamba1_decode_params& P = a.p;
  const sq_mamba1_params& S = P.ssm;
  constexpr int N = 16;
  const int di = S.d_inner, R = P.dt_rank, NX = R + 2 * N, Kc = P.conv_kernel, B = a.B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, gthreads = G * M1D_THREADS;
  const M1Ws L(B, di, NX);
  unsigned* bar = reinterpret_cast<unsigned*>(a.ws);
  int8_t* xc = reinterpret_cast<int8_t*>(a.ws + L.xc);
  int8_t* xd = reinterpret_cast<int8_t*>(a.ws + L.xd);
  float* y = reinterpret_cast<float*>(a.ws + L.y);
  extern __shared__ __align__(16) int8_t xw[];   // this CTA's x_proj rows n = blockIdx.x + k*G

  // ---- static operands before the grid dependency wait: x_proj rows (cp.async), the first
  // conv channel's and the first scan channel's parameters
  for (int n = blockIdx.x + warp * G; n < NX; n += G * (M1D_THREADS / 32)) {
    const int8_t* wr = P.xproj_w + (int64_t)n * di;
    int8_t* dst = xw + (int64_t)((n - blockIdx.x) / G) * di;
    for (int k = lane * 16; k < di; k += 32 * 16) cp_async16_m1(dst + k, wr + k);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  const int n2 = blockIdx.x + warp * G;   // this warp's first x_proj row
  const float xal = n2 < NX ? P.xproj_alpha[n2] : 0.f, xcs = n2 < NX ? P.xproj_cs[n2] : 1.f;
  const int blk = P.hadamard ? (di & -di) : di;
  const int nblk = di / blk;
  float gw[M1D_MAXBLK / M1D_THREADS];   // γ of this CTA's first (sequence, block) of phase 4
#pragma unroll
  for (int e = 0; e < M1D_MAXBLK / M1D_THREADS; ++e) {
    const int i = tid + e * M1D_THREADS;
    gw[e] = (P.hadamard && i < blk && blockIdx.x < B * nblk) ? P.norm_w[(blockIdx.x % nblk) * blk + i] : 0.f;
  }
  const int i1 = blockIdx.x * M1D_THREADS + tid;   // phase-1 (sequence, channel) of this thread
  float cw[8], cb = 0.f, csi = 0.f, cso = 1.f;
  if (i1 < B * di) {
    const int c = i1 % di;
    csi = P.conv_s_in[c];
    cso = P.conv_s_out[c];
    cb = P.conv_b[c];
#pragma unroll
    for (int j = 0; j < 8; ++j) cw[j] = j < Kc ? P.conv_w[c * Kc + j] : 0.f;
  }
  // phase 3: 8 threads per (sequence, channel), thread j owns states j and j + 8
  const int j8 = tid & 7;
  const int u3 = (blockIdx.x * M1D_THREADS + tid) >> 3;
  const int nw4 = R / 4;
  float A0 = 0.f, A1 = 0.f, dtb = 0.f, sx = 0.f, sh = 1.f, Dc = 0.f, dal = 0.f, dcs = 1.f;
  int dw[M1D_MAXRW];
  if (u3 < B * di) {
    const int c = u3 % di;
    A0 = S.A[(int64_t)c * N + j8];
    A1 = S.A[(int64_t)c * N + j8 + 8];
    dtb = S.dt_bias[c]; sx = S.s_x[c]; sh = S.s_h[c]; Dc = S.D[c];
    dal = P.dtproj_alpha[c]; dcs = P.dtproj_cs[c];
    const int* wr = reinterpret_cast<const int*>(P.dtproj_w + (int64_t)c * R);
#pragma unroll
    for (int t = 0; t < M1D_MAXRW; ++t) dw[t] = j8 + 8 * t < nw4 ? __ldg(wr + j8 + 8 * t) : 0;
  }
  M1D_MARK(0);
  pdl_wait();   // zx and the cached conv inputs / state come from earlier grids
  M1D_MARK(1);
  const int xrows = (NX + G - 1) / G;
  int8_t* xs_base = xw + (int64_t)xrows * di;          // xc staging [B x di] (phase 2)
  int8_t* us = xs_base + (int64_t)B * di;              // u codes [B x d_model] (phase 0)
  if (a.layer) {
    // ---------------- phase 0: the model's pre-norm + quant of h (rmsnorm16_kernel's math and
    // summation order: D/16 threads x 16 contiguous elements, f64 squares, warp xor trees, warps
    // in order), every CTA for itself; then in_proj rows, one per warp, dp4a over the u codes
    const sq_mamba1_layer_params& lp = a.lp;
    const int dm = lp.d_model, nthr = dm / 16, nwr = (nthr + 31) / 32;
    __shared__ double lred[M1D_THREADS / 32];
    for (int b = 0; b < B; ++b) {
      float v[16];
      double ss = 0.0;
      if (tid < nthr) {
        const float* hr = a.h + (int64_t)b * a.ldh + tid * 16;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float4 f = *reinterpret_cast<const float4*>(hr + e * 4);
          v[e * 4] = f.x; v[e * 4 + 1] = f.y; v[e * 4 + 2] = f.z; v[e * 4 + 3] = f.w;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) ss += (double)v[i] * (double)v[i];
      }
      if (warp < nwr) {
        ss = warp_sum_d(ss);
        if (lane == 0) lred[warp] = ss;
      }
      __syncthreads();
      double tot = 0.0;
      for (int w = 0; w < nwr; ++w) tot += lred[w];
      const float r = rms_factor_m1(tot, dm, lp.ln_eps);
      if (tid < nthr) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          us[(int64_t)b * dm + tid * 16 + i] = quant8(__fmul_rn(__fmul_rn(v[i], r), lp.ln_w[tid * 16 + i]), lp.s_u);
      }
      __syncthreads();   // lred reused by the next row; u codes visible
    }
    int8_t* zxw = const_cast<int8_t*>(a.zx);
    // rows of this warp, software-pipelined: the next row's weights and epilogue scales are in
    // flight while the current row is reduced
    const int nstep = G * (M1D_THREADS / 32);
    int n = blockIdx.x * (M1D_THREADS / 32) + warp;
    int4 wv[M1D_MAXKIN], wn[M1D_MAXKIN];
    float al = 0.f, cs = 1.f, aln = 0.f, csn = 1.f;
    auto load_row = [&](int row, int4 (&dst)[M1D_MAXKIN], float& a_, float& c_) {
      const int8_t* wr = lp.in_w + (int64_t)row * dm;
#pragma unroll
      for (int j = 0; j < M1D_MAXKIN; ++j)
        dst[j] = lane * 16 + j * 512 < dm ? __ldg(reinterpret_cast<const int4*>(wr + lane * 16 + j * 512))
                                          : make_int4(0, 0, 0, 0);
      a_ = __ldg(lp.in_alpha + row);
      c_ = __ldg(lp.in_cs + row);
    };
    if (n < 2 * di) load_row(n, wv, al, cs);
    for (; n < 2 * di; n += nstep) {
      if (n + nstep < 2 * di) load_row(n + nstep, wn, aln, csn);
      for (int b = 0; b < B; ++b) {
        int acc = 0;
#pragma unroll
        for (int j = 0; j < M1D_MAXKIN; ++j) {
          if (lane * 16 + j * 512 < dm) {
            const int4 x = *reinterpret_cast<const int4*>(us + (int64_t)b * dm + lane * 16 + j * 512);
            acc = __dp4a(wv[j].x, x.x, acc);
            acc = __dp4a(wv[j].y, x.y, acc);
            acc = __dp4a(wv[j].z, x.z, acc);
            acc = __dp4a(wv[j].w, x.w, acc);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) zxw[(int64_t)b * a.ldzx + n] = quant8(__fmul_rn((float)acc, al), cs);
      }
#pragma unroll
      for (int j = 0; j < M1D_MAXKIN; ++j) wv[j] = wn[j];
      al = aln;
      cs = csn;
    }
    M1D_MARK(9);
    grid_sync(bar);
  }

  // ---------------- phase 1: conv update (+ cache shift), one (sequence, channel) per thread
  for (int i = i1; i < B * di; i += gthreads) {
    const int b = i / di, c = i - b * di;
    if (i != i1) {
      csi = P.conv_s_in[c]; cso = P.conv_s_out[c]; cb = P.conv_b[c];
#pragma unroll
      for (int j = 0; j < 8; ++j) cw[j] = j < Kc ? P.conv_w[c * Kc + j] : 0.f;
    }
    int8_t* cr = a.cache + (int64_t)b * (Kc - 1) * di + c;
    int8_t q[8];
    for (int j = 0; j < Kc - 1; ++j) q[j] = cr[(int64_t)j * di];
    q[Kc - 1] = a.zx[(int64_t)b * a.ldzx + di + c];
    float acc = cb;
    for (int j = 0; j < Kc; ++j) acc = __fadd_rn(acc, __fmul_rn(cw[j], __fmul_rn((float)q[j], csi)));
    xc[(int64_t)b * di + c] = quant8(silu_f(acc), cso);
    for (int j = 0; j < Kc - 1; ++j) cr[(int64_t)j * di] = q[j + 1];
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  M1D_MARK(2);
  grid_sync(bar);
  M1D_MARK(3);

  // ---------------- phase 2: x_proj, one output row per warp (weights and xc from shared memory, dp4a)
  int8_t* xs = xs_base;   // xc [B x di] staged once per CTA
  if (blockIdx.x < NX) {   // CTA-uniform: the CTA owns at least one row
    for (int k = tid * 16; k < B * di; k += M1D_THREADS * 16) cp_async16_m1(xs + k, xc + k);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  for (int n = n2; n < NX; n += G * (M1D_THREADS / 32)) {
    const int8_t* wr = xw + (int64_t)((n - blockIdx.x) / G) * di;
    int acc[M1D_MAXB];
#pragma unroll
    for (int b = 0; b < M1D_MAXB; ++b) acc[b] = 0;
#pragma unroll 4
    for (int k = lane * 16; k < di; k += 32 * 16) {
      const int4 w = *reinterpret_cast<const int4*>(wr + k);
#pragma unroll
      for (int b = 0; b < M1D_MAXB; ++b) {
        if (b < B) {
          const int4 x = *reinterpret_cast<const int4*>(xs + (int64_t)b * di + k);
          acc[b] = __dp4a(w.x, x.x, acc[b]);
          acc[b] = __dp4a(w.y, x.y, acc[b]);
          acc[b] = __dp4a(w.z, x.z, acc[b]);
          acc[b] = __dp4a(w.w, x.w, acc[b]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < M1D_MAXB; ++b) {
      if (b < B) {
        int v = acc[b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0)
          xd[(int64_t)b * NX + n] = quant8(__fmul_rn((float)v, n == n2 ? xal : P.xproj_alpha[n]),
                                           n == n2 ? xcs : P.xproj_cs[n]);
      }
    }
  }
  M1D_MARK(4);
  grid_sync(bar);
  M1D_MARK(5);

  // ---------------- phase 3: dt_proj + scan step (a warp holds 4 whole channels: B * di % 4 == 0,
  // so the full-mask shuffles always see 32 lanes)
  for (int u = u3; (u & ~3) < B * di; u += gthreads / 8) {
    const int b = u / di, c = u - b * di;
    if (u != u3) {
      A0 = S.A[(int64_t)c * N + j8];
      A1 = S.A[(int64_t)c * N + j8 + 8];
      dtb = S.dt_bias[c]; sx = S.s_x[c]; sh = S.s_h[c]; Dc = S.D[c];
      dal = P.dtproj_alpha[c]; dcs = P.dtproj_cs[c];
      const int* wr = reinterpret_cast<const int*>(P.dtproj_w + (int64_t)c * R);
#pragma unroll
      for (int t = 0; t < M1D_MAXRW; ++t) dw[t] = j8 + 8 * t < nw4 ? __ldg(wr + j8 + 8 * t) : 0;
    }
    int8_t* st = a.state + ((int64_t)b * di + c) * N;
    const int8_t s0 = st[j8], s1 = st[j8 + 8];                   // issued ahead of the dt_proj chain
    const int8_t zc = a.zx[(int64_t)b * a.ldzx + c];
    const int8_t xcc = __ldcg(xc + (int64_t)b * di + c);
    const int* xr = reinterpret_cast<const int*>(xd + (int64_t)b * NX);
    int dacc = 0;
#pragma unroll
    for (int t = 0; t < M1D_MAXRW; ++t)
      if (j8 + 8 * t < nw4) dacc = __dp4a(dw[t], __ldcg(xr + j8 + 8 * t), dacc);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    const int8_t dcode = quant8(__fmul_rn((float)dacc, dal), dcs);
    // mamba1_step_kernel for states j8 and j8 + 8 of channel c
    const float delta = softplus_f(__fadd_rn(__fmul_rn((float)dcode, S.s_dt), dtb));
    const float xh = __fmul_rn((float)xcc, sx);
    const float dtx = __fmul_rn(delta, xh);
    const int8_t* bc = xd + (int64_t)b * NX + R;
    const float h0a = __fmul_rn((float)s0, sh), h0b = __fmul_rn((float)s1, sh);
    const float ha = __fadd_rn(__fmul_rn(expf(__fmul_rn(delta, A0)), h0a),
                               __fmul_rn(dtx, __fmul_rn((float)__ldcg(bc + j8), S.s_B)));
    const float hb = __fadd_rn(__fmul_rn(expf(__fmul_rn(delta, A1)), h0b),
                               __fmul_rn(dtx, __fmul_rn((float)__ldcg(bc + j8 + 8), S.s_B)));
    // the step kernel's 16-lane xor tree: level 8 pairs states n and n + 8 (here in one thread)
    float acc = __fmul_rn(ha, __fmul_rn((float)__ldcg(bc + N + j8), S.s_C)) +
                __fmul_rn(hb, __fmul_rn((float)__ldcg(bc + N + j8 + 8), S.s_C));
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    st[j8] = quant8(ha, sh);
    st[j8 + 8] = quant8(hb, sh);
    if (j8 == 0) {
      const float yv = __fadd_rn(acc, __fmul_rn(Dc, xh));
      y[(int64_t)b * di + c] = __fmul_rn(yv, silu_f(__fmul_rn((float)zc, S.s_z)));
    }
  }
  M1D_MARK(6);
  grid_sync(bar);
  M1D_MARK(7);
  pdl_trigger();   // every CTA is resident: out_proj may start its prologue

  // ---------------- phase 4: RMSNorm + FWHT (blocks of blk) + quant, one CTA per (sequence, block)
  __shared__ float hs[M1D_MAXBLK];
  __shared__ double red[M1D_THREADS / 32];
  constexpr int MAXV = 16;   // row values per thread (d_inner <= 8192)
  for (int jb = blockIdx.x; jb < B * nblk; jb += G) {
    const int b = jb / nblk, q = jb - b * nblk;
    const float* yr = y + (int64_t)b * di;
    float yv[MAXV];   // yv[k] = y[tid + k*512]; block q's elements are k = q*blk/512 + e
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) yv[k] = tid + k * M1D_THREADS < di ? __ldcg(yr + tid + k * M1D_THREADS) : 0.f;
#pragma unroll
    for (int k = 0; k < MAXV; ++k) ss += (double)yv[k] * (double)yv[k];
    ss = warp_sum_d(ss);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < M1D_THREADS / 32; ++w) tot += red[w];   // fixed order: every CTA of row b agrees
    const float r = rms_factor_m1(tot, di, P.eps);
    if (P.hadamard) {
      const int k0 = q * blk / M1D_THREADS;   // blk >= 512 here (else the smem index path below)
#pragma unroll
      for (int e = 0; e < M1D_MAXBLK / M1D_THREADS; ++e) {
        const int i = tid + e * M1D_THREADS;
        if (i < blk) {
          float v = 0.f;
#pragma unroll
          for (int k = 0; k < MAXV; ++k)
            if (k == k0 + e) v = yv[k];
          if (blk < M1D_THREADS) v = __ldcg(yr + q * blk + i);
          hs[i] = __fmul_rn(__fmul_rn(v, r), jb == blockIdx.x ? gw[e] : P.norm_w[q * blk + i]);
        }
      }
      int lg = 0;
      for (int h = 1; h < blk; h <<= 1, ++lg) {
        __syncthreads();
        for (int t = tid; t < blk / 2; t += M1D_THREADS) {
          const int i0 = ((t >> lg) << (lg + 1)) | (t & (h - 1)), i1 = i0 + h;
          const float v0 = hs[i0], v1 = hs[i1];
          hs[i0] = __fadd_rn(v0, v1);
          hs[i1] = __fsub_rn(v0, v1);
        }
      }
      __syncthreads();
      for (int i = tid; i < blk; i += M1D_THREADS) a.yq[(int64_t)b * a.ldyq + q * blk + i] = quant8(hs[i], P.s_y);
    } else {
      for (int i = tid; i < di; i += M1D_THREADS)
        a.yq[(int64_t)b * a.ldyq + i] = quant8(__fmul_rn(__fmul_rn(__ldcg(yr + i), r), P.norm_w[i]), P.s_y);
    }
    __syncthreads();   // red / hs reused by the next (sequence, block)
  }
  if (a.layer) {
    // ---------------- phase 5: out_proj rows, one per warp, over the yq codes staged in shared
    // memory; the GEMM's residual epilogue h += f32(acc) * alpha
    grid_sync(bar);
    const sq_mamba1_layer_params& lp = a.lp;
    const int dm = lp.d_model;
    int8_t* ys = xs_base;   // xc staging and u codes are dead: stage yq [B x di] over them
    for (int k = tid * 16; k < B * di; k += M1D_THREADS * 16) cp_async16_m1(ys + k, a.yq + k);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int n = blockIdx.x * (M1D_THREADS / 32) + warp; n < dm; n += G * (M1D_THREADS / 32)) {
      const int8_t* wr = lp.out_w + (int64_t)n * di;
      const float oal = __ldg(lp.out_alpha + n);
      float hv[M1D_MAXB];
#pragma unroll
      for (int b = 0; b < M1D_MAXB; ++b) hv[b] = (lane == 0 && b < B) ? a.h[(int64_t)b * a.ldh + n] : 0.f;
      int4 wv[M1D_MAXK16];
#pragma unroll
      for (int j = 0; j < M1D_MAXK16; ++j)
        wv[j] = lane * 16 + j * 512 < di ? __ldg(reinterpret_cast<const int4*>(wr + lane * 16 + j * 512))
                                         : make_int4(0, 0, 0, 0);
      for (int b = 0; b < B; ++b) {
        int acc = 0;
#pragma unroll
        for (int j = 0; j < M1D_MAXK16; ++j) {
          if (lane * 16 + j * 512 < di) {
            const int4 x = *reinterpret_cast<const int4*>(ys + (int64_t)b * di + lane * 16 + j * 512);
            acc = __dp4a(wv[j].x, x.x, acc);
            acc = __dp4a(wv[j].y, x.y, acc);
            acc = __dp4a(wv[j].z, x.z, acc);
            acc = __dp4a(wv[j].w, x.w, acc);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
          float hb = hv[0];
#pragma unroll
          for (int bb = 1; bb < M1D_MAXB; ++bb)
            if (bb == b) hb = hv[bb];
          a.h[(int64_t)b * a.ldh + n] = __fadd_rn(hb, __fmul_rn((float)acc, oal));
        }
      }
    }
  }
  M1D_MARK(8);
}

}  // namespace sq

using namespace sq;

extern "C" int64_t sq_mamba1_decode_ws_bytes(const sq_mamba1_decode_params* p, int B) {
  if (!p || B < 0) return -1;
  return M1Ws(B, p->ssm.d_inner, p->dt_rank + 2 * p->ssm.d_state).total;
}

extern "C" int sq_mamba1_decode_step_int8(const sq_mamba1_decode_params* p, int B, const int8_t* zx, int64_t ldzx,
                                          int8_t* conv_cache, int8_t* state, void* ws, int8_t* yq, int64_t ldyq,
                                          void* stream) {
  SQ_REQUIRE(p && B >= 0, SQ_ERR_ARG, "sq_mamba1_decode_step_int8: bad args");
  if (B == 0) return SQ_OK;
  const int di = p->ssm.d_inner, R = p->dt_rank;
  const int blk = p->hadamard ? (di & -di) : di;
  SQ_REQUIRE(p->ssm.d_state == 16 && B <= M1D_MAXB && di % 16 == 0 && di <= 8192 && R % 4 == 0 && R > 0 &&
                 p->conv_kernel >= 1 &&
                 p->conv_kernel <= 8 && (!p->hadamard || blk <= M1D_MAXBLK),
             SQ_ERR_SHAPE, "sq_mamba1_decode_step_int8: unsupported shape (d_state 16, B <= 8, d_inner %% 16, "
             "dt_rank %% 4, Hadamard block <= 4096)");
  SQ_REQUIRE(!((reinterpret_cast<uintptr_t>(p->xproj_w) | reinterpret_cast<uintptr_t>(p->dtproj_w) |
                reinterpret_cast<uintptr_t>(ws)) & 15),
             SQ_ERR_LAYOUT, "sq_mamba1_decode_step_int8: weights / workspace must be 16-B aligned");
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (sms[dev & 63] == 0) cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  const int G = sms[dev & 63];
  const int nx = R + 2 * p->ssm.d_state;
  const size_t smem = (size_t)((nx + G - 1) / G) * di + (size_t)B * di;   // x_proj rows of one CTA + xc
  SQ_REQUIRE(smem <= 160 * 1024 && R / 4 <= 8 * M1D_MAXRW, SQ_ERR_SHAPE,
             "sq_mamba1_decode_step_int8: x_proj rows per CTA exceed shared memory");
  static std::once_flag once[64];
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(mamba1_decode_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  });
  M1DecodeArgs a{*p, B, zx, ldzx, conv_cache, state, reinterpret_cast<uint8_t*>(ws), yq, ldyq, 0, {}, nullptr, 0};
  launch_k(PDL_SMALL8, mamba1_decode_fused_kernel, dim3(G), dim3(M1D_THREADS), smem, as_stream(stream), a);
  return check_launch("sq_mamba1_decode_step_int8");
}

extern "C" int sq_mamba1_decode_layer_int8(const sq_mamba1_decode_params* p, const sq_mamba1_layer_params* lp, int B,
                                           float* h, int64_t ldh, int8_t* conv_cache, int8_t* state, void* ws,
                                           void* stream) {
  SQ_REQUIRE(p && lp && h && B >= 0, SQ_ERR_ARG, "sq_mamba1_decode_layer_int8: bad args");
  if (B == 0) return SQ_OK;
  const int di = p->ssm.d_inner, R = p->dt_rank, dm = lp->d_model;
  const int blk = p->hadamard ? (di & -di) : di;
  SQ_REQUIRE(p->ssm.d_state == 16 && B <= M1D_MAXB && di % 16 == 0 && di <= 8192 && R % 4 == 0 && R > 0 &&
                 p->conv_kernel >= 1 && p->conv_kernel <= 8 && (!p->hadamard || blk <= M1D_MAXBLK) &&
                 dm % 16 == 0 && dm / 16 <= M1D_THREADS && dm <= 512 * M1D_MAXKIN && di <= 512 * M1D_MAXK16 &&
                 ldh % 4 == 0,
             SQ_ERR_SHAPE, "sq_mamba1_decode_layer_int8: unsupported shape");
  SQ_REQUIRE(!((reinterpret_cast<uintptr_t>(p->xproj_w) | reinterpret_cast<uintptr_t>(p->dtproj_w) |
                reinterpret_cast<uintptr_t>(lp->in_w) | reinterpret_cast<uintptr_t>(lp->out_w) |
                reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(ws)) & 15),
             SQ_ERR_LAYOUT, "sq_mamba1_decode_layer_int8: weights / h / workspace must be 16-B aligned");
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (sms[dev & 63] == 0) cudaDeviceGetAttribute(&sms[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  const int G = sms[dev & 63];
  const int nx = R + 2 * p->ssm.d_state;
  const M1Ws L(B, di, nx);
  // x_proj rows + xc staging + u codes; phase 5 stages yq over the last two
  const size_t smem = (size_t)((nx + G - 1) / G) * di + (size_t)B * di + (size_t)B * dm;
  SQ_REQUIRE(smem <= 160 * 1024, SQ_ERR_SHAPE, "sq_mamba1_decode_layer_int8: shared memory");
  static std::once_flag once[64];
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(mamba1_decode_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  });
  uint8_t* w8 = reinterpret_cast<uint8_t*>(ws);
  M1DecodeArgs a{*p, B, reinterpret_cast<const int8_t*>(w8 + L.zx), 2 * di, conv_cache, state, w8,
                 reinterpret_cast<int8_t*>(w8 + L.yq), di, 1, *lp, h, ldh};
  launch_k(PDL_SMALL8, mamba1_decode_fused_kernel, dim3(G), dim3(M1D_THREADS), smem, as_stream(stream), a);
  return check_launch("sq_mamba1_decode_layer_int8");
}
