// k_averis.cu — the Averis mean-residual NVFP4 forward GeMM (PAPER.md:391-429,
// Eq. averis_forward; format PAPER.md:488-491) behind include/avd_averis.h.
//
//   Y_hat = 1 (mu_bar W_bar) + X_R_bar W_bar,  X_R = X - 1 mu_X,  bar = NVFP4 Q_b
//
// Kernels (one forward = 6 launches, all on the context's stream):
//   av_colstats_kernel   HBM: column sums (fp64), max, min of X over row chunks
//   av_reduce_kernel     mu_X = sum / l (fp64), mu_f = fl32(mu), per-column amax of X_R from the
//                        column max / min (fl32 subtraction is monotone, so this is max |x_r|
//                        exactly), tensor amax by atomicMax on the bit patterns
//   av_quant_kernel      Q_b: x_r = fl32(x - mu_f), per 16-block amax, UE4M3 scale (cvt.rn.satfinite),
//                        E2M1 codes (cvt.rn.satfinite.e2m1x2 for nearest; counter-hash stochastic
//                        rounding in fp32 otherwise), codes packed K-major (tensor-core A / B
//                        operand), scales written straight into the tcgen05 scale-factor layout
//   av_bias_kernel       mu_bar W_bar: exact integer dot of the codes per 16-block, fp64 sum
//   av_gemm_kernel       X_R_bar W_bar^T on tcgen05.mma kind::mxf4nvf4 (block16 UE4M3 scales in TMEM
//                        via tcgen05.cp), fp32 TMEM accumulators (double-buffered), epilogue
//                        y = acc * g_X g_W + bias_j
// The decision arithmetic follows DESIGN.md readings A1-A8 in the same fp32 order as the oracle
// (oracle/averis.py) — which this file never includes or calls.
#include <cudaTypedefs.h>
#include <algorithm>
#include <vector>
#include "../../include/avd_averis.h"
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // k_gram.cu

struct AvCtx {
  avd_averis_config cfg{};
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t l = 0, m = 0, n = 0, l_pad = 0, n_pad = 0;
  int64_t kb4 = 0;  // 64-element scale chunks per 128-row tile (4 per 256-element stage, padded)
  int R = 1;        // row chunks of the column statistics
  int64_t launches = 0;
  bool weight_set = false;
  bool vanilla = false, sr = false, bf16_out = false;
  double* csum_part = nullptr;   // [R][m]
  float* cmax_part = nullptr;    // [R][m]
  float* cmin_part = nullptr;    // [R][m]
  double* mu = nullptr;          // [m]
  float* mu_f = nullptr;         // [m]
  uint8_t* xcodes = nullptr;     // [l_pad][m/2]
  uint8_t* xsf = nullptr;        // l_pad * kb4 * 4
  uint8_t* wcodes = nullptr;     // [n_pad][m/2]
  uint8_t* wsf = nullptr;        // n_pad * kb4 * 4
  uint8_t* mucodes = nullptr;    // [m/2]
  uint8_t* musf = nullptr;       // [m/16]
  float* gsc = nullptr;          // [8]: g_X, g_W, g_mu, amax_X, amax_W, amax_mu
  float* bias = nullptr;         // [n]
  CUtensorMap tmA{}, tmB{}, tmSA{}, tmSB{};
  float* X_stage = nullptr;
  void* Y_stage = nullptr;
  std::vector<void*> allocs;
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // AVD_AVERIS_TIMING: stage boundaries
};

namespace {
using namespace sm100;

// ---------------------------------------------------------------- number formats (A1-A3)
__device__ __forceinline__ uint32_t e4m3_rn(float s) {  // UE4M3 code of s >= 0, RNE, saturating at 448
  uint16_t h;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(h) : "f"(0.f), "f"(s));
  return h & 0xFFu;
}
__device__ __forceinline__ float e4m3_val(uint32_t c) {
  const uint32_t e = c >> 3, f = c & 7u;
  return e == 0 ? (float)f * 0.001953125f : __uint_as_float(((e + 120u) << 23) | (f << 20));
}
// two fp32 values -> one byte of E2M1 codes (lo -> low nibble), round to nearest even, saturating
__device__ __forceinline__ uint32_t e2m1x2_rn(float lo, float hi) {
  uint32_t r;
  asm("{\n\t.reg .b8 b;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b, %1, %2;\n\t"
      "cvt.u32.u8 %0, b;\n\t}"
      : "=r"(r)
      : "f"(hi), "f"(lo));
  return r;
}
// counter hash (A3): splitmix64 finaliser of idx + tid * golden + seed * c2, top 24 bits
__device__ __forceinline__ uint32_t ctr_u24(uint64_t seed, uint64_t tid, uint64_t idx) {
  uint64_t z = idx + tid * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (uint32_t)(z >> 40);
}
// stochastic rounding on the E2M1 grid: up with probability (|v| - g_lo) / (g_hi - g_lo), decided
// as u24 < frac * 2^24 (both sides exact in fp32)
__device__ __forceinline__ uint32_t e2m1_sr(float v, uint32_t u24) {
  const float a = fminf(fabsf(v), 6.f);
  const int lo = (a >= 0.5f) + (a >= 1.f) + (a >= 1.5f) + (a >= 2.f) + (a >= 3.f) + (a >= 4.f) + (a >= 6.f);
  const float glo = lo <= 4 ? 0.5f * (float)lo : (lo == 5 ? 3.f : (lo == 6 ? 4.f : 6.f));
  const float inv_gap = lo < 4 ? 2.f : (lo < 6 ? 1.f : 0.5f);
  const float frac = __fmul_rn(__fsub_rn(a, glo), inv_gap);
  const uint32_t up = (lo < 7 && (float)u24 < __fmul_rn(frac, 16777216.f)) ? 1u : 0u;
  return ((__float_as_uint(v) >> 31) << 3) | (uint32_t)(lo + (int)up);
}
__device__ __forceinline__ float tensor_g(float amax) {  // g = fl32(amax / 2688), 1 when 0 (A2)
  const float g = __fdiv_rn(amax, 2688.f);
  return g == 0.f ? 1.f : g;
}
// byte offset of the scale of (row r, 16-block b) in the tcgen05 scale-factor layout: 128-row tiles
// of 64-element chunks, 512 B each = 32 lanes x (4 row quarters x 4 blocks)
__device__ __forceinline__ int64_t sf_off(int64_t r, int64_t b, int64_t kb4) {
  return ((r >> 7) * kb4 + (b >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (b & 3);
}

// ---------------------------------------------------------------- column statistics
__global__ void __launch_bounds__(256) av_colstats_kernel(const float* __restrict__ X, int64_t l, int64_t m,
                                                          int64_t rows_per, double* __restrict__ csum,
                                                          float* __restrict__ cmax, float* __restrict__ cmin) {
  const int64_t j = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
  if (j >= m) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(l, r0 + rows_per);
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  float4 mx = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  float4 mn = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(X + (r + u) * m + j));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s0 += v[u].x; s1 += v[u].y; s2 += v[u].z; s3 += v[u].w;
      mx.x = fmaxf(mx.x, v[u].x); mx.y = fmaxf(mx.y, v[u].y); mx.z = fmaxf(mx.z, v[u].z); mx.w = fmaxf(mx.w, v[u].w);
      mn.x = fminf(mn.x, v[u].x); mn.y = fminf(mn.y, v[u].y); mn.z = fminf(mn.z, v[u].z); mn.w = fminf(mn.w, v[u].w);
    }
  }
  for (; r < r1; ++r) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(X + r * m + j));
    s0 += v.x; s1 += v.y; s2 += v.z; s3 += v.w;
    mx.x = fmaxf(mx.x, v.x); mx.y = fmaxf(mx.y, v.y); mx.z = fmaxf(mx.z, v.z); mx.w = fmaxf(mx.w, v.w);
    mn.x = fminf(mn.x, v.x); mn.y = fminf(mn.y, v.y); mn.z = fminf(mn.z, v.z); mn.w = fminf(mn.w, v.w);
  }
  const int64_t o = (int64_t)blockIdx.y * m + j;
  csum[o] = s0; csum[o + 1] = s1; csum[o + 2] = s2; csum[o + 3] = s3;
  *reinterpret_cast<float4*>(cmax + o) = mx;
  *reinterpret_cast<float4*>(cmin + o) = mn;
}

// mu (fixed-order sum of the row-chunk partials), mu_f, and the tensor amax of X_R and of mu_f.
// CTA = 32 columns x 8 partial-row groups: thread (g, c) sums the partials y = g (mod 8) of column
// c (coalesced 32-column rows), the 8 group sums are combined in a fixed order in shared memory.
__global__ void __launch_bounds__(256) av_reduce_kernel(const double* __restrict__ csum, const float* __restrict__ cmax,
                                                        const float* __restrict__ cmin, int R, int64_t l, int64_t m,
                                                        int vanilla, double* __restrict__ mu, float* __restrict__ mu_f,
                                                        float* __restrict__ gsc) {
  __shared__ double s_s[8][32];
  __shared__ float s_x[8][32], s_n[8][32];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + c;
  double s = 0;
  float mx = -INFINITY, mn = INFINITY;
  if (j < m) {
    for (int y = g; y < R; y += 8) {
      s += csum[(int64_t)y * m + j];
      mx = fmaxf(mx, cmax[(int64_t)y * m + j]);
      mn = fminf(mn, cmin[(int64_t)y * m + j]);
    }
  }
  s_s[g][c] = s; s_x[g][c] = mx; s_n[g][c] = mn;
  __syncthreads();
  if (g != 0) return;
  float a = 0.f, am = 0.f;
  if (j < m) {
    for (int h = 1; h < 8; ++h) { s += s_s[h][c]; mx = fmaxf(mx, s_x[h][c]); mn = fminf(mn, s_n[h][c]); }
    const double u = vanilla ? 0.0 : s / (double)l;
    const float uf = (float)u;
    mu[j] = u;
    mu_f[j] = uf;
    a = fmaxf(fabsf(__fsub_rn(mx, uf)), fabsf(__fsub_rn(mn, uf)));
    am = fabsf(uf);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
    am = fmaxf(am, __shfl_xor_sync(0xFFFFFFFFu, am, o));
  }
  if (c == 0) {
    atomicMax(reinterpret_cast<unsigned*>(gsc + 3), __float_as_uint(a));
    atomicMax(reinterpret_cast<unsigned*>(gsc + 5), __float_as_uint(am));
  }
}

__global__ void __launch_bounds__(256) av_amax_kernel(const float* __restrict__ A, int64_t count, float* __restrict__ dst) {
  float a = 0.f;
  for (int64_t i = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4; i < count; i += (int64_t)gridDim.x * 1024) {
    const float4 v = *reinterpret_cast<const float4*>(A + i);
    a = fmaxf(a, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned*>(dst), __float_as_uint(a));
}

// ---------------------------------------------------------------- quantiser Q_b
// Rows of a K-contiguous source (X_R, mu).  A CTA walks whole rows (grid-stride); per pass over a
// row its 256 threads cover 256 blocks of 16: four threads per block (one float4 each) and kU
// blocks per thread whose loads are issued first (a warp reads 512 contiguous bytes per load
// instruction).  The per-block scale decision (an IEEE division and reciprocal) is taken once per
// block: quad member u decides block u of the quad's kU blocks and broadcasts it.  sf_plain: scales
// in plain order (mu) instead of the tensor-core layout.
constexpr int kU = 4;
template <bool SR>
__global__ void __launch_bounds__(256) av_quant_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t K,
                                                            const float* __restrict__ mu_f, const float* __restrict__ amax_p,
                                                            float* __restrict__ g_out, uint8_t* __restrict__ codes,
                                                            uint8_t* __restrict__ sf, int64_t kb4, int sf_plain,
                                                            uint64_t seed, uint64_t tid) {
  static_assert(kU == 4, "one quad member per block of the quad");
  const int nb = (int)(K >> 4);
  const int lane = threadIdx.x & 31, qd = lane & 3;
  const int bw = (int)(threadIdx.x >> 5) * 32 + (lane >> 2);  // + 8 u: this thread's blocks in a pass
  const float g = tensor_g(*amax_p);
  if (blockIdx.x == 0 && threadIdx.x == 0 && g_out) *g_out = g;
  const float d6 = __fmul_rn(6.f, g);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* xr = src + r * K;
    for (int b0 = 0; b0 < nb; b0 += 256) {
      float4 x[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int b = b0 + bw + 8 * u;
        x[u] = b < nb ? __ldcs(reinterpret_cast<const float4*>(xr + b * 16 + qd * 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float am[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int b = b0 + bw + 8 * u;
        if (mu_f && b < nb) {
          const float4 mu = __ldg(reinterpret_cast<const float4*>(mu_f + b * 16 + qd * 4));
          x[u].x = __fsub_rn(x[u].x, mu.x); x[u].y = __fsub_rn(x[u].y, mu.y);
          x[u].z = __fsub_rn(x[u].z, mu.z); x[u].w = __fsub_rn(x[u].w, mu.w);
        }
        float a = fmaxf(fmaxf(fabsf(x[u].x), fabsf(x[u].y)), fmaxf(fabsf(x[u].z), fabsf(x[u].w)));
        a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, 1));
        am[u] = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, 2));
      }
      // quad member qd decides block u = qd
      const float amine = qd == 0 ? am[0] : (qd == 1 ? am[1] : (qd == 2 ? am[2] : am[3]));
      const uint32_t scm = e4m3_rn(__fdiv_rn(amine, d6));
      const float Rm = scm ? __frcp_rn(__fmul_rn(e4m3_val(scm), g)) : 0.f;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int b = b0 + bw + 8 * u;
        const int src_lane = (lane & ~3) | u;
        const uint32_t sc = __shfl_sync(0xFFFFFFFFu, scm, src_lane);
        const float R = __shfl_sync(0xFFFFFFFFu, Rm, src_lane);
        const float v0 = __fmul_rn(x[u].x, R), v1 = __fmul_rn(x[u].y, R), v2 = __fmul_rn(x[u].z, R), v3 = __fmul_rn(x[u].w, R);
        uint32_t out;
        if (SR) {
          const uint64_t li = (uint64_t)(r * K + b * 16 + qd * 4);
          out = e2m1_sr(v0, ctr_u24(seed, tid, li)) | (e2m1_sr(v1, ctr_u24(seed, tid, li + 1)) << 4) |
                (e2m1_sr(v2, ctr_u24(seed, tid, li + 2)) << 8) | (e2m1_sr(v3, ctr_u24(seed, tid, li + 3)) << 12);
        } else {
          out = e2m1x2_rn(v0, v1) | (e2m1x2_rn(v2, v3) << 8);
        }
        if (sc == 0) out = 0;  // all-zero block (A7)
        if (b < nb) {
          *reinterpret_cast<uint16_t*>(codes + r * (K >> 1) + b * 8 + qd * 2) = (uint16_t)out;
          if (qd == 0) sf[sf_plain ? (int64_t)b : sf_off(r, b, kb4)] = (uint8_t)sc;
        }
      }
    }
  }
}

// Columns of a row-major W [K][N] (blocks of 16 along K = m for each output column j): one thread
// per (j, block), j fastest (coalesced column reads); codes written as row j of [N][K/2].
template <bool SR>
__global__ void __launch_bounds__(256) av_quant_cols_kernel(const float* __restrict__ W, int64_t K, int64_t N,
                                                            const float* __restrict__ amax_p, float* __restrict__ g_out,
                                                            uint8_t* __restrict__ codes, uint8_t* __restrict__ sf,
                                                            int64_t kb4, uint64_t seed, uint64_t tid) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t nb = K >> 4;
  if (t >= N * nb) return;
  const int64_t j = t % N, b = t / N;
  const float g = tensor_g(*amax_p);
  if (t == 0 && g_out) *g_out = g;
  float x[16];
  float a = 0.f;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    x[u] = W[(b * 16 + u) * N + j];
    a = fmaxf(a, fabsf(x[u]));
  }
  const uint32_t sc = e4m3_rn(__fdiv_rn(a, __fmul_rn(6.f, g)));
  uint32_t w[2] = {0u, 0u};
  if (sc != 0) {
    const float R = __frcp_rn(__fmul_rn(e4m3_val(sc), g));
#pragma unroll
    for (int u = 0; u < 16; u += 2) {
      const float v0 = __fmul_rn(x[u], R), v1 = __fmul_rn(x[u + 1], R);
      uint32_t byte;
      if (SR) {
        byte = e2m1_sr(v0, ctr_u24(seed, tid, (uint64_t)((b * 16 + u) * N + j))) |
               (e2m1_sr(v1, ctr_u24(seed, tid, (uint64_t)((b * 16 + u + 1) * N + j))) << 4);
      } else {
        byte = e2m1x2_rn(v0, v1);
      }
      w[u >> 3] |= byte << (8 * ((u >> 1) & 3));
    }
  }
  *reinterpret_cast<uint2*>(codes + j * (K >> 1) + b * 8) = make_uint2(w[0], w[1]);
  sf[sf_off(j, b, kb4)] = (uint8_t)sc;
}

// ---------------------------------------------------------------- bias = mu_bar W_bar
__device__ __forceinline__ int e2m1_x2(uint32_t c) {  // 2 * E2M1 value (an integer)
  const int mag = (int)((0xC8643210u >> (4 * (c & 7u))) & 0xFu);  // 0,1,2,3,4,6,8,12
  return (c & 8u) ? -mag : mag;
}
__global__ void __launch_bounds__(256) av_bias_kernel(const uint8_t* __restrict__ mucodes, const uint8_t* __restrict__ musf,
                                                      const uint8_t* __restrict__ wcodes, const uint8_t* __restrict__ wsf,
                                                      const float* __restrict__ gsc, int64_t K, int64_t N, int64_t kb4,
                                                      float* __restrict__ bias) {
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= N) return;
  const int64_t nb = K >> 4;
  double acc = 0.0;
  for (int64_t b = lane; b < nb; b += 32) {
    const uint2 cm = *reinterpret_cast<const uint2*>(mucodes + b * 8);
    const uint2 cw = *reinterpret_cast<const uint2*>(wcodes + j * (K >> 1) + b * 8);
    int dot = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dot += e2m1_x2((cm.x >> (4 * u)) & 15u) * e2m1_x2((cw.x >> (4 * u)) & 15u);
      dot += e2m1_x2((cm.y >> (4 * u)) & 15u) * e2m1_x2((cw.y >> (4 * u)) & 15u);
    }
    acc += 0.25 * (double)dot * (double)e4m3_val(musf[b]) * (double)e4m3_val(wsf[sf_off(j, b, kb4)]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if (lane == 0) bias[j] = (float)(acc * (double)gsc[2] * (double)gsc[1]);
}

// ---------------------------------------------------------------- NVFP4 GeMM on tcgen05
// Y[i][j] = g_X g_W sum_k xr_ik w_kj + bias_j: A = X_R codes [l][m/2] (K-major), B = W codes
// [n][m/2] (K-major).  CTA pairs (cluster 2x1) own 256 x 256 output blocks with
// tcgen05.mma.cta_group::2.kind::mxf4nvf4 (M = 256: 128 A rows per CTA; N = 256: each CTA stages
// one 128-row half of B, so no operand byte is held twice), issued by the leader CTA.  K advances in
// stages of 256 elements (128 B of codes per row: one SWIZZLE_128B atom), 4 MMAs of K = 64 per
// stage; per stage each CTA receives 38 KB (A 16, B half 16, its A scales 2, all 256 B-row scales
// 4 — the scale chunks come as 2 KB TMA boxes of the quantiser's tensor-core layout) and every TMA
// completes on the leader's barrier.  The leader copies each CTA's scales to its own TMEM
// (tcgen05.cp.cta_group::2 32x128b.warpx4: 32 lanes x 16 B broadcast to the four lane quarters)
// ahead of the MMAs in issue order, and its commits arrive on both CTAs' barriers.  One fp32
// accumulator of 256 columns per CTA: eight epilogue warps per CTA drain it to registers (128
// values per thread), release it, apply y = acc * g_X g_W + bias_j while the next tile's MMAs run,
// and write Y by TMA bulk stores of 32 x 32 blocks staged in a 128B-swizzled buffer per warp
// (row-per-thread global stores cost about as much as the MMAs in L2 sector traffic).
constexpr uint32_t kAvA = 128 * 128, kAvB = 128 * 128, kAvSFA = 2048, kAvSFB = 4096;
constexpr uint32_t kAvStage = kAvA + kAvB + kAvSFA + kAvSFB;  // 38 KB per CTA (multiple of 1 KB)
constexpr uint32_t kAvOut = 32 * 128;                         // per epilogue warp: 32 rows x 32 fp32 (SW128)
constexpr int kAvGemmThreads = 320;                           // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue

// kind::mxf4nvf4, A/B E2M1 (format 1), UE4M3 scales (bit 23 = 0), K-major, K = 64
__host__ __device__ constexpr uint32_t idesc_nvf4(uint32_t M, uint32_t N) {
  return (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_nvf4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                              uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.scale_vec::4X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_sf_pair(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ uint32_t av_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void av_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t av_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void av_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// 2-D TMA load into this CTA's shared memory, completion counted on the leader's barrier
__device__ __forceinline__ void tma_load_2d_p(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int32_t c0,
                                              int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)),
               "r"(bar_cluster), "r"(c0), "r"(c1)
               : "memory");
}
// arrive on `bar` in both CTAs of the pair once the leader's previously issued MMAs completed
__device__ __forceinline__ void mma_commit_pair_mc(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {  // RNE, lo in the low half
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%"
      "29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

constexpr int kAvNS = 5;
template <bool BF>  // BF: Y in bf16 (RNE), else fp32
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kAvGemmThreads, 1) av_gemm_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
    const __grid_constant__ CUtensorMap tmSA, const __grid_constant__ CUtensorMap tmSB,
    const __grid_constant__ CUtensorMap tmY, int64_t l, int64_t n, int KB, int64_t MT2, int64_t NT, int64_t kb4,
    const float* __restrict__ gsc, const float* __restrict__ bias) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kAvNS], empty_bar[kAvNS], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_sh;
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = av_cluster_rank();
  const int64_t pairs = MT2 * NT;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int64_t st4 = kb4 / 4;  // 2 KB scale chunks per 128-row tile
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAvNS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 16);  // 8 epilogue warps x 2 CTAs (on the leader)
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA); tma_prefetch(&tmB); tma_prefetch(&tmSA); tma_prefetch(&tmSB); tma_prefetch(&tmY);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  av_cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  const uint32_t full0 = av_mapa(smem_u32(&full_bar[0]), 0);   // the leader's full barriers
  const uint32_t tempty0 = av_mapa(smem_u32(&tempty_bar), 0);  // the leader's tempty barrier

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int64_t pt = cid; pt < pairs; pt += ncl) {
        const int64_t mt = 2 * (pt / NT) + rank, nt = pt % NT;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % kAvNS, ph = (it / kAvNS) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kAvStage;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * kAvStage);
          const uint32_t fb = full0 + s * (uint32_t)sizeof(uint64_t);
          tma_load_2d_p(st, &tmA, fb, kb * 128, (int32_t)(mt * 128));
          tma_load_2d_p(st + kAvA, &tmB, fb, kb * 128, (int32_t)(nt * 256 + rank * 128));
          tma_load_2d_p(st + kAvA + kAvB, &tmSA, fb, 0, (int32_t)(mt * st4 + kb));
          tma_load_2d_p(st + kAvA + kAvB + kAvSFA, &tmSB, fb, 0, (int32_t)(2 * nt * st4 + kb));
          tma_load_2d_p(st + kAvA + kAvB + 2 * kAvSFA, &tmSB, fb, 0, (int32_t)((2 * nt + 1) * st4 + kb));
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_nvf4(256, 256);
      uint32_t it = 0, ui = 0;
      for (int64_t pt = cid; pt < pairs; pt += ncl, ++ui) {
        mbar_wait(&tempty_bar, (ui & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % kAvNS, ph = (it / kAvNS) & 1;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t base = smem_u32(smem + s * kAvStage);
            const uint32_t sfa_s = base + kAvA + kAvB, sfb_s = sfa_s + kAvSFA;
            const uint32_t tsf = tmem + 256 + (it & 3) * 48;  // 4 rotating slots: SFA 16 columns, SFB 32
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              tmem_cp_sf_pair(tsf + kk * 4, smem_desc(sfa_s + kk * 512, 0, 128, 0));
              tmem_cp_sf_pair(tsf + 16 + kk * 8, smem_desc(sfb_s + kk * 512, 0, 128, 0));
              tmem_cp_sf_pair(tsf + 16 + kk * 8 + 4, smem_desc(sfb_s + kAvSFA + kk * 512, 0, 128, 0));
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = smem_desc(base + kk * 32, 16, 1024, 2);
              const uint64_t bd = smem_desc(base + kAvA + kk * 32, 16, 1024, 2);
              mma_nvf4_pair(tmem, ad, bd, idesc, tsf + kk * 4, tsf + 16 + kk * 8, (kb | kk) ? 1u : 0u);
            }
            mma_commit_pair_mc(&empty_bar[s]);
          }
          __syncwarp();
        }
        if (elect_one()) mma_commit_pair_mc(&tfull_bar);
        __syncwarp();
      }
    }
  } else {
    const uint32_t q = warp & 3, h = (warp - 2) >> 2;
    const float gxw = __fmul_rn(gsc[0], gsc[1]);
    uint32_t ui = 0;
    for (int64_t pt = cid; pt < pairs; pt += ncl, ++ui) {
      const int64_t mt = 2 * (pt / NT) + rank, nt = pt % NT;
      mbar_wait(&tfull_bar, ui & 1);
      tc_fence_after();
      uint32_t v[128];
      const uint32_t tb = tmem + ((q * 32) << 16) + h * 128;
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tb + c * 32, v + c * 32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) av_arrive_remote(tempty0);
      const int64_t row0 = mt * 128 + q * 32;
      const int64_t col0 = nt * 256 + h * 128;
      if (row0 < l) {
        const uint32_t sw = lane & 7;
        // per store: 32 rows x 128 B (32 fp32 or 64 bf16 columns), 128B-swizzled
        constexpr int CW = BF ? 64 : 32;
#pragma unroll
        for (int c = 0; c < 128 / CW; ++c) {
          if (col0 + CW * c >= n) break;
          uint8_t* ob = smem + kAvNS * kAvStage + (warp - 2) * kAvOut;
          if (lane == 0) bulk_wait_read0();  // the previous block's bulk store has read the buffer
          __syncwarp();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if constexpr (BF) {
              const int cc = 64 * c + 8 * k;
              float y[8];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const float4 bb = col0 + cc + 4 * hh < n ? __ldg(reinterpret_cast<const float4*>(bias + col0 + cc + 4 * hh))
                                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                y[4 * hh] = __fmaf_rn(__uint_as_float(v[cc + 4 * hh]), gxw, bb.x);
                y[4 * hh + 1] = __fmaf_rn(__uint_as_float(v[cc + 4 * hh + 1]), gxw, bb.y);
                y[4 * hh + 2] = __fmaf_rn(__uint_as_float(v[cc + 4 * hh + 2]), gxw, bb.z);
                y[4 * hh + 3] = __fmaf_rn(__uint_as_float(v[cc + 4 * hh + 3]), gxw, bb.w);
              }
              uint4 pk;
              pk.x = bf16x2(y[0], y[1]); pk.y = bf16x2(y[2], y[3]); pk.z = bf16x2(y[4], y[5]); pk.w = bf16x2(y[6], y[7]);
              *reinterpret_cast<uint4*>(ob + lane * 128 + ((k ^ sw) << 4)) = pk;
            } else {
              const int cc = 32 * c + 4 * k;
              const float4 bb = col0 + cc < n ? __ldg(reinterpret_cast<const float4*>(bias + col0 + cc))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
              const float4 y = make_float4(__fmaf_rn(__uint_as_float(v[cc]), gxw, bb.x),
                                           __fmaf_rn(__uint_as_float(v[cc + 1]), gxw, bb.y),
                                           __fmaf_rn(__uint_as_float(v[cc + 2]), gxw, bb.z),
                                           __fmaf_rn(__uint_as_float(v[cc + 3]), gxw, bb.w));
              *reinterpret_cast<float4*>(ob + lane * 128 + ((k ^ sw) << 4)) = y;
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tma_store_2d(&tmY, ob, (int32_t)(col0 + CW * c), (int32_t)row0);
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  av_cluster_sync();  // no CTA leaves while its peer may still load into it / arrive on it
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

avd_status make_maps(AvCtx* c) {
  auto enc = tma_encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return AVD_ECUDA; }
  uint32_t box[2] = {128, 128}, es[2] = {1, 1};
  uint64_t strides[1] = {(uint64_t)(c->m / 2)};
  uint64_t da[2] = {(uint64_t)(c->m / 2), (uint64_t)c->l};
  CUresult r = enc(&c->tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->xcodes, da, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (Averis A) failed: " + std::to_string((int)r)); return AVD_ECUDA; }
  uint64_t db[2] = {(uint64_t)(c->m / 2), (uint64_t)c->n};
  r = enc(&c->tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->wcodes, db, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (Averis B) failed: " + std::to_string((int)r)); return AVD_ECUDA; }
  // scale chunks: 2 KB boxes (256 x u64) of the tensor-core layout, one per (128-row tile, stage)
  uint32_t sbox[2] = {256, 1};
  uint64_t sstr[1] = {2048};
  uint64_t dsa[2] = {256, (uint64_t)(c->l_pad / 128 * (c->kb4 / 4))};
  r = enc(&c->tmSA, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, c->xsf, dsa, sstr, sbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (Averis SFA) failed: " + std::to_string((int)r)); return AVD_ECUDA; }
  uint64_t dsb[2] = {256, (uint64_t)(c->n_pad / 128 * (c->kb4 / 4))};
  r = enc(&c->tmSB, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, c->wsf, dsb, sstr, sbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (Averis SFB) failed: " + std::to_string((int)r)); return AVD_ECUDA; }
  return AVD_OK;
}

template <typename T>
avd_status av_alloc(AvCtx* c, T** p, size_t bytes) {
  void* q = nullptr;
  if (cudaMalloc(&q, bytes < 16 ? 16 : bytes) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc of " + std::to_string(bytes) + " bytes failed (Averis workspace)");
    return AVD_ENOMEM;
  }
  c->allocs.push_back(q);
  AVD_CUDA(cudaMemsetAsync(q, 0, bytes, c->stream));
  *p = static_cast<T*>(q);
  return AVD_OK;
}

avd_status av_forward(AvCtx* c, const float* X, void* Y) {
  if (!c->weight_set) { set_error("avd_averis_forward: no weight (call avd_averis_set_weight first)"); return AVD_ESTATE; }
  if (!X || !Y || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Y) & 15)) {
    set_error("avd_averis_forward: X / Y must be non-null and 16-byte aligned");
    return AVD_EINVAL;
  }
  const int64_t l = c->l, m = c->m, n = c->n;
  if (c->timing) AVD_CUDA(cudaEventRecord(c->ev[0], c->stream));
  AVD_CUDA(cudaMemsetAsync(c->gsc + 3, 0, sizeof(float), c->stream));
  AVD_CUDA(cudaMemsetAsync(c->gsc + 5, 0, sizeof(float), c->stream));
  const int64_t rows_per = ceil_div(l, c->R);
  av_colstats_kernel<<<dim3((unsigned)ceil_div(m, 1024), (unsigned)c->R), 256, 0, c->stream>>>(
      X, l, m, rows_per, c->csum_part, c->cmax_part, c->cmin_part);
  AVD_LAUNCHED(c);
  av_reduce_kernel<<<(unsigned)ceil_div(m, 32), 256, 0, c->stream>>>(c->csum_part, c->cmax_part, c->cmin_part, c->R,
                                                                      l, m, c->vanilla ? 1 : 0, c->mu, c->mu_f, c->gsc);
  AVD_LAUNCHED(c);
  const uint64_t seed = c->cfg.seed;
  if (!c->vanilla) {
    const unsigned gmu = 1;
    if (c->sr)
      av_quant_rows_kernel<true><<<gmu, 256, 0, c->stream>>>(c->mu_f, 1, m, nullptr, c->gsc + 5, c->gsc + 2, c->mucodes,
                                                             c->musf, 0, 1, seed, 2);
    else
      av_quant_rows_kernel<false><<<gmu, 256, 0, c->stream>>>(c->mu_f, 1, m, nullptr, c->gsc + 5, c->gsc + 2, c->mucodes,
                                                              c->musf, 0, 1, seed, 2);
    AVD_LAUNCHED(c);
    av_bias_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, c->stream>>>(c->mucodes, c->musf, c->wcodes, c->wsf, c->gsc, m, n,
                                                                    c->kb4, c->bias);
    AVD_LAUNCHED(c);
  }
  if (c->timing) AVD_CUDA(cudaEventRecord(c->ev[1], c->stream));
  const unsigned gx = (unsigned)std::min<int64_t>(l, 16 * c->num_sms);  // CTAs walk rows
  const float* muf = c->vanilla ? nullptr : c->mu_f;
  if (c->sr)
    av_quant_rows_kernel<true><<<gx, 256, 0, c->stream>>>(X, l, m, muf, c->gsc + 3, c->gsc + 0, c->xcodes, c->xsf, c->kb4,
                                                          0, seed, 1);
  else
    av_quant_rows_kernel<false><<<gx, 256, 0, c->stream>>>(X, l, m, muf, c->gsc + 3, c->gsc + 0, c->xcodes, c->xsf, c->kb4,
                                                           0, seed, 1);
  AVD_LAUNCHED(c);
  if (c->timing) AVD_CUDA(cudaEventRecord(c->ev[2], c->stream));
  const int64_t MT2 = c->l_pad / 256, NT = c->n_pad / 256;
  const int KB = (int)ceil_div(m, 256);
  const int smem = kAvNS * kAvStage + 8 * kAvOut + 1024;
  auto kern = c->bf16_out ? av_gemm_kernel<true> : av_gemm_kernel<false>;
  AVD_CUDA(smem_attr(kern, smem));
  CUtensorMap tmY;
  {
    auto enc = tma_encode_fn();
    const bool bf = c->bf16_out;
    uint64_t dims[2] = {(uint64_t)n, (uint64_t)l}, strides[1] = {(uint64_t)n * (bf ? 2 : 4)};
    uint32_t box[2] = {bf ? 64u : 32u, 32}, es[2] = {1, 1};
    const CUresult r = enc(&tmY, bf ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Y, dims,
                           strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled (Averis Y) failed: " + std::to_string((int)r)); return AVD_ECUDA; }
  }
  const int grid = 2 * (int)std::min<int64_t>(MT2 * NT, c->num_sms / 2);
  kern<<<grid, kAvGemmThreads, smem, c->stream>>>(c->tmA, c->tmB, c->tmSA, c->tmSB, tmY, l, n, KB, MT2, NT,
                                                            c->kb4, c->gsc, c->bias);
  AVD_LAUNCHED(c);
  if (c->timing) AVD_CUDA(cudaEventRecord(c->ev[3], c->stream));
  return AVD_OK;
}

}  // namespace
}  // namespace avd

using avd::AvCtx;

extern "C" {

struct avd_averis_ctx {
  AvCtx c;
};

avd_status avd_averis_create(const avd_averis_config* cfg, avd_averis_handle* out) {
  if (!cfg || !out) { avd::set_error("avd_averis_create: null argument"); return AVD_EINVAL; }
  *out = nullptr;
  if (cfg->l < 1 || cfg->m < 32 || cfg->m % 32 || cfg->n < 16 || cfg->n % 16) {
    avd::set_error("avd_averis_create: need l >= 1, m a multiple of 32, n a multiple of 16");
    return AVD_EINVAL;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cfg->device) != cudaSuccess || prop.major != 10 || prop.minor != 0) {
    cudaGetLastError();
    avd::set_error("avd_averis_create: device is not an sm_100 (B200) GPU");
    return AVD_ECUDA;
  }
  AVD_CUDA(cudaSetDevice(cfg->device));
  auto* h = new avd_averis_ctx();
  AvCtx* c = &h->c;
  c->cfg = *cfg;
  c->stream = static_cast<cudaStream_t>(cfg->stream);
  c->num_sms = prop.multiProcessorCount;
  c->l = cfg->l; c->m = cfg->m; c->n = cfg->n;
  c->l_pad = avd::round_up(c->l, 256);  // cluster pairs of 128-row tiles
  c->n_pad = avd::round_up(c->n, 256);
  c->kb4 = 4 * avd::ceil_div(c->m, 256);
  c->vanilla = (cfg->flags & AVD_AVERIS_VANILLA) != 0;
  c->sr = (cfg->flags & AVD_AVERIS_STOCHASTIC) != 0;
  c->bf16_out = (cfg->flags & AVD_AVERIS_BF16_OUT) != 0;
  c->timing = (cfg->flags & AVD_AVERIS_TIMING) != 0;
  for (int i = 0; i < 4 && c->timing; ++i)
    if (cudaEventCreate(&c->ev[i]) != cudaSuccess) { cudaGetLastError(); avd::set_error("cudaEventCreate failed"); delete h; return AVD_ECUDA; }
  c->R = (int)std::max<int64_t>(1, std::min<int64_t>(c->l, 4 * c->num_sms / std::max<int64_t>(1, avd::ceil_div(c->m, 1024))));
  const int64_t m = c->m;
  avd_status st = AVD_OK;
  auto A = [&](auto** p, size_t bytes) { if (st == AVD_OK) st = avd::av_alloc(c, p, bytes); };
  A(&c->csum_part, sizeof(double) * c->R * m);
  A(&c->cmax_part, sizeof(float) * c->R * m);
  A(&c->cmin_part, sizeof(float) * c->R * m);
  A(&c->mu, sizeof(double) * m);
  A(&c->mu_f, sizeof(float) * m);
  A(&c->xcodes, (size_t)c->l_pad * m / 2);
  A(&c->xsf, (size_t)c->l_pad * c->kb4 * 4);
  A(&c->wcodes, (size_t)c->n_pad * m / 2);
  A(&c->wsf, (size_t)c->n_pad * c->kb4 * 4);
  A(&c->mucodes, (size_t)m / 2);
  A(&c->musf, (size_t)m / 16);
  A(&c->gsc, sizeof(float) * 8);
  A(&c->bias, sizeof(float) * c->n);
  if (st == AVD_OK) st = avd::make_maps(c);
  if (st == AVD_OK && cudaStreamSynchronize(c->stream) != cudaSuccess) {
    avd::set_error("avd_averis_create: workspace initialisation failed");
    st = AVD_ECUDA;
  }
  if (st != AVD_OK) { avd_averis_destroy(h); return st; }
  *out = h;
  return AVD_OK;
}

avd_status avd_averis_destroy(avd_averis_handle h) {
  if (!h) return AVD_OK;
  for (void* p : h->c.allocs) cudaFree(p);
  if (h->c.X_stage) cudaFree(h->c.X_stage);
  if (h->c.Y_stage) cudaFree(h->c.Y_stage);
  for (cudaEvent_t e : h->c.ev)
    if (e) cudaEventDestroy(e);
  delete h;
  return AVD_OK;
}

avd_status avd_averis_set_weight(avd_averis_handle h, const float* W) {
  if (!h || !W || (reinterpret_cast<uintptr_t>(W) & 15)) {
    avd::set_error("avd_averis_set_weight: null handle / W, or W not 16-byte aligned");
    return AVD_EINVAL;
  }
  AvCtx* c = &h->c;
  AVD_CUDA(cudaMemsetAsync(c->gsc + 4, 0, sizeof(float), c->stream));
  const int64_t cnt = c->m * c->n;
  avd::av_amax_kernel<<<(unsigned)std::min<int64_t>(avd::ceil_div(cnt, 1024), 4 * c->num_sms), 256, 0, c->stream>>>(
      W, cnt, c->gsc + 4);
  AVD_LAUNCHED(c);
  const unsigned g = (unsigned)avd::ceil_div(c->n * (c->m / 16), 256);
  if (c->sr)
    avd::av_quant_cols_kernel<true><<<g, 256, 0, c->stream>>>(W, c->m, c->n, c->gsc + 4, c->gsc + 1, c->wcodes, c->wsf,
                                                              c->kb4, c->cfg.seed, 3);
  else
    avd::av_quant_cols_kernel<false><<<g, 256, 0, c->stream>>>(W, c->m, c->n, c->gsc + 4, c->gsc + 1, c->wcodes, c->wsf,
                                                               c->kb4, c->cfg.seed, 3);
  AVD_LAUNCHED(c);
  c->weight_set = true;
  return AVD_OK;
}

avd_status avd_averis_forward(avd_averis_handle h, const float* X, void* Y) {
  if (!h) { avd::set_error("avd_averis_forward: null handle"); return AVD_EINVAL; }
  return avd::av_forward(&h->c, X, Y);
}

avd_status avd_averis_forward_host(avd_averis_handle h, const float* Xh, void* Yh) {
  if (!h || !Xh || !Yh) { avd::set_error("avd_averis_forward_host: null argument"); return AVD_EINVAL; }
  AvCtx* c = &h->c;
  const size_t xb = sizeof(float) * c->l * c->m, yb = (c->bf16_out ? 2 : 4) * (size_t)c->l * c->n;
  if (!c->X_stage) {
    if (cudaMalloc(&c->X_stage, xb) != cudaSuccess || cudaMalloc(&c->Y_stage, yb) != cudaSuccess) {
      cudaGetLastError();
      avd::set_error("avd_averis_forward_host: staging allocation failed");
      return AVD_ENOMEM;
    }
  }
  AVD_CUDA(cudaMemcpyAsync(c->X_stage, Xh, xb, cudaMemcpyHostToDevice, c->stream));
  AVD_TRY(avd::av_forward(c, c->X_stage, c->Y_stage));
  AVD_CUDA(cudaMemcpyAsync(Yh, c->Y_stage, yb, cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  return AVD_OK;
}

avd_status avd_averis_buffer(avd_averis_handle h, int32_t which, void** dev, size_t* bytes) {
  if (!h || !dev || !bytes) { avd::set_error("avd_averis_buffer: null argument"); return AVD_EINVAL; }
  AvCtx* c = &h->c;
  const int64_t m = c->m;
  switch (which) {
    case AVD_AV_MU: *dev = c->mu; *bytes = sizeof(double) * m; break;
    case AVD_AV_XCODES: *dev = c->xcodes; *bytes = (size_t)c->l_pad * m / 2; break;
    case AVD_AV_XSF: *dev = c->xsf; *bytes = (size_t)c->l_pad * c->kb4 * 4; break;
    case AVD_AV_WCODES: *dev = c->wcodes; *bytes = (size_t)c->n_pad * m / 2; break;
    case AVD_AV_WSF: *dev = c->wsf; *bytes = (size_t)c->n_pad * c->kb4 * 4; break;
    case AVD_AV_MUCODES: *dev = c->mucodes; *bytes = (size_t)m / 2; break;
    case AVD_AV_MUSF: *dev = c->musf; *bytes = (size_t)m / 16; break;
    case AVD_AV_GSCALE: *dev = c->gsc; *bytes = sizeof(float) * 4; break;
    case AVD_AV_BIAS: *dev = c->bias; *bytes = sizeof(float) * c->n; break;
    default: avd::set_error("avd_averis_buffer: unknown buffer id"); return AVD_EINVAL;
  }
  return AVD_OK;
}

int64_t avd_averis_launch_count(avd_averis_handle h) { return h ? h->c.launches : 0; }

avd_status avd_averis_stage_ms(avd_averis_handle h, float* ms) {
  if (!h || !ms || !h->c.timing) {
    avd::set_error("avd_averis_stage_ms: null argument or context created without AVD_AVERIS_TIMING");
    return AVD_EINVAL;
  }
  AVD_CUDA(cudaEventSynchronize(h->c.ev[3]));
  for (int i = 0; i < 3; ++i) AVD_CUDA(cudaEventElapsedTime(ms + i, h->c.ev[i], h->c.ev[i + 1]));
  return AVD_OK;
}

}  // extern "C"
