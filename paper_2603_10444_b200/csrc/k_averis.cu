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
  bool vanilla = false, sr = false;
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
  CUtensorMap tmA{}, tmB{};
  float* X_stage = nullptr;
  float* Y_stage = nullptr;
  std::vector<void*> allocs;
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

// mu (fixed-order sum of the row-chunk partials), mu_f, and the tensor amax of X_R and of mu_f
__global__ void __launch_bounds__(256) av_reduce_kernel(const double* __restrict__ csum, const float* __restrict__ cmax,
                                                        const float* __restrict__ cmin, int R, int64_t l, int64_t m,
                                                        int vanilla, double* __restrict__ mu, float* __restrict__ mu_f,
                                                        float* __restrict__ gsc) {
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  float a = 0.f, am = 0.f;
  if (j < m) {
    double s = 0;
    float mx = -INFINITY, mn = INFINITY;
    for (int y = 0; y < R; ++y) {
      s += csum[(int64_t)y * m + j];
      mx = fmaxf(mx, cmax[(int64_t)y * m + j]);
      mn = fminf(mn, cmin[(int64_t)y * m + j]);
    }
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
  if ((threadIdx.x & 31) == 0) {
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
// Rows of a K-contiguous source (X_R, mu): four threads per 16-block, one float4 each (a warp reads
// 512 contiguous bytes).  sf_plain: scales in plain order (mu) instead of the tensor-core layout.
template <bool SR>
__global__ void __launch_bounds__(256) av_quant_rows_kernel(const float* __restrict__ src, int64_t rows, int64_t K,
                                                            const float* __restrict__ mu_f, const float* __restrict__ amax_p,
                                                            float* __restrict__ g_out, uint8_t* __restrict__ codes,
                                                            uint8_t* __restrict__ sf, int64_t kb4, int sf_plain,
                                                            uint64_t seed, uint64_t tid) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t nb = K >> 4;
  const int64_t blk = t >> 2;
  const int qd = (int)(t & 3);
  const bool ok = blk < rows * nb;
  const int64_t r = ok ? blk / nb : 0, b = ok ? blk - r * nb : 0;
  const int64_t k0 = b * 16 + qd * 4;
  const float g = tensor_g(*amax_p);
  if (t == 0 && g_out) *g_out = g;
  float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    x = __ldcs(reinterpret_cast<const float4*>(src + r * K + k0));
    if (mu_f) {
      const float4 u = __ldg(reinterpret_cast<const float4*>(mu_f + k0));
      x.x = __fsub_rn(x.x, u.x); x.y = __fsub_rn(x.y, u.y); x.z = __fsub_rn(x.z, u.z); x.w = __fsub_rn(x.w, u.w);
    }
  }
  float a = fmaxf(fmaxf(fabsf(x.x), fabsf(x.y)), fmaxf(fabsf(x.z), fabsf(x.w)));
  a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, 1));
  a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, 2));
  const uint32_t sc = e4m3_rn(__fdiv_rn(a, __fmul_rn(6.f, g)));
  uint32_t out = 0;
  if (sc != 0) {
    const float R = __frcp_rn(__fmul_rn(e4m3_val(sc), g));
    const float v0 = __fmul_rn(x.x, R), v1 = __fmul_rn(x.y, R), v2 = __fmul_rn(x.z, R), v3 = __fmul_rn(x.w, R);
    if (SR) {
      const uint64_t li = (uint64_t)(r * K + k0);
      out = e2m1_sr(v0, ctr_u24(seed, tid, li)) | (e2m1_sr(v1, ctr_u24(seed, tid, li + 1)) << 4) |
            (e2m1_sr(v2, ctr_u24(seed, tid, li + 2)) << 8) | (e2m1_sr(v3, ctr_u24(seed, tid, li + 3)) << 12);
    } else {
      out = e2m1x2_rn(v0, v1) | (e2m1x2_rn(v2, v3) << 8);
    }
  }
  if (ok) {
    *reinterpret_cast<uint16_t*>(codes + r * (K >> 1) + (k0 >> 1)) = (uint16_t)out;
    if (qd == 0) sf[sf_plain ? b : sf_off(r, b, kb4)] = (uint8_t)sc;
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
// [n][m/2] (K-major), one 128 x 128 output tile per unit, persistent CTAs (one per SM), K in
// stages of 256 elements (128 B of codes per row: one SWIZZLE_128B atom), 4 MMAs of K = 64 per
// stage.  Per stage the TMA brings A (16 KB), B (16 KB) and the stage's scale chunks (2 x 2 KB,
// 1-D bulk copies: the quantiser wrote them in the tensor-core layout); the MMA warp copies the
// scales to TMEM (tcgen05.cp 32x128b.warpx4: 32 lanes x 16 B broadcast to the four lane quarters)
// and issues the block-scaled MMAs, which execute after the copies in issue order.  Two fp32
// accumulators (TMEM columns 0-127, 128-255) let the epilogue of one tile overlap the next.
constexpr int kAvNS = 5;
constexpr uint32_t kAvA = 128 * 128, kAvB = 128 * 128, kAvSF = 2048;
constexpr uint32_t kAvStage = kAvA + kAvB + 2 * kAvSF;  // 36 KB (multiple of 1 KB)
constexpr int kAvGemmThreads = 192;                    // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue

// kind::mxf4nvf4, A/B E2M1 (format 1), UE4M3 scales (bit 23 = 0), K-major, M = 128, N = 128, K = 64
__host__ __device__ constexpr uint32_t idesc_nvf4(uint32_t M, uint32_t N) {
  return (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_nvf4(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                         uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.scale_vec::4X [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void tmem_cp_sf(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__global__ void __launch_bounds__(kAvGemmThreads, 1) av_gemm_kernel(
    const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const uint8_t* __restrict__ sfa,
    const uint8_t* __restrict__ sfb, int64_t l, int64_t n, int KB, int64_t MT, int64_t NT, int64_t kb4,
    const float* __restrict__ gsc, const float* __restrict__ bias, float* __restrict__ Y) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kAvNS], empty_bar[kAvNS], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_sh;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t tiles = MT * NT;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAvNS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 128); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 1) tmem_alloc<512>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t mt = t / NT, nt = t - (t / NT) * NT;
        for (int kb = 0; kb < KB; ++kb, ++it) {
          const uint32_t s = it % kAvNS, ph = (it / kAvNS) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kAvStage;
          mbar_arrive_expect_tx(&full_bar[s], kAvStage);
          tma_load_2d(st, &tmA, &full_bar[s], kb * 128, (int32_t)(mt * 128));
          tma_load_2d(st + kAvA, &tmB, &full_bar[s], kb * 128, (int32_t)(nt * 128));
          bulk_load_1d(st + kAvA + kAvB, sfa + (mt * kb4 + kb * 4) * 512, kAvSF, &full_bar[s]);
          bulk_load_1d(st + kAvA + kAvB + kAvSF, sfb + (nt * kb4 + kb * 4) * 512, kAvSF, &full_bar[s]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_nvf4(128, 128);
    uint32_t it = 0, ui = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++ui) {
      const uint32_t b = ui & 1, br = ui >> 1;
      mbar_wait(&tempty_bar[b], (br & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + b * 128;
      for (int kb = 0; kb < KB; ++kb, ++it) {
        const uint32_t s = it % kAvNS, ph = (it / kAvNS) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + s * kAvStage);
          const uint32_t tsf = tmem + 256 + (it & 3) * 32;  // 4 rotating scale slots: SFA 16 cols, SFB 16
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            tmem_cp_sf(tsf + kk * 4, smem_desc(base + kAvA + kAvB + kk * 512, 0, 128, 0));
            tmem_cp_sf(tsf + 16 + kk * 4, smem_desc(base + kAvA + kAvB + kAvSF + kk * 512, 0, 128, 0));
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = smem_desc(base + kk * 32, 16, 1024, 2);
            const uint64_t bd = smem_desc(base + kAvA + kk * 32, 16, 1024, 2);
            mma_nvf4(d, ad, bd, idesc, tsf + kk * 4, tsf + 16 + kk * 4, (kb | kk) ? 1u : 0u);
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&tfull_bar[b]);
      __syncwarp();
    }
  } else {
    const uint32_t q = warp & 3;
    const float gxw = __fmul_rn(gsc[0], gsc[1]);
    uint32_t ui = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++ui) {
      const uint32_t b = ui & 1, br = ui >> 1;
      const int64_t mt = t / NT, nt = t - (t / NT) * NT;
      mbar_wait(&tfull_bar[b], br & 1);
      tc_fence_after();
      const int64_t row = mt * 128 + q * 32 + lane;
      const uint32_t tb = tmem + ((q * 32) << 16) + b * 128;
#pragma unroll 1
      for (int c = 0; c < 128; c += 16) {
        uint32_t rv[16];
        tmem_ld16(tb + c, rv);
        tmem_ld_wait();
        const int64_t col = nt * 128 + c;
        if (row < l && col < n) {
          float y[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) y[u] = __fmaf_rn(__uint_as_float(rv[u]), gxw, __ldg(bias + col + u));
          float4* dst = reinterpret_cast<float4*>(Y + row * n + col);
#pragma unroll
          for (int u = 0; u < 4; ++u) __stcs(dst + u, make_float4(y[4 * u], y[4 * u + 1], y[4 * u + 2], y[4 * u + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
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

avd_status av_forward(AvCtx* c, const float* X, float* Y) {
  if (!c->weight_set) { set_error("avd_averis_forward: no weight (call avd_averis_set_weight first)"); return AVD_ESTATE; }
  if (!X || !Y || (reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Y) & 15)) {
    set_error("avd_averis_forward: X / Y must be non-null and 16-byte aligned");
    return AVD_EINVAL;
  }
  const int64_t l = c->l, m = c->m, n = c->n;
  AVD_CUDA(cudaMemsetAsync(c->gsc + 3, 0, sizeof(float), c->stream));
  AVD_CUDA(cudaMemsetAsync(c->gsc + 5, 0, sizeof(float), c->stream));
  const int64_t rows_per = ceil_div(l, c->R);
  av_colstats_kernel<<<dim3((unsigned)ceil_div(m, 1024), (unsigned)c->R), 256, 0, c->stream>>>(
      X, l, m, rows_per, c->csum_part, c->cmax_part, c->cmin_part);
  AVD_LAUNCHED(c);
  av_reduce_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, c->stream>>>(c->csum_part, c->cmax_part, c->cmin_part, c->R,
                                                                       l, m, c->vanilla ? 1 : 0, c->mu, c->mu_f, c->gsc);
  AVD_LAUNCHED(c);
  const uint64_t seed = c->cfg.seed;
  if (!c->vanilla) {
    const unsigned gmu = (unsigned)ceil_div(m / 16 * 4, 256);
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
  const unsigned gx = (unsigned)ceil_div(l * (m / 16) * 4, 256);
  const float* muf = c->vanilla ? nullptr : c->mu_f;
  if (c->sr)
    av_quant_rows_kernel<true><<<gx, 256, 0, c->stream>>>(X, l, m, muf, c->gsc + 3, c->gsc + 0, c->xcodes, c->xsf, c->kb4,
                                                          0, seed, 1);
  else
    av_quant_rows_kernel<false><<<gx, 256, 0, c->stream>>>(X, l, m, muf, c->gsc + 3, c->gsc + 0, c->xcodes, c->xsf, c->kb4,
                                                           0, seed, 1);
  AVD_LAUNCHED(c);
  const int64_t MT = c->l_pad / 128, NT = c->n_pad / 128;
  const int KB = (int)ceil_div(m, 256);
  const int smem = kAvNS * kAvStage + 1024;
  AVD_CUDA(smem_attr(av_gemm_kernel, smem));
  const int grid = (int)std::min<int64_t>(MT * NT, c->num_sms);
  av_gemm_kernel<<<grid, kAvGemmThreads, smem, c->stream>>>(c->tmA, c->tmB, c->xsf, c->wsf, l, n, KB, MT, NT, c->kb4,
                                                            c->gsc, c->bias, Y);
  AVD_LAUNCHED(c);
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
  c->l_pad = avd::round_up(c->l, 128);
  c->n_pad = avd::round_up(c->n, 128);
  c->kb4 = 4 * avd::ceil_div(c->m, 256);
  c->vanilla = (cfg->flags & AVD_AVERIS_VANILLA) != 0;
  c->sr = (cfg->flags & AVD_AVERIS_STOCHASTIC) != 0;
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

avd_status avd_averis_forward(avd_averis_handle h, const float* X, float* Y) {
  if (!h) { avd::set_error("avd_averis_forward: null handle"); return AVD_EINVAL; }
  return avd::av_forward(&h->c, X, Y);
}

avd_status avd_averis_forward_host(avd_averis_handle h, const float* Xh, float* Yh) {
  if (!h || !Xh || !Yh) { avd::set_error("avd_averis_forward_host: null argument"); return AVD_EINVAL; }
  AvCtx* c = &h->c;
  const size_t xb = sizeof(float) * c->l * c->m, yb = sizeof(float) * c->l * c->n;
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

}  // extern "C"
