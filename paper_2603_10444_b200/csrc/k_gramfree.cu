// k_gramfree.cu — Gram-free products for the subspace iteration (SPEC.md:91
// "randomized subspace iteration"; PAPER.md:311-313 randomized / distributed low-rank methods).
//
// With AVD_FLAG_GRAM_FREE the m x m Gram is never formed (l m (m+1) tensor ops): every product
// Y = G Q the eigensolver needs (its power steps and its Rayleigh-Ritz checks) is evaluated as
//
//     Y = X^T (X Q)       X = the centred Gram operand (the fused pass's int8 digit planes)
//
// in two streaming passes over the digit planes (2 B per entry at 2 digits), 4 l m p tensor ops:
//   F0 gf_w_kernel     W = 2^-s Q in four balanced base-128 digits per column (26 bits), and the
//                      centring term corr_r = sum_j qbar_j W_jr (qbar = exact column means of q)
//   F1 gf_xq_kernel    P = Xq W - corr on tcgen05.mma kind::i8 (A: digit planes, K-major over m;
//                      B: W digits), exact int32 accumulation by digit-product class (all classes
//                      kept), fp64 combine
//   F2 gf_pq_kernel    P -> four balanced base-128 digits per column (global per-column scale)
//   F3 gf_xtp_kernel   Z = Xq^T Pd on tcgen05.mma kind::i8 with both operands MN-major from the
//                      row-major planes (K = rows, split over row ranges), exact (two int64 words)
//   F4 gf_fin_kernel   Y = 2^-s (Zi - qbar sum_i Pd) in fp64 (+ fp32 mirror), scratch reset
// X_hat = (q - qbar) 2^-s is the same quantised, exactly centred operand the Gram path forms
// X_hat^T X_hat of, with the diagonal replaced by the exact centred energies as in the Gram path,
// so both iterate on the same matrix up to P's 26-bit quantisation (relative to each column's max:
// a massive activation sets the max of the rows it touches, the other rows keep >= 16 bits).  Every kernel takes the device
// `skip` gate of the graph-resident loop (the first product of a power step that follows a check).
#include <cudaTypedefs.h>
#include <algorithm>
#include <vector>
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // k_gram.cu

namespace {
using namespace sm100;

constexpr int kGfThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr uint32_t kBox = 128 * 128;

__device__ __forceinline__ void mma_i8x(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// kind::i8, S32 accumulator, signed operands; a_mn / b_mn: MN-major
__host__ __device__ constexpr uint32_t idesc_gf(uint32_t M, uint32_t N, uint32_t mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (mn << 15) | (mn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm((uint32_t)a, (uint32_t)b, 0x0040), __byte_perm((uint32_t)c, (uint32_t)d, 0x0040), 0x5410);
}

// ---------------------------------------------------------------- F0: W digits
// one CTA per column r < KQ (r >= p: zero); also resets the per-product scratch (pmax, zsum)
__global__ void __launch_bounds__(256) gf_w_kernel(const double* __restrict__ In, int p, int64_t m, int64_t m_pad,
                                                   const int32_t* __restrict__ shift, const long long* __restrict__ qsum,
                                                   double inv_l, int KQ, int8_t* __restrict__ wd,
                                                   double* __restrict__ wsc, unsigned* __restrict__ pmax,
                                                   long long* __restrict__ zsum, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double sh[256];
  const int r = blockIdx.x;
  if (threadIdx.x == 0) { pmax[r] = 0u; zsum[r] = 0ll; }
  auto vval = [&](int64_t j) -> double { return (r < p && j < m) ? In[j * p + r] : 0.0; };
  double mx = 0.0, cr = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double w = ldexp(vval(j), -shift[j]);
    mx = fmax(mx, fabs(w));
    cr = fma((double)qsum[j] * inv_l, w, cr);
  }
  sh[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double wmax = sh[0];
  __syncthreads();
  sh[threadIdx.x] = cr;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const int te = (wmax > 0.0 && wmax < 1e300) ? ilogb(wmax) + 1 - 26 : 0;  // |z| < 2^26
  if (threadIdx.x == 0) { wsc[r] = ldexp(1.0, te); wsc[KQ + r] = sh[0]; }
  const int64_t plane = (int64_t)KQ * m_pad;
  int8_t* w0 = wd + (int64_t)r * m_pad;
  for (int64_t j = threadIdx.x; j < m_pad; j += 256) {
    const long long z = (wmax > 0.0 && j < m) ? llrint(ldexp(vval(j), -shift[j] - te)) : 0ll;
    const long long zz = z + 64ll * (1 + 128 + 16384 + 2097152);  // balanced base-128, 4 digits
    w0[j] = (int8_t)((zz >> 21) - 64);
    w0[plane + j] = (int8_t)(((zz >> 14) & 127) - 64);
    w0[2 * plane + j] = (int8_t)(((zz >> 7) & 127) - 64);
    w0[3 * plane + j] = (int8_t)((zz & 127) - 64);
  }
}

// ---------------------------------------------------------------- F1: P = Xhat Q
// unit = (128-row block, N-column slice h of P; persistent CTAs): K = m in 128-column stages,
// A = ND digit planes (K-major, SWIZZLE_128B), B = the 4 W digit planes' rows h*N .. +N; EVERY
// digit-product class c = e + d (0 .. ND+2, weight 128^(ND+2-c)) has its own int32 TMEM accumulator:
// the low classes cannot be dropped — in a column whose scale a massive activation sets, the other
// rows live in the low digits only.  N = p when the (ND + 3) classes fit TMEM (one slice, X read
// once), else 64; DB: two accumulators (the epilogue of one unit overlaps the next) when 2 (ND+3) N
// <= 512.  Epilogue: P_ir = t_r sum_c acc_c 128^(ND+2-c) - corr_r (fp64, stored fp32, rows >= l
// zero) and per-column max |P| (atomicMax on the bit patterns).
template <int ND, int NS, int N, bool DB>
__global__ void __launch_bounds__(kGfThreads, 1) gf_xq_kernel(const CUtensorMap* __restrict__ tms, int64_t l_local,
                                                              int64_t m_pad, int64_t l_pad, int KQ, int NH,
                                                              const double* __restrict__ wsc, float* __restrict__ P,
                                                              unsigned* __restrict__ pmax, const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int NCLS = ND + 3;
  constexpr uint32_t kAcc = NCLS * N;  // TMEM columns of one accumulator set
  static_assert((DB ? 2 : 1) * kAcc <= 512, "TMEM");
  constexpr uint32_t kB = N * 128;
  constexpr uint32_t kStage = ((ND * kBox + 4 * kB + 1023) / 1024) * 1024;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[NS], empty_bar[NS], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_sh;
  const CUtensorMap* tmD = tms;
  const CUtensorMap* tmW = tms + (ND == 2 ? 3 : 4);  // W digits in N-row boxes
  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t n_units = ceil_div(l_local, 128) * NH;
  const int NC = (int)(m_pad / 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 8); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(tmD); tma_prefetch(tmW); }
  if (warp == 1) tmem_alloc<512>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int64_t rb = u / NH;
        const int h = (int)(u - rb * NH);
        for (int c = 0; c < NC; ++c, ++it) {
          const uint32_t s = it % NS, ph = (it / NS) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kStage;
          mbar_arrive_expect_tx(&full_bar[s], ND * kBox + 4 * kB);
#pragma unroll
          for (int e = 0; e < ND; ++e) tma_load_2d(st + e * kBox, tmD, &full_bar[s], c * 128, (int32_t)(e * l_pad + rb * 128));
#pragma unroll
          for (int d = 0; d < 4; ++d) tma_load_2d(st + ND * kBox + d * kB, tmW, &full_bar[s], c * 128, d * KQ + h * N);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_gf(128, N, 0);
    uint32_t it = 0, ui = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++ui) {
      const uint32_t b = DB ? (ui & 1) : 0, br = DB ? (ui >> 1) : ui;
      mbar_wait(&tempty_bar[b], (br & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + b * kAcc;
      for (int c = 0; c < NC; ++c, ++it) {
        const uint32_t s = it % NS, ph = (it / NS) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + s * kStage);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int e = 0; e < ND; ++e) {
              const uint64_t a = smem_desc(base + e * kBox + kk * 32, 16, 1024, 2);
#pragma unroll
              for (int d = 0; d < 4; ++d) {
                const uint64_t bd = smem_desc(base + ND * kBox + d * kB + kk * 32, 16, 1024, 2);
                // first product of each class in the unit: e = 0 (classes 0..3), d = 3 (classes 4..)
                const bool first = c == 0 && kk == 0 && (e == 0 || d == 3);
                mma_i8x(d0 + (e + d) * N, a, bd, idesc, first ? 0u : 1u);
              }
            }
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
    const int half = (int)(warp - 2) >> 2;
    uint32_t ui = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++ui) {
      const uint32_t b = DB ? (ui & 1) : 0, br = DB ? (ui >> 1) : ui;
      const int64_t rb = u / NH;
      const int h = (int)(u - rb * NH);
      mbar_wait(&tfull_bar[b], br & 1);
      tc_fence_after();
      const int64_t row = rb * 128 + q * 32 + lane;
      const bool rok = row < l_local;
      const uint32_t tb = tmem + ((q * 32) << 16) + b * kAcc;
#pragma unroll 1
      for (int g = 0; g < N / 16; ++g) {
        const int t0 = half * (N / 2) + 8 * g;  // TMEM column in the slice
        const int c0 = h * N + t0;              // column of P
        double acc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = 0.0;
#pragma unroll
        for (int cl = 0; cl < NCLS; ++cl) {
          uint32_t rv[8];
          tmem_ld8(tb + cl * N + t0, rv);
          tmem_ld_wait();
          const double wgt = (double)(1ll << (7 * (ND + 2 - cl)));
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[t] = fma((double)(int)rv[t], wgt, acc[t]);
        }
        float pv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          pv[t] = rok ? (float)(__ldg(wsc + c0 + t) * acc[t] - __ldg(wsc + KQ + c0 + t)) : 0.f;
          float a = fabsf(pv[t]);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xFFFFFFFFu, a, o));
          if (lane == 0 && a > 0.f) atomicMax(pmax + c0 + t, __float_as_uint(a));
        }
        float4* dst = reinterpret_cast<float4*>(P + row * KQ + c0);
        dst[0] = make_float4(pv[0], pv[1], pv[2], pv[3]);
        dst[1] = make_float4(pv[4], pv[5], pv[6], pv[7]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- F2: P digits
// z_ir = rint(P_ir 2^(26 - e_r)) (|z| <= 2^26, e_r = exponent of the column max), four balanced
// base-128 digits -> pd[d][row][KQ]; t_r = 2^(e_r - 26); exact integer column sums of z (zsum)
__global__ void __launch_bounds__(256) gf_pq_kernel(const float* __restrict__ P, int64_t l_pad, int KQ,
                                                    const unsigned* __restrict__ pmax, int8_t* __restrict__ pd,
                                                    long long* __restrict__ zsum, double* __restrict__ tq,
                                                    const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ long long sz[256];
  const int G = KQ / 4;                          // column groups of 4 per row
  const int cg = threadIdx.x % G, r0 = threadIdx.x / G, RS = 256 / G;
  int e[4];
  float sc[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float mx = __uint_as_float(pmax[4 * cg + t]);
    e[t] = mx > 0.f ? ilogbf(mx) + 1 : 0;
    sc[t] = mx > 0.f ? ldexpf(1.f, 26 - e[t]) : 0.f;
  }
  if (blockIdx.x == 0 && r0 == 0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) tq[4 * cg + t] = ldexp(1.0, e[t] - 26);
  }
  long long zs[4] = {0, 0, 0, 0};
  const int64_t plane = l_pad * KQ;
  for (int64_t row = (int64_t)blockIdx.x * RS + r0; row < l_pad; row += (int64_t)gridDim.x * RS) {
    const float4 v = *reinterpret_cast<const float4*>(P + row * KQ + 4 * cg);
    const float vv[4] = {v.x, v.y, v.z, v.w};
    int dd[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int z = __float2int_rn(vv[t] * sc[t]);  // |z| <= 2^26: four balanced digits
      zs[t] += z;
      const int zz = z + 64 * (1 + 128 + 16384 + 2097152);
      dd[0][t] = (zz >> 21) - 64;
      dd[1][t] = ((zz >> 14) & 127) - 64;
      dd[2][t] = ((zz >> 7) & 127) - 64;
      dd[3][t] = (zz & 127) - 64;
    }
#pragma unroll
    for (int d = 0; d < 4; ++d)
      *reinterpret_cast<uint32_t*>(pd + d * plane + row * KQ + 4 * cg) = pack4(dd[d][0], dd[d][1], dd[d][2], dd[d][3]);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    sz[threadIdx.x] = zs[t];
    __syncthreads();
    if (r0 == 0) {
      long long s = 0;
      for (int rr = 0; rr < RS; ++rr) s += sz[rr * G + cg];
      if (s) atomicAdd(reinterpret_cast<unsigned long long*>(zsum + 4 * cg + t), (unsigned long long)s);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- F3: Zi = Xq^T Pd
// unit = (128 X-columns ta, 64-column slice h of P, row range s): K = rows in 128-row stages,
// A = ND digit planes and B = the slice of the 4 P digit planes, both MN-major (SWIZZLE_128B for
// the 128-column X tiles, SWIZZLE_64B for the 64-byte P rows); every class c = e + d has its own
// int32 accumulator (see F1: no class may be dropped), combined exactly into two int64 words,
// Zhi (weight 2^28) and Zlo, with atomics (order-free): sum_i q_ij z_ir = Zhi 2^28 + Zlo.
template <int ND, int NS>
__global__ void __launch_bounds__(kGfThreads, 1) gf_xtp_kernel(const CUtensorMap* __restrict__ tms, int64_t m_pad,
                                                               int64_t l_pad, int KQ, int64_t NK, int T, int S,
                                                               long long* __restrict__ Zhi, long long* __restrict__ Zlo,
                                                               const int* __restrict__ skip) {
  if (skip && *skip) return;
  constexpr int NCLS = ND + 3;
  constexpr uint32_t kB = 64 * 128;
  constexpr uint32_t kStage = ND * kBox + 4 * kB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[NS], empty_bar[NS], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_sh;
  const CUtensorMap* tmD = tms;
  const CUtensorMap* tmP = tms + 2;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int NH = KQ / 64;
  const int64_t n_units = (int64_t)T * S * NH;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 8);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(tmD); tma_prefetch(tmP); }
  if (warp == 1) tmem_alloc<512>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;
  // h fastest: the slices of one X tile run on neighbouring CTAs (the second read hits L2)
  auto coords = [&](int64_t u, int& ta, int& h, int64_t& k0, int64_t& k1) {
    h = (int)(u % NH);
    const int64_t t2 = u / NH;
    ta = (int)(t2 % T);
    const int s = (int)(t2 / T);
    k0 = NK * s / S;
    k1 = NK * (s + 1) / S;
  };

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        int ta, h;
        int64_t k0, k1;
        coords(u, ta, h, k0, k1);
        for (int64_t ks = k0; ks < k1; ++ks, ++it) {
          const uint32_t s = it % NS, ph = (it / NS) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* st = smem + s * kStage;
          mbar_arrive_expect_tx(&full_bar[s], kStage);
#pragma unroll
          for (int e = 0; e < ND; ++e)
            tma_load_2d(st + e * kBox, tmD, &full_bar[s], ta * 128, (int32_t)(e * l_pad + ks * 128));
#pragma unroll
          for (int d = 0; d < 4; ++d)
            tma_load_2d(st + ND * kBox + d * kB, tmP, &full_bar[s], h * 64, (int32_t)(d * l_pad + ks * 128));
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_gf(128, 64, 1);
    uint32_t it = 0, ui = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++ui) {
      int ta, h;
      int64_t k0, k1;
      coords(u, ta, h, k0, k1);
      mbar_wait(&tempty_bar, (ui & 1) ^ 1);
      tc_fence_after();
      for (int64_t ks = k0; ks < k1; ++ks, ++it) {
        const uint32_t s = it % NS, ph = (it / NS) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + s * kStage);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int e = 0; e < ND; ++e) {
              // MN-major SW128: the K = 32 rows slice kk starts 32 rows (4 KB) in, SBO = 1 KB per 8 rows
              const uint64_t a = smem_desc(base + e * kBox + kk * 4096, 16384, 1024, 2);
#pragma unroll
              for (int d = 0; d < 4; ++d) {
                const uint64_t b = smem_desc(base + ND * kBox + d * kB + kk * 2048, 8192, 512, 4);  // MN-major SW64
                const bool first = ks == k0 && kk == 0 && (e == 0 || d == 3);
                mma_i8x(tmem + (e + d) * 64, a, b, idesc, first ? 0u : 1u);
              }
            }
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&tfull_bar);
      __syncwarp();
    }
  } else {
    const uint32_t q = warp & 3;
    const int half = (int)(warp - 2) >> 2;
    uint32_t ui = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x, ++ui) {
      int ta, h;
      int64_t k0, k1;
      coords(u, ta, h, k0, k1);
      mbar_wait(&tfull_bar, ui & 1);
      tc_fence_after();
      const int64_t j = (int64_t)ta * 128 + q * 32 + lane;
      const uint32_t tb = tmem + ((q * 32) << 16);
#pragma unroll 1
      for (int g = 0; g < 4; ++g) {
        const int t0 = half * 32 + 8 * g;
        const int c0 = h * 64 + t0;
        long long vh[8], vl[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) { vh[t] = 0; vl[t] = 0; }
#pragma unroll
        for (int cl = 0; cl < NCLS; ++cl) {
          uint32_t rv[8];
          tmem_ld8(tb + cl * 64 + t0, rv);
          tmem_ld_wait();
          const int w = 7 * (ND + 2 - cl);  // class weight 2^w
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const long long a = (long long)(int32_t)rv[t];
            if (w >= 28) vh[t] += a << (w - 28);
            else vl[t] += a << w;
          }
        }
        unsigned long long* hrow = reinterpret_cast<unsigned long long*>(Zhi + j * KQ + c0);
        unsigned long long* lrow = reinterpret_cast<unsigned long long*>(Zlo + j * KQ + c0);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (vh[t] != 0) atomicAdd(hrow + t, (unsigned long long)vh[t]);
          if (vl[t] != 0) atomicAdd(lrow + t, (unsigned long long)vl[t]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- F4: Y = Xhat^T Phat + D In
// Y_jr = 2^-s_j t_r (Zhi_jr 2^28 + Zlo_jr - qbar_j zsum_r) + dd_j In_jr; Zhi, Zlo are reset for the next
// product.  dd_j = G_jj (exact centred energy) - (Xhat^T Xhat)_jj replaces the quantised diagonal by
// the exact one, as the Gram path's G has it: a massive activation's own rounding would otherwise
// enter its eigenvalue at first order (2 x e: ~1e-4 of lambda_1 for a 5000 entry).
__global__ void __launch_bounds__(256) gf_fin_kernel(long long* __restrict__ Zhi, long long* __restrict__ Zlo, int KQ,
                                                     int p, int64_t m,
                                                     const int32_t* __restrict__ shift, const long long* __restrict__ qsum,
                                                     double inv_l, const double* __restrict__ tq,
                                                     const long long* __restrict__ zsum, const double* __restrict__ dd,
                                                     const double* __restrict__ In, double* __restrict__ Y,
                                                     float* __restrict__ Y32, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (t >= m * KQ) return;
  const int64_t j = t / KQ;
  const int r = (int)(t - j * KQ);
  const double z = fma((double)Zhi[t], 268435456.0, (double)Zlo[t]);  // sum_i q_ij z_ir
  Zhi[t] = 0;
  Zlo[t] = 0;
  if (r >= p) return;
  const double y = fma(dd[j], In[j * p + r],
                       ldexp(tq[r] * (z - (double)qsum[j] * inv_l * (double)zsum[r]), -shift[j]));
  Y[j * p + r] = y;
  if (Y32) Y32[j * p + r] = (float)y;
}

int gf_kq(int p) { return p <= 64 ? 64 : 128; }

// F1's slice width for (ND, p): p itself when the ND + 3 classes fit TMEM, else 64
int gf_n1(int nd, int p) {
  const int n = ((p + 15) / 16) * 16;
  return (nd + 3) * n <= 512 ? n : 64;
}

template <int ND, int N>
avd_status launch_xq(Ctx* c, int KQ, const int* skip) {
  if constexpr ((ND + 3) * N > 512) {  // never chosen by gf_n1
    set_error("Gram-free slice width exceeds TMEM");
    return AVD_EINVAL;
  } else {
  constexpr bool DB = 2 * (ND + 3) * N <= 512;
  constexpr uint32_t st = ((ND * kBox + 4 * N * 128 + 1023) / 1024) * 1024;
  constexpr int NS = (int)std::min<uint32_t>(4, (220 * 1024) / st);
  const int sm = NS * (int)st + 1024;
  const int NH = (c->p + N - 1) / N;
  const int64_t grid = std::min<int64_t>(ceil_div(c->cfg.l_local, 128) * NH, c->num_sms);
  AVD_CUDA(smem_attr(gf_xq_kernel<ND, NS, N, DB>, sm));
  gf_xq_kernel<ND, NS, N, DB><<<(unsigned)grid, kGfThreads, sm, c->stream>>>(
      c->gf_tm, c->cfg.l_local, c->m_pad, c->l_pad, KQ, NH, c->gf_wsc, c->gf_P, c->gf_pmax, skip);
  AVD_LAUNCHED(c);
  return AVD_OK;
  }
}

template <int ND>
avd_status launch_gf(Ctx* c, int KQ, int T, int S, int grid3, const int* skip) {
  switch (gf_n1(ND, c->p)) {
#define CASE(NN) case NN: AVD_TRY((launch_xq<ND, NN>(c, KQ, skip))); break;
    CASE(16) CASE(32) CASE(48) CASE(64) CASE(80) CASE(96)
#undef CASE
    default: set_error("unsupported Gram-free slice width"); return AVD_EINVAL;
  }
  gf_pq_kernel<<<(unsigned)std::min<int64_t>(4 * c->num_sms, ceil_div(c->l_pad, 256 / (KQ / 4))), 256, 0, c->stream>>>(
      c->gf_P, c->l_pad, KQ, c->gf_pmax, c->gf_pd, c->gf_zsum, c->gf_tq, skip);
  AVD_LAUNCHED(c);
  constexpr int NS = ND == 2 ? 3 : 2;  // <= 227 KB of shared memory (64 / 80 KB stages)
  constexpr uint32_t st = ND * kBox + 4 * 64 * 128;
  const int sm = NS * (int)st + 1024;
  AVD_CUDA(smem_attr(gf_xtp_kernel<ND, NS>, sm));
  gf_xtp_kernel<ND, NS><<<(unsigned)grid3, kGfThreads, sm, c->stream>>>(c->gf_tm, c->m_pad, c->l_pad, KQ, c->l_pad / 128,
                                                                      T, S, c->gf_zi, c->gf_zlo, skip);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace

// workspace and tensor maps of the Gram-free products (once per context)
avd_status gf_prepare(Ctx* c) {
  if (c->gf_tm) return AVD_OK;
  const int KQ = gf_kq(c->p);
  auto alloc = [&](auto** ptr, size_t bytes) -> avd_status {
    void* q = nullptr;
    if (cudaMalloc(&q, bytes) != cudaSuccess) {
      cudaGetLastError();
      set_error("cudaMalloc failed (Gram-free workspace, " + std::to_string(bytes) + " bytes)");
      return AVD_ENOMEM;
    }
    c->gf_allocs.push_back(q);
    AVD_CUDA(cudaMemsetAsync(q, 0, bytes, c->stream));
    *ptr = static_cast<std::remove_reference_t<decltype(*ptr)>>(q);
    return AVD_OK;
  };
  AVD_TRY(alloc(&c->gf_wd, (size_t)4 * KQ * c->m_pad));
  AVD_TRY(alloc(&c->gf_wsc, sizeof(double) * 2 * KQ));
  AVD_TRY(alloc(&c->gf_tq, sizeof(double) * KQ));
  AVD_TRY(alloc(&c->gf_pmax, sizeof(unsigned) * KQ));
  AVD_TRY(alloc(&c->gf_zsum, sizeof(long long) * KQ));
  AVD_TRY(alloc(&c->gf_P, sizeof(float) * c->l_pad * KQ));
  AVD_TRY(alloc(&c->gf_pd, (size_t)4 * c->l_pad * KQ));
  AVD_TRY(alloc(&c->gf_zi, sizeof(long long) * c->m_pad * KQ));
  AVD_TRY(alloc(&c->gf_zlo, sizeof(long long) * c->m_pad * KQ));
  AVD_TRY(alloc(&c->gf_dd, sizeof(double) * c->m_pad));
  AVD_TRY(alloc(&c->gf_qsq, sizeof(long long) * c->m_pad));
  AVD_TRY(alloc(&c->gf_tm, 5 * sizeof(CUtensorMap)));
  CUtensorMap tm[5];
  auto enc = tma_encode_fn();
  uint32_t es[2] = {1, 1};
  {  // X digit planes [nd_max][l_pad][m_pad], 128 x 128 boxes (K-major for F1, MN-major for F3)
    uint64_t dims[2] = {(uint64_t)c->m_pad, (uint64_t)(c->nd_max * c->l_pad)}, str[1] = {(uint64_t)c->m_pad};
    uint32_t box[2] = {128, 128};
    if (enc(&tm[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->digits, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (Gram-free X map)");
      return AVD_ECUDA;
    }
  }
  {  // W digits [4][KQ][m_pad]: 128-column x 64-row boxes
    uint64_t dims[2] = {(uint64_t)c->m_pad, (uint64_t)(4 * KQ)}, str[1] = {(uint64_t)c->m_pad};
    uint32_t box[2] = {128, 64};
    if (enc(&tm[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->gf_wd, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (Gram-free W map)");
      return AVD_ECUDA;
    }
  }
  {  // P digits [4][l_pad][KQ]: 64-column x 128-row boxes (SWIZZLE_64B rows)
    uint64_t dims[2] = {(uint64_t)KQ, (uint64_t)(4 * c->l_pad)}, str[1] = {(uint64_t)KQ};
    uint32_t box[2] = {64, 128};
    if (enc(&tm[2], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->gf_pd, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (Gram-free P map)");
      return AVD_ECUDA;
    }
  }
  for (int nd = 2; nd <= 3; ++nd) {  // W digits in F1's N-row boxes (tm[3]: 2 digits, tm[4]: 3)
    uint64_t dims[2] = {(uint64_t)c->m_pad, (uint64_t)(4 * KQ)}, str[1] = {(uint64_t)c->m_pad};
    uint32_t box[2] = {128, (uint32_t)gf_n1(nd, c->p)};
    if (enc(&tm[1 + nd], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->gf_wd, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (Gram-free W slice map)");
      return AVD_ECUDA;
    }
  }
  AVD_CUDA(cudaMemcpyAsync(c->gf_tm, tm, sizeof(tm), cudaMemcpyHostToDevice, c->stream));
  return AVD_OK;
}

// Y = G In evaluated as Xhat^T (Xhat In) (F0-F4); In, Y fp64 [m][p], Y32 optional fp32 mirror
avd_status gf_product(Ctx* c, const double* In, double* Y, float* Y32, const int* skip) {
  const int KQ = gf_kq(c->p);
  const int64_t m = c->cfg.m;
  const double inv_l = 1.0 / (double)c->cfg.l_global;
  gf_w_kernel<<<KQ, 256, 0, c->stream>>>(In, c->p, m, c->m_pad, c->shift, c->qsum, inv_l, KQ, c->gf_wd, c->gf_wsc,
                                          c->gf_pmax, c->gf_zsum, skip);
  AVD_LAUNCHED(c);
  const int NH = KQ / 64;  // F3's 64-column slices
  const int T = (int)(c->m_pad / 128);
  const int64_t NK = c->l_pad / 128;
  // row-range splits: every unit <= 256 stages (int32 class sums stay exact); among those, the S
  // whose whole waves of units finish first (time ~ waves x stages per unit, plus a small
  // per-unit epilogue cost)
  int S = 1;
  {
    double best = 1e300;
    const int64_t tiles = (int64_t)T * NH;
    for (int64_t s = std::max<int64_t>(1, ceil_div(NK, 256)); s <= std::min<int64_t>(NK, 64); ++s) {
      const double t = (double)ceil_div(tiles * s, c->num_sms) * ((double)ceil_div(NK, s) + 4.0);
      if (t < best - 1e-9) { best = t; S = (int)s; }
    }
  }
  const int grid3 = (int)std::min<int64_t>((int64_t)T * S * NH, c->num_sms);
  const bool nd3 = c->nd == 3;
  AVD_TRY(nd3 ? launch_gf<3>(c, KQ, T, S, grid3, skip) : launch_gf<2>(c, KQ, T, S, grid3, skip));
  gf_fin_kernel<<<(unsigned)ceil_div(m * KQ, 256), 256, 0, c->stream>>>(c->gf_zi, c->gf_zlo, KQ, c->p, m, c->shift,
                                                                        c->qsum, inv_l, c->gf_tq, c->gf_zsum, c->gf_dd, In,
                                                                        Y, Y32, skip);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// Sum_i q_ij^2 from the digit planes (the fused pass does not carry it): sixteen columns per
// thread (one 16-byte load per plane and row, four rows in flight), a row chunk per CTA row,
// exact int64 atomics (order-free)
__global__ void __launch_bounds__(256) gf_qsq_kernel(const int8_t* __restrict__ digits, int nd, int64_t l_local,
                                                     int64_t l_pad, int64_t m, int64_t m_pad, int64_t rows_per,
                                                     unsigned long long* __restrict__ qsq) {
  const int64_t j = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 16;
  if (j >= m_pad) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(l_local, r0 + rows_per);
  long long s[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) s[t] = 0;
  for (int64_t r = r0; r < r1; r += 4) {
    uint4 w[3][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int e = 0; e < 3; ++e)
        w[e][u] = (e < nd && r + u < r1)
                      ? __ldcs(reinterpret_cast<const uint4*>(digits + ((int64_t)e * l_pad + r + u) * m_pad + j))
                      : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        int q = 0;
#pragma unroll
        for (int e = 0; e < 3; ++e) {
          if (e >= nd) break;
          const uint32_t word = t < 4 ? w[e][u].x : (t < 8 ? w[e][u].y : (t < 12 ? w[e][u].z : w[e][u].w));
          q = q * 128 + (int)(int8_t)(word >> (8 * (t & 3)));
        }
        s[t] += (long long)q * q;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 16; ++t)
    if (j + t < m && s[t]) atomicAdd(qsq + j + t, (unsigned long long)s[t]);
}

// the diagonal of G (exact centred energies, as gram_finalize writes it) for tr(G) and the
// precision bound, and dd = that diagonal minus the quantised operand's (F4); the off-diagonal
// of G is never formed
__global__ void gf_diag_kernel(int64_t m, int64_t m_pad, const double* __restrict__ ysq, const double* __restrict__ mu,
                               const float* __restrict__ mu0, double l, const long long* __restrict__ qsum,
                               const unsigned long long* __restrict__ qsq, const int32_t* __restrict__ shift,
                               double* __restrict__ G, double* __restrict__ dd) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double dm = mu[j] - (double)mu0[j];
  const double g = ysq[j] - l * dm * dm;
  G[j * m_pad + j] = g;
  // (Xhat^T Xhat)_jj = (sum q^2 - S^2 / l) 2^-2s  (S: exact column sum of q)
  const double S = (double)qsum[j];
  dd[j] = g - ldexp((double)(long long)qsq[j] - S * S / l, -2 * shift[j]);
}
avd_status gf_diag(Ctx* c) {
  const int64_t rows_per = 256;
  AVD_CUDA(cudaMemsetAsync(c->gf_qsq, 0, sizeof(long long) * c->m_pad, c->stream));
  dim3 grid((unsigned)ceil_div(c->m_pad, 4096), (unsigned)ceil_div(c->cfg.l_local, rows_per));
  gf_qsq_kernel<<<grid, 256, 0, c->stream>>>(c->digits, c->nd, c->cfg.l_local, c->l_pad, c->cfg.m, c->m_pad, rows_per,
                                             reinterpret_cast<unsigned long long*>(c->gf_qsq));
  AVD_LAUNCHED(c);
  gf_diag_kernel<<<(unsigned)ceil_div(c->cfg.m, 256), 256, 0, c->stream>>>(
      c->cfg.m, c->m_pad, c->ysq, c->mu, c->mu0, (double)c->cfg.l_global, c->qsum,
      reinterpret_cast<const unsigned long long*>(c->gf_qsq), c->shift, c->G, c->gf_dd);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
