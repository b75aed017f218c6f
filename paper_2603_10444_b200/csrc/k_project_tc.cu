// k_project_tc.cu — K5 and K8 on the 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32).
//
// K5 (projection: spike = U_k S_k V_k^T = (Xc V_k) V_k^T):
//     P[128-row block] = Xc_blk V_k      M = 128 rows, N = KP (k padded to 16), K = m
//   X tiles arrive by TMA (SWIZZLE_128B, K-major: X is row-major with K = column); four converter
//   warps centre them (x - mu_j, fp64 subtract) and split x_c = hi + lo (cvt.rna.tf32) in place
//   of the swizzled layout; the MMA warp issues hi*Vhi + hi*Vlo + lo*Vhi.  The tcgen05 fp32
//   accumulator truncates (profiles/r01_umma_probe.txt), so the K range is spread over up to
//   8 TMEM slots (<= 64 K-steps each, bias <= ~4e-6) that the epilogue adds in fp32.
//   Epilogue writes P (fp32, for K7) and its hi/lo planes (K8's A operand), column sums of P
//   (column means of the spike) and sum xc^2.
// K8 (energies):
//     S[128-row block, N-col chunk] = P_blk V_k^T     M = 128, N = 128 (64 if KP > 64), K = KP
//   A = P hi/lo (TMA, resident per row block), B = V hi/lo (TMA ring); epilogue warps read the
//   spike tile from TMEM, x from global, and accumulate sum spike^2, tail^2, spike*tail in fp64
//   (tail = xc - spike).
// Roles (192 threads): warp 0 TMA, warp 1 TMEM alloc + MMA issue, warps 2-5 convert/epilogue.
#include <cudaTypedefs.h>
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // k_gram.cu

namespace {
using namespace sm100;

constexpr int kPThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 convert / epilogue
constexpr uint32_t kTile = 128 * 128;  // bytes of a 128-row x 32-fp32 swizzled tile

// round to the nearest tf32 (10 mantissa bits), ties away from zero: add half of the dropped 13-bit
// field to the magnitude bits and clear it (two integer ops; the cvt.rna.tf32.f32 instruction is
// emulated by a longer sequence on sm_100a).  Finite inputs below 2^127 only (X is checked finite).
__device__ __forceinline__ float rna_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// fp64 V (m x k, row-major) -> V_hl [2][m_pad128][KP32] (tf32 hi plane then lo plane; K8's B
// operand); padding is zero (column k, the mean direction of K5's W, stays zero here so the spike
// S = P V_k^T is unaffected).
__global__ void split_v_kernel(const double* __restrict__ V, int64_t m, int k, int KP32, int64_t m_pad128,
                               float* __restrict__ V_hl) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m_pad128 * KP32) return;
  const int64_t j = t / KP32;
  const int r = (int)(t % KP32);
  const float v = (j < m && r < k) ? (float)V[j * k + r] : 0.f;
  const float hi = rna_tf32(v), lo = rna_tf32(v - hi);
  V_hl[j * KP32 + r] = hi;
  V_hl[(m_pad128 + j) * KP32 + r] = lo;
}

// ======================================================================= K5
// P = Xc V_k from the Gram operand itself (the nd digit planes of the fused pass, k_pass1.cu) on
// tcgen05.mma kind::i8 — exact integer products, 1 B per digit read instead of 4 B of X, no
// conversion pass in shared memory.  The planes hold q_ij = round_dither((x_ij - mu0_j) 2^s_j)
// (balanced base-128 digits, plane 0 most significant), so
//   P_ir = sum_j x~_ij V_jr = sum_j q_ij 2^-s_j V_jr - corr_r,  corr_r = sum_j (mu_j - mu0_j) V_jr,
// up to the operand's dithered rounding (the same quantisation the Gram and V_k come from;
// DESIGN.md §8).  W_jr = 2^-s_j V_jr is held per column r as t_r z_jr with an integer
// |z_jr| < 2^26 in four balanced base-128 digits (split_w_kernel); the nd x 4 digit products
// accumulate exactly in int32 TMEM by weight class c = e + d (weight 128^(nd + 2 - c)); the
// classes c <= 3 are kept (the rest weigh <= 2^-28 of the leading one), combined per row in
// fp64 in the epilogue, then P = t_r (q . z) - corr_r.
// Column k carries the mean direction mu / ||mu|| (f2 diagnostics: p_i = P[i][k] + ||mu||).
constexpr int kK5Threads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue (two per TMEM lane quadrant)

// Spiky columns: a column whose range is > 64x its rms (a few massive activations)
// gets a quantisation step far coarser than its typical entries, and when such a column carries a
// spike direction (v_r ~ e_j) that step would show in P.  The first kMaxSpiky such columns (by
// index) are taken out of the integer product and added exactly from X in the K5 epilogue.
// One CTA: spk[0] = count, spk[1 ..] = ascending column indices.
constexpr int kMaxSpiky = 16;
__global__ void __launch_bounds__(1024) spiky_kernel(const float* __restrict__ colmax, const double* __restrict__ ysq,
                                                    int64_t m, double l, int* __restrict__ spk) {
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t j0 = 0; j0 < m; j0 += 1024) {
    const int64_t j = j0 + threadIdx.x;
    bool f = false;
    if (j < m) {
      const double rms = sqrt(ysq[j] / l);
      f = (double)colmax[j] > 64.0 * rms && rms > 0.0;
    }
    const unsigned b = __ballot_sync(0xFFFFFFFFu, f);
    __shared__ int wcnt[32];
    if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(b);
    __syncthreads();
    int off = base;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) off += wcnt[w];
    off += __popc(b & ((1u << (threadIdx.x & 31)) - 1u));
    if (f && off < kMaxSpiky) spk[1 + off] = (int)j;
    __syncthreads();
    if (threadIdx.x == 0) { int t = 0; for (int w = 0; w < 32; ++w) t += wcnt[w]; base += t; }
    __syncthreads();
  }
  if (threadIdx.x == 0) spk[0] = base < kMaxSpiky ? base : kMaxSpiky;
}

// one CTA per column r < KP of W (r < k: V_k; r == k: mu_hat; else zero); spiky columns are zero
// in W and left out of corr_r (the K5 epilogue adds their exact contribution)
__global__ void __launch_bounds__(256) split_w_kernel(const double* __restrict__ V, const double* __restrict__ mu,
                                                     const float* __restrict__ mu0, const double* __restrict__ diag,
                                                     const int32_t* __restrict__ shift, int64_t m, int64_t m_pad,
                                                     int k, int KP, int8_t* __restrict__ wd, double* __restrict__ wsc,
                                                     const int* __restrict__ spk) {
  __shared__ double sh[256];
  __shared__ int sj[kMaxSpiky];
  const int r = blockIdx.x;
  const double nrm = diag[0];
  const int nsp = spk[0];
  if ((int)threadIdx.x < nsp) sj[threadIdx.x] = spk[1 + threadIdx.x];
  __syncthreads();
  auto vval = [&](int64_t j) -> double {
    if (j >= m) return 0.0;
    for (int t = 0; t < nsp; ++t)
      if (sj[t] == (int)j) return 0.0;
    if (r < k) return V[j * k + r];
    if (r == k) return nrm > 0.0 ? mu[j] / nrm : 0.0;
    return 0.0;
  };
  // max |W_jr| and corr_r = sum_j (mu_j - mu0_j) v_jr (fixed order)
  double mx = 0.0, cr = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double v = vval(j);
    mx = fmax(mx, fabs(ldexp(v, -shift[j])));
    cr = fma(mu[j] - (double)mu0[j], v, cr);
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
  // t_r = 2^(e - 26) with wmax < 2^e: |z| = |W / t| < 2^26 fits four balanced digits (< 1.33e8);
  // 26 bits relative to the column's largest |W_jr| leave >= 18 bits for columns whose scale
  // 2^-s_j is up to 2^8 smaller (a massive-activation column sets its own coarse scale)
  const int e = (wmax > 0.0 && wmax < 1e300) ? ilogb(wmax) + 1 : 0;
  const int te = e - 26;
  if (threadIdx.x == 0) { wsc[r] = ldexp(1.0, te); wsc[KP + r] = sh[0]; }
  int8_t* w0 = wd + (int64_t)r * m_pad;
  const int64_t plane = (int64_t)KP * m_pad;
  for (int64_t j = threadIdx.x; j < m_pad; j += 256) {
    const double v = vval(j);
    const long long z = (wmax > 0.0) ? llrint(ldexp(v, -shift[min(j, m - 1)] - te)) : 0ll;
    // balanced base-128: z = w0 128^3 + w1 128^2 + w2 128 + w3, w in [-64, 63]
    const long long zz = z + 64ll * (1 + 128 + 16384 + 2097152);
    w0[j] = (int8_t)((zz >> 21) - 64);
    w0[plane + j] = (int8_t)(((zz >> 14) & 127) - 64);
    w0[2 * plane + j] = (int8_t)(((zz >> 7) & 127) - 64);
    w0[3 * plane + j] = (int8_t)((zz & 127) - 64);
  }
}

// kind::i8, int32 accumulator, signed A/B, both K-major
__host__ __device__ constexpr uint32_t idesc_i8k(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8k(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int KP, int ND, int NS, bool DB>
__global__ void __launch_bounds__(kK5Threads, 1) proj_i8_kernel(
    const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmW, int64_t l_local, int64_t m_pad,
    int64_t l_pad, const double* __restrict__ wsc, float* __restrict__ P, float* __restrict__ P_hl,
    double* __restrict__ colsumP_part, const float* __restrict__ X, int64_t m, const int* __restrict__ spk,
    const double* __restrict__ V, const double* __restrict__ mu, const double* __restrict__ diag, int k) {
  constexpr int KP32 = (KP + 31) / 32 * 32;
  constexpr int NCLS = 4;                           // weight classes c = e + d <= 3 (e < ND, d < 4)
  constexpr uint32_t kA = 128 * 128;               // one digit plane: 128 rows x 128 K-bytes
  constexpr uint32_t kB = KP * 128;                // one W digit plane: KP rows x 128 K-bytes
  constexpr uint32_t kStage = ((ND * kA + 4 * kB + 1023) / 1024) * 1024;
  constexpr uint32_t kAcc = NCLS * KP;             // TMEM columns of one row block
  constexpr uint32_t kTmem = DB ? (2 * kAcc <= 256 ? 256 : 512) : (kAcc <= 256 ? 256 : 512);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[NS], empty_bar[NS], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_sh;
  __shared__ double colsum_w[8][KP];
  __shared__ double s_t[KP], s_c[KP];
  __shared__ double s_vsp[kMaxSpiky][KP];  // V rows (and mu_hat) of the spiky columns
  __shared__ double s_msp[kMaxSpiky];
  __shared__ int s_jsp[kMaxSpiky];
  const int nsp = spk[0];

  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t nrb = ceil_div(l_local, 128);
  const int NC = (int)(m_pad / 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 8); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmD); tma_prefetch(&tmW); }
  if (warp == 1) tmem_alloc<kTmem>(&tmem_sh);
  if (warp >= 2) {
    for (int r = lane; r < KP; r += 32) colsum_w[warp - 2][r] = 0.0;
  }
  for (int r = threadIdx.x; r < KP; r += blockDim.x) { s_t[r] = wsc[r]; s_c[r] = wsc[KP + r]; }
  for (int t = threadIdx.x; t < nsp * KP; t += blockDim.x) {
    const int u = t / KP, r = t % KP;
    const int64_t j = spk[1 + u];
    const double nrm = diag[0];
    s_vsp[u][r] = r < k ? V[j * k + r] : (r == k && nrm > 0.0 ? mu[j] / nrm : 0.0);
    if (r == 0) { s_msp[u] = mu[j]; s_jsp[u] = (int)j; }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
        for (int c = 0; c < NC; ++c, ++it) {
          const uint32_t s = it % NS, r = it / NS;
          mbar_wait(&empty_bar[s], (r & 1) ^ 1);
          uint8_t* st = smem + s * kStage;
          mbar_arrive_expect_tx(&full_bar[s], ND * kA + 4 * kB);
#pragma unroll
          for (int e = 0; e < ND; ++e)
            tma_load_2d(st + e * kA, &tmD, &full_bar[s], c * 128, (int32_t)(e * l_pad + rb * 128));
#pragma unroll
          for (int d = 0; d < 4; ++d)
            tma_load_2d(st + ND * kA + d * kB, &tmW, &full_bar[s], c * 128, d * KP);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_i8k(128, KP);
    uint32_t it = 0, ui = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
      const uint32_t b = DB ? (ui & 1) : 0, br = DB ? (ui >> 1) : ui;
      mbar_wait(&tempty_bar[b], (br & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem + b * kAcc;
      for (int c = 0; c < NC; ++c, ++it) {
        const uint32_t s = it % NS, r = it / NS;
        mbar_wait(&full_bar[s], r & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + s * kStage);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int e = 0; e < ND; ++e) {
              const uint64_t a = smem_desc(base + e * kA + kk * 32, 16, 1024, 2);
#pragma unroll
              for (int d = 0; d < 4; ++d) {
                if (e + d > 3) continue;  // dropped class (<= 2^-28 of the leading weight)
                const uint64_t bd = smem_desc(base + ND * kA + d * kB + kk * 32, 16, 1024, 2);
                // the first product of each class in the row block starts its accumulator
                const bool first = c == 0 && kk == 0 && e == 0;
                mma_i8k(d0 + (e + d) * KP, a, bd, idesc, first ? 0u : 1u);
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
    // ================= epilogue (8 warps: lane quadrant q, column half h): P row i, columns r
    const int ew = warp - 2;
    const uint32_t q = warp & 3;
    const int half = ew >> 2;
    uint32_t ui = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
      const uint32_t b = DB ? (ui & 1) : 0, br = DB ? (ui >> 1) : ui;
      mbar_wait(&tfull_bar[b], br & 1);
      tc_fence_after();
      const int64_t row = rb * 128 + q * 32 + lane;
      const bool rok = row < l_local;
      const uint32_t tb = tmem + ((q * 32) << 16) + b * kAcc;
#pragma unroll 1
      for (int c0 = half * (KP / 2); c0 < (half + 1) * (KP / 2); c0 += 8) {
        double acc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = 0.0;
#pragma unroll
        for (int cl = 0; cl < NCLS; ++cl) {
          uint32_t rv[8];
          tmem_ld8(tb + cl * KP + c0, rv);
          tmem_ld_wait();
          const double wgt = (double)(1ll << (7 * (ND + 2 - cl)));  // 128^(nd + 2 - c), exact
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[t] = fma((double)(int)rv[t], wgt, acc[t]);
        }
        double ex[8];  // exact contribution of the spiky columns, (x_ij - mu_j) v_jr in fp64
#pragma unroll
        for (int t = 0; t < 8; ++t) ex[t] = 0.0;
        for (int u = 0; u < nsp; ++u) {
          const double xt = rok ? (double)__ldg(X + row * m + s_jsp[u]) - s_msp[u] : 0.0;
#pragma unroll
          for (int t = 0; t < 8; ++t) ex[t] = fma(xt, s_vsp[u][c0 + t], ex[t]);
        }
        float pv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) pv[t] = (float)((s_t[c0 + t] * acc[t] - s_c[c0 + t]) + ex[t]);
        if (rok) {
          float4* dst = reinterpret_cast<float4*>(P + row * KP + c0);
          dst[0] = make_float4(pv[0], pv[1], pv[2], pv[3]);
          dst[1] = make_float4(pv[4], pv[5], pv[6], pv[7]);
          float hv[8], lv[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) { hv[t] = rna_tf32(pv[t]); lv[t] = rna_tf32(pv[t] - hv[t]); }
          float4* hrow = reinterpret_cast<float4*>(P_hl + row * KP32 + c0);
          float4* lrow = reinterpret_cast<float4*>(P_hl + (l_pad + row) * KP32 + c0);
          hrow[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
          hrow[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
          lrow[0] = make_float4(lv[0], lv[1], lv[2], lv[3]);
          lrow[1] = make_float4(lv[4], lv[5], lv[6], lv[7]);
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          double v = rok ? (double)pv[t] : 0.0;
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
          if (lane == 0) colsum_w[ew][c0 + t] += v;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < KP) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += colsum_w[w][threadIdx.x];
    colsumP_part[(int64_t)blockIdx.x * KP + threadIdx.x] = t;
  }
  if (warp == 1) tmem_dealloc<kTmem>(tmem);
}

// ======================================================================= K8
// Stage ring: V hi/lo tiles (B operand) + the matching X tile (for the epilogue), both by TMA.
// A stage is released when the MMA has consumed it AND the 8 epilogue warps have read its X.
template <int KP32, int NCOL, int NS>
__global__ void __launch_bounds__(kPThreads, 1) energy_tc_kernel(
    const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmV,
    const __grid_constant__ CUtensorMap tmX, int64_t l_local, int64_t m, int64_t l_pad, int64_t m_pad128,
    const float* __restrict__ mu_hl, int64_t m_pad, double* __restrict__ en_part) {
  constexpr int NA = KP32 / 32;                       // 32-wide K atoms
  constexpr int NXB = NCOL / 32;                      // X boxes (32 columns) per chunk
  constexpr uint32_t kATile = kTile;                  // 128 rows x 128 B
  constexpr uint32_t kBTile = NCOL * 128;             // NCOL rows x 128 B
  constexpr uint32_t kA = 2 * NA * kATile;            // P hi + lo
  constexpr uint32_t kVB = 2 * NA * kBTile;           // V hi + lo
  constexpr uint32_t kStage = kVB + NXB * kTile;      // + X tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned in the shared window; derived from smem_raw by an offset so the compiler keeps
  // the shared address space (LDS/STS instead of generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kA;
  __shared__ uint64_t afull_bar, aempty_bar, full_bar[NS], empty_bar[NS], tfull_bar[2], tempty_bar[2];
  __shared__ uint32_t tmem_sh;
  __shared__ double red[8][3];

  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t nrb = ceil_div(l_local, 128);
  const int NC = (int)((m + NCOL - 1) / NCOL);
  if (threadIdx.x == 0) {
    mbar_init(&afull_bar, 1);
    mbar_init(&aempty_bar, 1);
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1 + 8); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull_bar[b], 1); mbar_init(&tempty_bar[b], 8); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmP); tma_prefetch(&tmV); tma_prefetch(&tmX); }
  if (warp == 1) tmem_alloc<(2 * NCOL < 32 ? 32 : 2 * NCOL)>(&tmem_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0, ui = 0;
      for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
        mbar_wait(&aempty_bar, (ui & 1) ^ 1);
        mbar_arrive_expect_tx(&afull_bar, kA);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int a = 0; a < NA; ++a)
            tma_load_2d(sA + (h * NA + a) * kATile, &tmP, &afull_bar, a * 32, (int32_t)(h * l_pad + rb * 128));
        for (int c = 0; c < NC; ++c, ++it) {
          const uint32_t s = it % NS, r = it / NS;
          mbar_wait(&empty_bar[s], (r & 1) ^ 1);
          uint8_t* st = sB + s * kStage;
          mbar_arrive_expect_tx(&full_bar[s], kStage);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int a = 0; a < NA; ++a)
              tma_load_2d(st + (h * NA + a) * kBTile, &tmV, &full_bar[s], a * 32, (int32_t)(h * m_pad128 + c * NCOL));
#pragma unroll
          for (int xb = 0; xb < NXB; ++xb)
            tma_load_2d(st + kVB + xb * kTile, &tmX, &full_bar[s], c * NCOL + xb * 32, (int32_t)(rb * 128));
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_tf32(128, NCOL, 0, 0);
    uint32_t it = 0, ui = 0, ci = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
      mbar_wait(&afull_bar, ui & 1);
      tc_fence_after();
      for (int c = 0; c < NC; ++c, ++it, ++ci) {
        const uint32_t s = it % NS, r = it / NS;
        const uint32_t b = ci & 1, br = ci >> 1;
        mbar_wait(&tempty_bar[b], (br & 1) ^ 1);
        mbar_wait(&full_bar[s], r & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t abase = smem_u32(sA), bbase = smem_u32(sB + s * kStage);
          const uint32_t d = tmem + b * NCOL;
#pragma unroll
          for (int a = 0; a < NA; ++a) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ahi = smem_desc(abase + a * kATile + kk * 32, 16, 1024, 2);
              const uint64_t alo = smem_desc(abase + (NA + a) * kATile + kk * 32, 16, 1024, 2);
              const uint64_t bhi = smem_desc(bbase + a * kBTile + kk * 32, 16, 1024, 2);
              const uint64_t blo = smem_desc(bbase + (NA + a) * kBTile + kk * 32, 16, 1024, 2);
              mma_tf32(d, ahi, bhi, idesc, (a == 0 && kk == 0) ? 0u : 1u);
              mma_tf32(d, ahi, blo, idesc, 1u);
              mma_tf32(d, alo, bhi, idesc, 1u);
            }
          }
          mma_commit(&empty_bar[s]);
          mma_commit(&tfull_bar[b]);
          if (c == NC - 1) mma_commit(&aempty_bar);
        }
        __syncwarp();
      }
    }
  } else {
    // ================= epilogue warps (8: two per TMEM lane quadrant, each half of the columns)
    const int ew = warp - 2;
    const uint32_t q = warp & 3;
    const int half = ew >> 2;
    const int rloc = q * 32 + lane;                   // row inside the 128-row tile
    double eS = 0.0, eT = 0.0, eST = 0.0;
    uint32_t it = 0, ci = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
      const bool rok = rb * 128 + rloc < l_local;
      for (int c = 0; c < NC; ++c, ++it, ++ci) {
        const uint32_t s = it % NS, r = it / NS;
        const uint32_t b = ci & 1, br = ci >> 1;
        static_assert(NCOL == 32, "epilogue handles 16 columns per warp half");
        const int c0 = half * 16;
        const int64_t j0 = (int64_t)c * NCOL + c0;
        float mh[16], ml[16];
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // mu loads issued before the barrier waits
          const float4 a = __ldg(reinterpret_cast<const float4*>(mu_hl + j0) + u);
          const float4 bb = __ldg(reinterpret_cast<const float4*>(mu_hl + m_pad + j0) + u);
          mh[4 * u] = a.x; mh[4 * u + 1] = a.y; mh[4 * u + 2] = a.z; mh[4 * u + 3] = a.w;
          ml[4 * u] = bb.x; ml[4 * u + 1] = bb.y; ml[4 * u + 2] = bb.z; ml[4 * u + 3] = bb.w;
        }
        mbar_wait(&full_bar[s], r & 1);
        mbar_wait(&tfull_bar[b], br & 1);
        tc_fence_after();
        const uint32_t tb = tmem + ((q * 32) << 16) + b * NCOL;
        const uint8_t* sx = sB + s * kStage + kVB;
        float s2 = 0.f, t2 = 0.f, st = 0.f;
        {
          uint32_t rv[16];
          tmem_ld16(tb + c0, rv);
          float xv[16];
          const float4* xrow = reinterpret_cast<const float4*>(sx + rloc * 128);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int g = (c0 >> 2) + u;              // logical 16-byte group of the row
            const float4 v = xrow[g ^ (rloc & 7)];    // SWIZZLE_128B
            xv[4 * u] = v.x; xv[4 * u + 1] = v.y; xv[4 * u + 2] = v.z; xv[4 * u + 3] = v.w;
          }
          tmem_ld_wait();
          float s2b = 0.f, t2b = 0.f, stb = 0.f;  // two chains per sum (even / odd t)
          const bool inside = rok && j0 + 16 <= m;  // no per-entry bounds selects
#pragma unroll
          for (int t = 0; t < 16; t += 2) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float xc = (xv[t + e] - mh[t + e]) - ml[t + e];
              float S = __uint_as_float(rv[t + e]);
              float T = xc - S;
              if (!inside) {
                const bool ok = rok && j0 + t + e < m;
                S = ok ? S : 0.f;
                T = ok ? T : 0.f;
              }
              float& a2 = e ? s2b : s2;
              float& b2 = e ? t2b : t2;
              float& c2 = e ? stb : st;
              a2 = fmaf(S, S, a2);
              b2 = fmaf(T, T, b2);
              c2 = fmaf(S, T, c2);
            }
          }
          s2 += s2b;
          t2 += t2b;
          st += stb;
        }
        eS += (double)s2;
        eT += (double)t2;
        eST += (double)st;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&tempty_bar[b]);
          mbar_arrive(&empty_bar[s]);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      eS += __shfl_xor_sync(0xFFFFFFFFu, eS, o);
      eT += __shfl_xor_sync(0xFFFFFFFFu, eT, o);
      eST += __shfl_xor_sync(0xFFFFFFFFu, eST, o);
    }
    if (lane == 0) { red[ew][0] = eS; red[ew][1] = eT; red[ew][2] = eST; }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    en_part[(int64_t)blockIdx.x * 4 + threadIdx.x] = t;
  }
  if (warp == 1) tmem_dealloc<(2 * NCOL < 32 ? 32 : 2 * NCOL)>(tmem);
}

CUresult encode2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                  uint32_t box_in, uint32_t box_out) {
  uint64_t dims[2] = {inner, outer};
  uint64_t strides[1] = {row_bytes};
  uint32_t box[2] = {box_in, box_out};
  uint32_t es[2] = {1, 1};
  return tma_encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int KP, int ND>
avd_status launch_k5(Ctx* c, const CUtensorMap& tmD, const CUtensorMap& tmW, int grid, const float* X) {
  constexpr uint32_t kStage = ((ND * 128 * 128 + 4 * KP * 128 + 1023) / 1024) * 1024;
  constexpr int NS = (int)((196u * 1024u) / kStage) > 6 ? 6 : (int)((196u * 1024u) / kStage);  // + ~26 KB static smem
  constexpr bool DB = 2 * 4 * KP <= 512;
  const size_t smem = (size_t)NS * kStage + 1024;
  AVD_CUDA(smem_attr(proj_i8_kernel<KP, ND, NS, DB>, (int)smem));
  proj_i8_kernel<KP, ND, NS, DB><<<grid, kK5Threads, smem, c->stream>>>(
      tmD, tmW, c->cfg.l_local, c->m_pad, c->l_pad, c->wsc, c->P, c->P_hl, c->colsumP_part, X, c->cfg.m,
      reinterpret_cast<const int*>(c->wsc + 384), c->V, c->mu, c->diag, c->k);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

template <int KP32, int NCOL>
avd_status launch_k8(Ctx* c, const CUtensorMap& tmP, const CUtensorMap& tmV, const CUtensorMap& tmX, int grid) {
  constexpr uint32_t kA = 2 * (KP32 / 32) * kTile;
  constexpr uint32_t kStage = 2 * (KP32 / 32) * NCOL * 128 + (NCOL / 32) * kTile;
  constexpr int NSF = (int)((220u * 1024u - kA) / kStage);
  constexpr int NS = NSF > 6 ? 6 : (NSF < 2 ? 2 : NSF);
  const size_t smem = kA + NS * kStage + 1024;
  AVD_CUDA(smem_attr(energy_tc_kernel<KP32, NCOL, NS>, (int)smem));
  energy_tc_kernel<KP32, NCOL, NS><<<grid, kPThreads, smem, c->stream>>>(tmP, tmV, tmX, c->cfg.l_local, c->cfg.m,
                                                                         c->l_pad, c->m_pad, c->mu_hl, c->m_pad,
                                                                         c->en_part);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace

bool project_tc_supported(const Ctx* c, const float* X) {
  return (c->cfg.m % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && c->k_pad <= 96;
}

// V_k -> tf32 hi/lo operand copy for K8 (once per pass)
avd_status launch_split_v(Ctx* c) {
  const int KP32 = (c->k_pad + 31) / 32 * 32;
  const int64_t n = c->m_pad * KP32;
  split_v_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c->stream>>>(c->V, c->cfg.m, c->k, KP32, c->m_pad, c->V_hl);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_project_tc(Ctx* c, const float* X) {
  const int KP = c->k_pad;
  const int KP32 = (KP + 31) / 32 * 32;
  const int64_t nrb = ceil_div(c->cfg.l_local, 128);
  const int grid = (int)std::min<int64_t>(nrb, c->num_sms);
  int8_t* wd = reinterpret_cast<int8_t*>(c->Vt_hl);  // W digit planes [4][KP][m_pad] (Vt_hl storage)
  CUtensorMap tmW, tmX, tmP, tmV;
  uint64_t wdims[2] = {(uint64_t)c->m_pad, (uint64_t)(4 * KP)};
  uint64_t wstr[1] = {(uint64_t)c->m_pad};
  uint32_t wbox[2] = {128, (uint32_t)KP}, es[2] = {1, 1};
  if (tma_encode_fn()(&tmW, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, wd, wdims, wstr, wbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      encode2d(&tmX, X, c->cfg.m, c->cfg.l_local, c->cfg.m * 4, 32, 128) != CUDA_SUCCESS ||
      encode2d(&tmP, c->P_hl, KP32, 2 * c->l_pad, KP32 * 4, 32, 128) != CUDA_SUCCESS ||
      encode2d(&tmV, c->V_hl, KP32, 2 * c->m_pad, KP32 * 4, 32, 32) != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (projection maps)");
    return AVD_ECUDA;
  }
  AVD_CUDA(cudaMemsetAsync(c->en_part, 0, sizeof(double) * 4 * c->n_proj_ctas, c->stream));
  AVD_CUDA(cudaMemsetAsync(c->colsumP_part, 0, sizeof(double) * KP * c->n_proj_ctas, c->stream));
  AVD_TRY(launch_split_v(c));
  int* spk = reinterpret_cast<int*>(c->wsc + 384);
  spiky_kernel<<<1, 1024, 0, c->stream>>>(c->colmax, c->ysq, c->cfg.m, (double)c->cfg.l_global, spk);
  AVD_LAUNCHED(c);
  split_w_kernel<<<KP, 256, 0, c->stream>>>(c->V, c->mu, c->mu0, c->diag, c->shift, c->cfg.m, c->m_pad, c->k, KP, wd,
                                             c->wsc, spk);
  AVD_LAUNCHED(c);
  const bool nd3 = c->nd == 3;
  switch (KP) {
#define CASE(K)                                                                      \
  case K:                                                                            \
    AVD_TRY((nd3 ? launch_k5<K, 3>(c, c->tmap_digits, tmW, grid, X) : launch_k5<K, 2>(c, c->tmap_digits, tmW, grid, X))); \
    break;
    CASE(16) CASE(32) CASE(48) CASE(64) CASE(80) CASE(96)
#undef CASE
    default: set_error("unsupported k_pad"); return AVD_EINVAL;
  }
  switch (KP32) {
    case 32: AVD_TRY((launch_k8<32, 32>(c, tmP, tmV, tmX, grid))); break;
    case 64: AVD_TRY((launch_k8<64, 32>(c, tmP, tmV, tmX, grid))); break;
    case 96: AVD_TRY((launch_k8<96, 32>(c, tmP, tmV, tmX, grid))); break;
    default: set_error("unsupported k_pad"); return AVD_EINVAL;
  }
  return AVD_OK;
}

}  // namespace avd
