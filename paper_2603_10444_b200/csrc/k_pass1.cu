// k_pass1.cu — K1+K2: the single HBM-streaming pass over X that feeds the rest of the path.
//
// One read of X (4 B/entry) produces, fused:
//   * fp64 column sums (mu = (1/l) X^T 1) and sum x^2 (||X||_F^2), whose
//     finiteness is the non-finite check; (#nonzero for |E_top| = min(n_top,
//     #nonzero), R4, comes exactly from the K6 level-0 histogram, k_select.cu);
//   * the Gram operand: every entry centred on a PROVISIONAL column centre mu0 (from a row
//     sample) and scaled by the column's power of two 2^shift_j, rounded with a deterministic
//     dither d (uniform on a 2^-9 grid in (-1/2, 1/2)):  q = rint((x - mu0_j) 2^shift_j + d) — nd balanced
//     base-128 int8 digits into ROW-MAJOR planes D_d[i][j] (MN-major operands of the tcgen05
//     kind::i8 Gram, k_gram.cu); and the exact integer column sums S_j = sum_i q_ij;
//   * the top-set candidates: entries whose |x| bit pattern falls in a first-level bin >= b0 are
//     appended as (key, global linear index).
// The Gram of the quantised matrix is then centred EXACTLY (k_eig.cu gram_finalize):
//   sum_i (q_ia - S_a/l)(q_ib - S_b/l) = sum_i q_ia q_ib - S_a S_b / l,
// its diagonal is taken from the exact sum_i q_ia^2 accumulated here (with 3 digits the Gram drops
// the two lowest digit-product classes, whose diagonal part is a positive bias) minus
// E_a = sum_i (q_ia^2 - y_ia^2) = sum_i e_ia (e_ia + 2 y_ia), e = q - y the rounding error, so the
// diagonal is the centred energy sum_i y_ia^2 - S_a^2 / l itself, free of the dither's noise
// (which would otherwise put an error of ~2 |x| d e on the energy of a column holding a massive
// activation x); the off-diagonal dither noise is zero-mean and independent across columns,
// so X~ = X - 1 mu^T never needs the exact mu before the pass.
//
// mu0, shift and b0 come from a 1/s row sample (sample_kernel, s = 16 at large l): shift maps
// the sampled max |x - mu0| below 2^(7nd-1); the digit range admits twice that.  An entry
// outside the range is counted (stats[m+3]); if any rank saw one, the quantisation is redone
// with the exact column ranges (requant path, same kernel without the statistics).
#include <cfloat>
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

namespace {
using namespace sm100;

constexpr int kT = 256;  // threads of the streaming kernels
constexpr int kNStg = 4;  // bulk-copy ring depth of the fused pass (stage = U = 4 rows x kT x 16 B)

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void hist_add(unsigned int* sh, uint32_t key, bool valid) {
  // warp-aggregated shared-memory histogram update (one atomic per distinct bin per warp)
  const uint32_t bin = valid ? (key >> 19) : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bin);
  const int leader = __ffs(peers) - 1;
  if (valid && (int)(threadIdx.x & 31) == leader) atomicAdd(&sh[bin], (unsigned)__popc(peers));
}

// ---------------------------------------------------------------- row sample
// Rows with global index gi % s == 0: column sums (fp64), max, min, and the 4096-bin histogram
// of |x| bits [30:19] that seeds the candidate threshold b0.
constexpr int kHistSub = 4;  // histogram on 1 of kHistSub sampled rows
template <int VEC>
__global__ void __launch_bounds__(kT) sample_kernel(const float* __restrict__ X, int64_t l, int64_t m, int64_t i0,
                                                   int s, int64_t row_offset, int64_t n_rows, int64_t rpc,
                                                   double* __restrict__ colsum_part,
                                                   float* __restrict__ colmax_part, float* __restrict__ colmin_part,
                                                   unsigned long long* __restrict__ hist1) {
  __shared__ unsigned int sh[kHistBins];
  for (int b = threadIdx.x; b < kHistBins; b += kT) sh[b] = 0;
  __syncthreads();
  const int64_t c0 = ((int64_t)blockIdx.x * kT + threadIdx.x) * VEC;
  const int64_t j0 = (int64_t)blockIdx.y * rpc, j1 = min(n_rows, j0 + rpc);
  const bool active = c0 < m;
  double cs[VEC];
  float mx[VEC], mn[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { cs[v] = 0.0; mx[v] = -FLT_MAX; mn[v] = FLT_MAX; }
  // sampled row jr has global sampled index gb + jr ((i0 + row_offset) is a multiple of s)
  const uint64_t gb = ((uint64_t)i0 + (uint64_t)row_offset) / (uint64_t)s;
  constexpr int R = 4;  // sampled rows in flight per thread
  for (int64_t jr = j0; jr < j1; jr += R) {
    float x[R][VEC];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const bool ok = active && jr + u < j1;
      const int64_t i = i0 + (jr + u) * s;
      if constexpr (VEC == 4) {
        const float4 t = ok ? __ldg(reinterpret_cast<const float4*>(X + i * m + c0)) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
      } else {
        x[u][0] = ok ? __ldg(X + i * m + c0) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
      if (jr + u >= j1) break;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const uint32_t key = __float_as_uint(x[u][v]) & 0x7FFFFFFFu;
        const bool fin = key < 0x7F800000u;
        if (active && fin) {
          cs[v] += (double)x[u][v];
          mx[v] = fmaxf(mx[v], x[u][v]);
          mn[v] = fminf(mn[v], x[u][v]);
        }
      }
      // the |x| histogram only needs every kHistSub-th sampled row (enough for a top-0.1% bin)
      if ((gb + (uint64_t)(jr + u)) % kHistSub == 0) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const uint32_t key = __float_as_uint(x[u][v]) & 0x7FFFFFFFu;
          hist_add(sh, key, active && key < 0x7F800000u && key != 0);
        }
      }
    }
  }
  if (active)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      colsum_part[(int64_t)blockIdx.y * m + c0 + v] = cs[v];
      colmax_part[(int64_t)blockIdx.y * m + c0 + v] = mx[v];
      colmin_part[(int64_t)blockIdx.y * m + c0 + v] = mn[v];
    }
  __syncthreads();
  for (int b = threadIdx.x; b < kHistBins; b += kT)
    if (sh[b]) atomicAdd(&hist1[b], (unsigned long long)sh[b]);
}

// fixed-order reduction of the sample partials -> samp[0..m) column sums, samp[m] = #rows;
// CTA = 32 columns x 8 row groups as in pass1_reduce_kernel
__global__ void __launch_bounds__(256) sample_reduce_kernel(int64_t m, int r1, double n_rows,
                                                            const double* __restrict__ colsum_part,
                                                            const float* __restrict__ colmax_part,
                                                            const float* __restrict__ colmin_part,
                                                            double* __restrict__ samp, float* __restrict__ smax,
                                                            float* __restrict__ smin) {
  __shared__ double s_s[8][32];
  __shared__ float s_mx[8][32], s_mn[8][32];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + c;
  double s = 0.0;
  float mx = -FLT_MAX, mn = FLT_MAX;
  if (j < m) {
    // four partial rows in flight (independent accumulators, combined in a fixed order)
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    int r = g;
    for (; r + 24 < r1; r += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t o = (int64_t)(r + 8 * u) * m + j;
        s4[u] += colsum_part[o];
        mx = fmaxf(mx, colmax_part[o]);
        mn = fminf(mn, colmin_part[o]);
      }
    }
    for (; r < r1; r += 8) {
      s4[0] += colsum_part[(int64_t)r * m + j];
      mx = fmaxf(mx, colmax_part[(int64_t)r * m + j]);
      mn = fminf(mn, colmin_part[(int64_t)r * m + j]);
    }
    s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
  }
  s_s[g][c] = s; s_mx[g][c] = mx; s_mn[g][c] = mn;
  __syncthreads();
  if (g == 0 && j < m) {
    for (int h = 1; h < 8; ++h) { s += s_s[h][c]; mx = fmaxf(mx, s_mx[h][c]); mn = fminf(mn, s_mn[h][c]); }
    samp[j] = s;
    smax[j] = mx;
    smin[j] = mn;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) samp[m] = n_rows;
}

// Quantiser parameters from column centres and ranges:
//   mu0_j = fl32(centre), shift_j = (7 nd - 1) - (ilogb(a_j) + 1), a_j = max|x - mu0_j| over the
//   range given, so the range maps below 2^(7nd-1) and the digit range (2^(7nd) - 2^7) admits a
//   factor 2 beyond it;  qscale = 2^shift (fp32, exact), qoff = -mu0 * 2^shift (exact).
// exact == 0: centre = sample mean, range = sample max/min; also picks b0 from the sampled
// histogram: the largest bin whose scaled tail count covers 2 n_top + 256 s (conservative; K6
// verifies with exact counts and falls back to streaming X when it does not cover |E_top|).
// exact == 1: the same centre, range = the exact max |x - mu0| of the fused pass (requant path).
__global__ void prepare_kernel(int64_t m, int64_t m_pad, int nd, int exact, int64_t n_top, int s,
                               const double* __restrict__ centre_sum, float* __restrict__ mu0,
                               const float* __restrict__ cmax, const float* __restrict__ cmin,
                               const unsigned long long* __restrict__ hist1, int32_t* __restrict__ shift,
                               float* __restrict__ qscale, float* __restrict__ qoff, DevPlan* __restrict__ dp) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m_pad) {
    int32_t sh = 0;
    float sc = 0.f, off = 0.f;
    if (j < m) {
      // sample: centre = fl32(sample mean), a = sampled max |x - centre|; exact (requant): the
      // same centre (kept in mu0) and a = the exact max |x - mu0| measured by the fused pass
      const float c0 = exact ? mu0[j] : (centre_sum[m] > 0.0 ? (float)(centre_sum[j] / centre_sum[m]) : 0.f);
      const double a = exact ? (double)cmax[j] : fmax((double)cmax[j] - (double)c0, (double)c0 - (double)cmin[j]);
      if (!exact) mu0[j] = c0;
      if (a > 0.0 && a < 1e300) sh = (7 * nd - 1) - (ilogb(a) + 1);
      else if (!exact) sh = 100;  // no sampled range: any deviation overflows -> exact requant
      // 2^sh stays a normal fp32 and mu0 2^sh stays finite (qoff); a finite fp32 range a < 2^128
      // gives sh >= 7 nd - 129 > -126, so the exact-range requant can never overflow the digits
      // (|y| <= a 2^sh < 2^(7 nd - 1)), and for x != mu0, |x - mu0| >= |mu0| 2^-25 keeps
      // |mu0| 2^sh <= 2^(7 nd + 24) whenever the range is measured
      sh = max(-126, min(126, sh));
      if (c0 != 0.f) sh = min(sh, 125 - ilogbf(fabsf(c0)));
      sc = __int_as_float((sh + 127) << 23);
      off = -c0 * sc;
    }
    shift[j] = sh;
    qscale[j] = sc;
    qoff[j] = off;
  }
  if (exact || blockIdx.x != 0 || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const unsigned long long sh = (unsigned long long)s * kHistSub;  // rows per histogrammed row
  const unsigned long long need = 2ull * (unsigned long long)n_top + 256ull * sh;
  constexpr int per = kHistBins / 32;
  const int hi = kHistBins - 1 - lane * per;  // lane covers bins (hi-per, hi]
  unsigned long long mine = 0;
  for (int b = hi; b > hi - per; --b) mine += hist1[b] * sh;
  unsigned long long incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned long long excl = incl - mine;
  int b0 = -1;
  if (excl < need && incl >= need) {
    unsigned long long cum = excl;
    int b = hi;
    for (; b > hi - per; --b) {
      cum += hist1[b] * sh;
      if (cum >= need) break;
    }
    b0 = b;
  }
  // lowest lane holding a crossing wins; none -> every nonzero entry is a candidate (b0 = 0)
  for (int o = 16; o > 0; o >>= 1) b0 = max(b0, __shfl_xor_sync(0xFFFFFFFFu, b0, o));
  if (lane == 0) {
    dp->b0 = b0 < 0 ? 0 : b0;
    dp->b1 = 0;
    dp->b2 = 0;
    dp->cnt_gt = 0;
    dp->cand_count = 0;
  }
}

// pack the low bytes of four ints into one word (byte v <- value v)
__device__ __forceinline__ uint32_t pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm((uint32_t)a, (uint32_t)b, 0x0040), __byte_perm((uint32_t)c, (uint32_t)d, 0x0040), 0x5410);
}

// ---------------------------------------------------------------- the fused pass
// FULL: statistics + candidates + digits; !FULL: digits + S + E only (requant path).
// Thread: VEC consecutive columns, rows [r0, r1) of its chunk, U rows in flight.  Per entry the
// hot loop does the dithered rounding, the digit split and packing, the exact integer sums of q
// and q^2, the rounding-error term q^2 - y^2, |y| max (the digit-range check and the exact range for a
// requant), the x and x^2 sums and a running max of the |x| bit patterns; only when that max
// reaches the candidate bin does the warp build candidate masks and append them (one scan and
// one atomic per warp).  Full U-row groups run without bounds checks; pointers are advanced,
// not recomputed.
// Candidate slots: each warp owns a block of slots [base, base + cap) of the candidate list,
// reserved from the global cursor cand_cnt[0]; unused slots of a closed block are holes with
// key 0 (never a candidate key, skipped by K6).  cand_cnt[1] counts the real candidates.
constexpr uint32_t kCandBlk = 64;
struct CandBlk {
  unsigned long long base;
  uint32_t used, cap, real, pad;
};
__device__ __forceinline__ void close_cand_block(uint32_t* __restrict__ cand_key, int64_t cand_cap,
                                                 unsigned long long base, uint32_t used, uint32_t cap, int lane) {
  for (uint32_t t = used + (uint32_t)lane; t < cap; t += 32)
    if (base + t < (unsigned long long)cand_cap) cand_key[base + t] = 0u;
}

template <int ND, int VEC, bool FULL, bool SMEM>
__device__ __forceinline__ void pass1_rows(int nrows, const float* __restrict__ xp, const float4* xs, int64_t m, int8_t* __restrict__ dp,
                                           int64_t plane, int64_t m_pad, uint32_t srow0, uint32_t kd, const float* sc,
                                           const float* off, const uint32_t* colh, uint32_t klo, uint32_t kspan,
                                           uint64_t lin0, int lane, CandBlk* cb, uint32_t* __restrict__ cand_key,
                                           uint64_t* __restrict__ cand_idx, unsigned long long* __restrict__ cand_cnt,
                                           int64_t cand_cap, double* s, double* yq,
                                           std::conditional_t<ND == 2, int, long long>* ws, float* es, float* ym, bool active, bool writer) {
  constexpr int U = 4;
  constexpr int DB = ND == 2 ? 9 : 2;  // dither grid bits (see below)
  constexpr int kW0 = ND == 2 ? 64 : 64 + 64 * 128;
  float x[U][VEC];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = active && u < nrows;
    if constexpr (SMEM) {  // prefetched by cp.async (zero-filled past the end)
      const float4 t = u < nrows ? xs[u * kT] : make_float4(0.f, 0.f, 0.f, 0.f);  // tail: stale slot
      x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
    } else if constexpr (VEC == 4) {
      const float4 t = ok ? __ldcs(reinterpret_cast<const float4*>(xp + u * m)) : make_float4(0.f, 0.f, 0.f, 0.f);
      x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
    } else {
      x[u][0] = ok ? __ldcs(xp + u * m) : 0.f;
    }
  }
  // kd = 1.0f | (1 << (22 - DB)) (the exponent and the half-step of the dither grid) arrives as a
  // kernel argument so the mask-and-or below is one LOP3 (two immediates do not fit one)
  float kmax = 0.f;
  float py[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) py[v] = 0.f;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (u >= nrows) break;
    const uint32_t srow = srow0 + (uint32_t)u * 0x9E3779B1u;
    int w[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      // dithered rounding: q = floor(y + u) with u = (k + 1/2) 2^-DB uniform, k < 2^DB (unbiased
      // stochastic rounding), taken as floor(y + D) - 1 with D = 1 + u built from hash bits;
      // y = (x - mu0) 2^shift.  y + D is exact in fp32 for integer y (|y| < 2^(7nd) - 2), so
      // exactly representable data stays exact (tests/test_gpu_parity.py planted case)
      // DB bits from the high word of a 32 x 32 multiplicative hash, in place at mantissa bits
      // 22 .. 23 - DB
      const uint32_t h = __umulhi(srow ^ colh[v], 0x85EBCA6Bu);
      const float D = __uint_as_float((h & (((1u << DB) - 1u) << (23 - DB))) | kd);
      const float y = fmaf(x[u][v], sc[v], off[v]);
      const float t = __fadd_rd(y + D, 12582912.0f);  // 1.5 * 2^23 + floor(y + D)
      // w = q + kW0 (kW0 = 64 sum_{i < nd-1} 128^i): every digit is a plain bit field of w
      w[v] = __float_as_int(t) - (0x4B400000 + 1 - kW0);
      const float e = (t - 12582913.0f) - y;  // q - y
      es[v] = fmaf(e, e, es[v]);
      if (FULL) py[v] = fmaf(y, y, py[v]);  // the exact centred energy (diagonal of G)
      ym[v] = fmaxf(ym[v], fabsf(y));
      ws[v] += w[v];
      if (FULL) kmax = fmaxf(kmax, fabsf(x[u][v]));
    }
    if (writer) {
      int8_t* row = dp + u * m_pad;
      if constexpr (ND == 2 && VEC == 4) {
        // balanced base-128 digits of q = w - 64, four entries at a time: hi = w >> 7 (bits
        // 14..7 of w), lo = (w & 127) - 64 (bits 6..0 of w, minus 64 as a byte)
        const uint32_t A = __byte_perm((uint32_t)w[0], (uint32_t)w[1], 0x5140);
        const uint32_t B = __byte_perm((uint32_t)w[2], (uint32_t)w[3], 0x5140);
        const uint32_t P0 = __byte_perm(A, B, 0x5410);  // byte v = bits 7..0 of w[v]
        const uint32_t P1 = __byte_perm(A, B, 0x7632);  // byte v = bits 15..8 of w[v]
        const uint32_t hi = ((P1 << 1) & 0xFEFEFEFEu) | ((P0 >> 7) & 0x01010101u);
        const uint32_t lo = ((P0 & 0x7F7F7F7Fu) | ((P0 << 1) & 0x80808080u)) ^ 0xC0C0C0C0u;
        __stcs(reinterpret_cast<unsigned int*>(row), hi);
        __stcs(reinterpret_cast<unsigned int*>(row + plane), lo);
      } else {
        // plane 0 = most significant digit w >> 7(nd-1); plane nd-1-i = ((w >> 7i) & 127) - 64
        int dg[ND][VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          dg[0][v] = w[v] >> (7 * (ND - 1));
#pragma unroll
          for (int i = 0; i < ND - 1; ++i) dg[ND - 1 - i][v] = ((w[v] >> (7 * i)) & 127) - 64;
        }
#pragma unroll
        for (int dd = 0; dd < ND; ++dd) {
          if constexpr (VEC == 4) {
            __stcs(reinterpret_cast<unsigned int*>(row + dd * plane), pack4(dg[dd][0], dg[dd][1], dg[dd][2], dg[dd][3]));
          } else {
            row[dd * plane] = (int8_t)dg[dd][0];
          }
        }
      }
    }
  }
  if (FULL) {
    // candidates (key in [klo, 0x7F800000)): rare, so only warps that saw one build masks
    // (as fp32 compares against thr = float(klo): NaN fails them; an infinity passes, but a
    // non-finite X ends the call with AVD_ENONFINITE before the candidates are used)
    const float thr = __uint_as_float(klo);
    if (__any_sync(0xFFFFFFFFu, kmax >= thr)) {
      uint32_t cmask = 0;
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          if (fabsf(x[u][v]) >= thr) cmask |= 1u << (u * VEC + v);  // rows past the end hold 0
        }
      const uint32_t cnt = __popc(cmask);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
      // slots come from this warp's block (reserved from the global cursor kCandBlk at a time);
      // only a warp whose block runs out goes to the global atomic
      unsigned long long bbase = cb->base;
      uint32_t used = cb->used, bcap = cb->cap;
      if (used + total > bcap) {
        close_cand_block(cand_key, cand_cap, bbase, used, bcap, lane);
        const uint32_t want = max((uint32_t)kCandBlk, total);
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(cand_cnt, (unsigned long long)want);
        bbase = __shfl_sync(0xFFFFFFFFu, b, 0);
        used = 0;
        bcap = want;
      }
      unsigned long long base = bbase + used + (incl - cnt);
      __syncwarp();
      if (lane == 0) { cb->base = bbase; cb->used = used + total; cb->cap = bcap; cb->real += total; }
      __syncwarp();
      if constexpr (SMEM) {
        // one step per candidate of this thread; the values are re-read from its ring slot
        const float* xsf = reinterpret_cast<const float*>(xs);
        while (cmask) {
          const int bit = __ffs(cmask) - 1;
          cmask &= cmask - 1u;
          const int u = bit / VEC, v = bit % VEC;
          if (base < (unsigned long long)cand_cap) {
            cand_key[base] = __float_as_uint(xsf[u * kT * 4 + v]) & 0x7FFFFFFFu;
            cand_idx[base] = lin0 + (uint64_t)u * (uint64_t)m + (uint64_t)v;
          }
          ++base;
        }
      } else if (cmask) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int v = 0; v < VEC; ++v)
            if ((cmask >> (u * VEC + v)) & 1u) {
              if (base < (unsigned long long)cand_cap) {
                cand_key[base] = __float_as_uint(x[u][v]) & 0x7FFFFFFFu;
                cand_idx[base] = lin0 + (uint64_t)u * (uint64_t)m + (uint64_t)v;
              }
              ++base;
            }
      }
    }
    // fp64 accumulation of U-row fp32 partial sums (each partial rounds once, ~2^-24 relative)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float ps = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) ps += x[u][v];  // rows past the end were loaded as 0
      s[v] += (double)ps;
      yq[v] += (double)py[v];
    }
  }
}

template <int ND, int VEC, bool FULL>
__global__ void __launch_bounds__(kT, ND == 2 ? 3 : 2) pass1_kernel(
    const float* __restrict__ X, int64_t l, int64_t m, int64_t m_pad, int64_t l_pad, int64_t rpc, int64_t row_offset,
    const float* __restrict__ qscale, const float* __restrict__ qoff, uint32_t seed32, uint32_t kd,
    int8_t* __restrict__ digits,
    const DevPlan* __restrict__ dplan, uint32_t* __restrict__ cand_key, uint64_t* __restrict__ cand_idx,
    unsigned long long* __restrict__ cand_cnt, int64_t cand_cap, double* __restrict__ colsum_part,
    float* __restrict__ ymax_part, long long* __restrict__ qsum_part, double* __restrict__ ysq_part,
    float* __restrict__ qerr_part) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const int64_t c0 = ((int64_t)blockIdx.x * kT + threadIdx.x) * VEC;
  const int64_t r0 = (int64_t)blockIdx.y * rpc;
  const int64_t r1 = min(l, r0 + rpc);
  const bool active = c0 < m;
  const bool writer = c0 < m_pad;  // digit columns [m, m_pad) come out zero (x = 0, scale 1, centre 0)
  const int64_t plane = l_pad * m_pad;
  __shared__ CandBlk cblk[kT / 32];
  CandBlk* cb = &cblk[threadIdx.x >> 5];
  if (lane == 0) *cb = CandBlk{0ull, 0u, 0u, 0u, 0u};
  __syncwarp();
  // VEC == 4: the bulk-copy ring's barriers; empty_bar counts the warps holding a digit column
  __shared__ __align__(8) uint64_t full_bar[kNStg], empty_bar[kNStg];
  if constexpr (VEC == 4) {
    if (threadIdx.x == 0) {
      const int64_t cols = m_pad - (int64_t)blockIdx.x * kT * 4;  // > 0 for every launched CTA
      const uint32_t nw = (uint32_t)min((int64_t)kT / 32, ceil_div(cols, (int64_t)128));
      for (int t = 0; t < kNStg; ++t) { mbar_init(&full_bar[t], 1); mbar_init(&empty_bar[t], nw); }
      fence_mbar_init();
    }
    __syncthreads();
  }
  // whole warps take part (the candidate append uses warp collectives); lanes past m load nothing
  if (__any_sync(0xFFFFFFFFu, writer)) {
    const int64_t cc = writer ? c0 : 0;
    float sc[VEC], off[VEC];
    uint32_t colh[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      sc[v] = active ? qscale[c0 + v] : 1.f;
      off[v] = active ? qoff[c0 + v] : 0.f;
      colh[v] = ((uint32_t)(c0 + v) * 0x2545F491u) ^ 0x68E31DA4u;  // cheap to rematerialise
    }
    // candidate test as one unsigned compare: key in [max(1, b0 << 19), 0x7F800000)
    const uint32_t klo = FULL ? max(1u, (uint32_t)dplan->b0 << 19) : 0xFFFFFFFFu;
    const uint32_t kspan = 0x7F800000u - klo;
    double s[VEC];
    // sums of w = q + kW0 and of w^2 (the digit offset; removed below)
    std::conditional_t<ND == 2, int, long long> ws[VEC];
    double yq[VEC];
    float es[VEC], ym[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) { s[v] = 0.0; yq[v] = 0.0; ws[v] = 0; es[v] = 0.f; ym[v] = 0.f; }
    const float* xp = X + r0 * m + (active ? c0 : 0);
    int8_t* dp = digits + r0 * m_pad + cc;
    uint32_t srow0 = (uint32_t)(row_offset + r0) * 0x9E3779B1u + seed32;
    uint64_t lin0 = (uint64_t)(row_offset + r0) * (uint64_t)m + (uint64_t)c0;
    if constexpr (VEC == 4) {
      // bulk-copy ring: thread 0 streams group g (U rows x the CTA's kT * 16 B, contiguous in X)
      // into stage g % kNStg with cp.async.bulk, kNStg - 1 groups ahead; the warps release a
      // stage through empty_bar once they have computed on it.  Slots of lanes past m are
      // zeroed once and never written by the copies.
      extern __shared__ __align__(16) float4 xring[];  // [kNStg][U][kT]
      const int ng = (int)ceil_div(r1 - r0, U);
      const int64_t cblk = (int64_t)blockIdx.x * kT * 4;
      const uint32_t row_bytes = (uint32_t)max((int64_t)0, min((int64_t)kT * 4, m - cblk)) * 4u;
      if (!active)
        for (int t = 0; t < kNStg * U; ++t) xring[t * kT + threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
      auto issue = [&](int g) {  // thread 0
        const int st = g % kNStg;
        const int64_t i = r0 + (int64_t)g * U;
        const int nr = (int)min((int64_t)U, r1 - i);
        mbar_arrive_expect_tx(&full_bar[st], (uint32_t)nr * row_bytes);
        if (row_bytes)
          for (int u = 0; u < nr; ++u)
            bulk_load_1d(&xring[(st * U + u) * kT], X + (i + u) * m + cblk, row_bytes, &full_bar[st]);
      };
      if (threadIdx.x == 0)
        for (int g = 0; g < kNStg - 1 && g < ng; ++g) issue(g);
      for (int g = 0; g < ng; ++g) {
        const int st = g % kNStg;
        if (threadIdx.x == 0 && g + kNStg - 1 < ng) {
          const int gn = g + kNStg - 1;
          if (gn >= kNStg) mbar_wait_sleep(&empty_bar[gn % kNStg], (uint32_t)((gn / kNStg) - 1) & 1u);
          issue(gn);
        }
        mbar_wait_sleep(&full_bar[st], (uint32_t)(g / kNStg) & 1u);
        const int nrows = (int)min((int64_t)U, r1 - (r0 + (int64_t)g * U));
        pass1_rows<ND, VEC, FULL, true>(nrows, xp, &xring[(st * U) * kT + threadIdx.x], m, dp, plane, m_pad,
                                        srow0, kd, sc, off, colh, klo, kspan, lin0, lane, cb, cand_key, cand_idx, cand_cnt,
                                        cand_cap, s, yq, ws, es, ym, active, writer);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
        dp += U * m_pad;
        srow0 += (uint32_t)U * 0x9E3779B1u;
        lin0 += (uint64_t)U * (uint64_t)m;
      }
    } else {
      int64_t i = r0;
      for (; i + U <= r1; i += U) {
        pass1_rows<ND, VEC, FULL, false>(U, xp, nullptr, m, dp, plane, m_pad, srow0, kd, sc, off, colh, klo, kspan, lin0,
                                         lane, cb, cand_key, cand_idx, cand_cnt, cand_cap, s, yq, ws, es, ym,
                                         active, writer);
        xp += U * m;
        dp += U * m_pad;
        srow0 += (uint32_t)U * 0x9E3779B1u;
        lin0 += (uint64_t)U * (uint64_t)m;
      }
      if (i < r1)
        pass1_rows<ND, VEC, FULL, false>((int)(r1 - i), xp, nullptr, m, dp, plane, m_pad, srow0, kd, sc, off, colh, klo,
                                         kspan, lin0, lane, cb, cand_key, cand_idx, cand_cnt, cand_cap, s, yq, ws,
                                         es, ym, active, writer);
    }
    if (FULL) {  // close this warp's candidate block; publish its real count
      __syncwarp();
      const CandBlk st = *cb;
      close_cand_block(cand_key, cand_cap, st.base, st.used, st.cap, lane);
      if (lane == 0 && st.real) atomicAdd(cand_cnt + 1, (unsigned long long)st.real);
    }
    if (active) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int64_t o = (int64_t)blockIdx.y * m + c0 + v;
        constexpr long long W0 = ND == 2 ? 64 : 64 + 64 * 128;
        const long long n = r1 - r0, sw = (long long)ws[v];
        qsum_part[o] = sw - W0 * n;                     // sum q
        if (FULL) ysq_part[o] = yq[v];                  // sum (x - mu0)^2 2^(2 shift)
        qerr_part[o] = es[v];
        ymax_part[o] = ym[v];
        if (FULL) colsum_part[o] = s[v];
      }
    }
  }
}

// Fixed-order reduction of the per-chunk partials -> stats[0..m) colsum, stats[m+3] = #columns
// whose digits overflowed, colmax[j] = max |x - mu0_j| (the exact range about the quantiser
// centre, for a requant), qsum_local / qerr_local, and ysq[j] = sum_i (x_ij - mu0_j)^2 (fp64, in
// units of x: the scale 2^shift is a power of two) from which the diagonal of G and ||X||^2 are
// formed exactly (k_eig.cu gram_finalize / trace).
// CTA = 32 columns x 8 row groups (256 threads): thread (g, c) sums the chunks r = g (mod 8) of
// column j0 + c (coalesced 32-column rows), the 8 group sums are combined in a fixed order.
template <int ND>
__global__ void __launch_bounds__(256) pass1_reduce_kernel(
    int64_t m, int r1, int full, const double* __restrict__ colsum_part, const float* __restrict__ ymax_part,
    const long long* __restrict__ qsum_part, const double* __restrict__ ysq_part,
    const float* __restrict__ qerr_part, const float* __restrict__ qscale, double* __restrict__ stats,
    float* __restrict__ colmax, long long* __restrict__ qsum_local, double* __restrict__ qerr_local,
    double* __restrict__ ysq) {
  __shared__ long long s_qs[8][32];
  __shared__ double s_qe[8][32], s_cs[8][32], s_qq[8][32];
  __shared__ float s_ym[8][32];
  const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + c;
  long long qs = 0;
  double qe = 0.0, cs = 0.0, qq = 0.0;
  float ym = 0.f;
  if (j < m) {
    // four partial rows in flight (independent accumulators, combined in a fixed order)
    double qe4[4] = {0, 0, 0, 0}, cs4[4] = {0, 0, 0, 0}, qq4[4] = {0, 0, 0, 0};
    int r = g;
    for (; r + 24 < r1; r += 32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t o = (int64_t)(r + 8 * u) * m + j;
        qs += qsum_part[o];
        qe4[u] += (double)qerr_part[o];
        ym = fmaxf(ym, ymax_part[o]);
        if (full) { cs4[u] += colsum_part[o]; qq4[u] += ysq_part[o]; }
      }
    }
    for (; r < r1; r += 8) {
      const int64_t o = (int64_t)r * m + j;
      qs += qsum_part[o];
      qe4[0] += (double)qerr_part[o];
      ym = fmaxf(ym, ymax_part[o]);
      if (full) { cs4[0] += colsum_part[o]; qq4[0] += ysq_part[o]; }
    }
    qe = (qe4[0] + qe4[1]) + (qe4[2] + qe4[3]);
    cs = (cs4[0] + cs4[1]) + (cs4[2] + cs4[3]);
    qq = (qq4[0] + qq4[1]) + (qq4[2] + qq4[3]);
  }
  s_qs[g][c] = qs; s_qq[g][c] = qq; s_qe[g][c] = qe; s_cs[g][c] = cs; s_ym[g][c] = ym;
  __syncthreads();
  if (g == 0 && j < m) {
    for (int h = 1; h < 8; ++h) {
      qs += s_qs[h][c]; qq += s_qq[h][c]; qe += s_qe[h][c]; cs += s_cs[h][c]; ym = fmaxf(ym, s_ym[h][c]);
    }
    qsum_local[j] = qs;
    qsum_local[m + j] = 0;  // (unused half of the exchange buffer)
    qerr_local[j] = qe;
    if (full) {
      stats[j] = cs;
      const float isc = 1.0f / qscale[j];  // 2^-shift, exact
      ysq[j] = qq * (double)isc * (double)isc;
      // exact max |x - mu0_j| (power-of-two scale: exact), the range of a requant; |y| beyond
      // the digit range (top digit outside [-127, 127]) counts as an overflow of column j
      constexpr float kYLim = ND == 2 ? 16319.0f : 2088895.0f;
      colmax[j] = ym / qscale[j];
      if (!(ym <= kYLim)) atomicAdd(&stats[m + 3], 1.0);
    }
  }
}

// After the statistics exchange: mu (fp64) and its fp32 hi/lo pair for the projection pass,
// |E_top| = min(n_top, #nonzero), the non-finite count.
__global__ void finish_kernel(int64_t m, int64_t m_pad, int64_t l_global, int64_t n_top,
                              const double* __restrict__ stats, double* __restrict__ mu, float* __restrict__ mu_hl,
                              DevPlan* __restrict__ dp, const float* __restrict__ colmax,
                              const int32_t* __restrict__ shift, int nd) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m && !isfinite(stats[j])) atomicAdd(reinterpret_cast<unsigned long long*>(&dp->nonfinite), 1ull);
  // bits of resolution an exact-range re-quantisation would cost column j: the measured
  // max |x - mu0| against the range the sampled scale planned for (2^(7nd-1) in y units)
  if (j < m) {
    const double r = ldexp((double)colmax[j], shift[j] - (7 * nd - 1));
    if (r > 1.0 && r < 1e300) atomicMax(&dp->range_bits, ilogb(r) + 1);
  }
  if (j < m_pad) {
    float mh = 0.f, ml = 0.f;
    if (j < m) {
      const double mj = stats[j] / (double)l_global;
      mu[j] = mj;
      mh = (float)mj;
      ml = (float)(mj - (double)mh);
    }
    mu_hl[j] = mh;
    mu_hl[m_pad + j] = ml;
  }
}

// exchange slot for the global candidate decision: [count, overflowed]
__global__ void cand_publish_kernel(const unsigned long long* __restrict__ cnt, int64_t cap,
                                    long long* __restrict__ out) {
  out[0] = (long long)cnt[1];                                   // real candidates
  out[1] = (long long)(cnt[0] > (unsigned long long)cap ? 1 : 0);  // slots (with holes) past cap
}

bool vec4(const Ctx* c, const float* X) {
  return (c->cfg.m % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
}

uint32_t dither_seed(const Ctx* c) {
  return (uint32_t)(c->cfg.seed * 0x9E3779B97F4A7C15ull >> 32) ^ 0xA5A5A5A5u;
}

}  // namespace

int stats_sample_step(int64_t l_global) {
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(16, l_global / 4096));
  int s = 1;
  while (s * 2 <= want) s *= 2;  // power of two
  return s;
}

// Stage 1: the row sample -> samp, smax, smin, hist1 (exchange buffers).
avd_status launch_sample(Ctx* c, const float* X) {
  const int64_t m = c->cfg.m, l = c->cfg.l_local;
  const int s = stats_sample_step(c->cfg.l_global);
  const int64_t i0 = (s - c->cfg.row_offset % s) % s;  // first local row with global index % s == 0
  const int64_t n_rows = i0 < l ? ceil_div(l - i0, s) : 0;
  const bool vec = vec4(c, X);
  const int VEC = vec ? 4 : 1;
  const int ncb = (int)ceil_div(m, (int64_t)kT * VEC);
  const int r1 = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>((int64_t)c->r1, ceil_div(4LL * c->num_sms, ncb)), std::max<int64_t>(n_rows, 1)));
  const int64_t rpc = ceil_div(std::max<int64_t>(n_rows, 1), r1);
  AVD_CUDA(cudaMemsetAsync(c->hist1, 0, sizeof(unsigned long long) * kHistBins, c->stream));
  dim3 grid(ncb, r1);
  if (vec)
    sample_kernel<4><<<grid, kT, 0, c->stream>>>(X, l, m, i0, s, c->cfg.row_offset, n_rows, rpc, c->colsum_part, c->colmax_part,
                                                 c->colmin_part, c->hist1);
  else
    sample_kernel<1><<<grid, kT, 0, c->stream>>>(X, l, m, i0, s, c->cfg.row_offset, n_rows, rpc, c->colsum_part, c->colmax_part,
                                                 c->colmin_part, c->hist1);
  AVD_LAUNCHED(c);
  sample_reduce_kernel<<<(unsigned)ceil_div(m, 32), 256, 0, c->stream>>>(m, r1, (double)n_rows, c->colsum_part,
                                                                         c->colmax_part, c->colmin_part, c->samp,
                                                                         c->smax, c->smin);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// Stage 2: quantiser parameters from the (exchanged) sample, then the fused pass.
avd_status launch_pass1(Ctx* c, const float* X, bool full) {
  const int64_t m = c->cfg.m, l = c->cfg.l_local;
  const int s = stats_sample_step(c->cfg.l_global);
  if (full) {
    prepare_kernel<<<(unsigned)ceil_div(c->m_pad, 256), 256, 0, c->stream>>>(
        m, c->m_pad, c->nd, 0, c->plan.n_top, s, c->samp, c->mu0, c->smax, c->smin, c->hist1, c->shift, c->qscale,
        c->qoff, c->dplan);
    AVD_LAUNCHED(c);
  } else {
    prepare_kernel<<<(unsigned)ceil_div(c->m_pad, 256), 256, 0, c->stream>>>(
        m, c->m_pad, c->nd, 1, c->plan.n_top, s, c->stats, c->mu0, c->colmax, c->colmin, c->hist1,
        c->shift, c->qscale, c->qoff, c->dplan);
    AVD_LAUNCHED(c);
  }
  const bool vec = vec4(c, X);
  const int VEC = vec ? 4 : 1;
  const int ncb = (int)ceil_div(c->m_pad, (int64_t)kT * VEC);
  // one full wave: (CTAs resident per SM) x SMs, split over the column blocks (<= c->r1 chunks,
  // <= 65536 rows per chunk for the int32 sums of q)
  const int per_sm = (c->nd == 2 && vec) ? 3 : 2;
  int64_t want = std::max<int64_t>(1, (int64_t)per_sm * c->num_sms / ncb);
  want = std::min<int64_t>(want, c->r1);
  want = std::max<int64_t>(want, ceil_div(l, 65536));
  const int64_t rpc = round_up(ceil_div(l, want), 4);
  const int r1 = (int)ceil_div(l, rpc);
  if (full) {
    AVD_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(double) * (m + 4), c->stream));
    AVD_CUDA(cudaMemsetAsync(c->cand_cnt, 0, 2 * sizeof(unsigned long long), c->stream));
  }
  // digit-plane rows [l_local, l_pad) are zero (the Gram sums over them)
  if (c->l_pad > l)
    for (int d = 0; d < c->nd; ++d)
      AVD_CUDA(cudaMemsetAsync(c->digits + ((int64_t)d * c->l_pad + l) * c->m_pad, 0, (size_t)(c->l_pad - l) * c->m_pad,
                               c->stream));
  dim3 grid(ncb, r1);
  const uint32_t seed32 = dither_seed(c);
  const uint32_t kd = 0x3F800000u | (1u << (22 - (c->nd == 2 ? 9 : 2)));  // see pass1_rows
  const int ring = VEC == 4 ? kNStg * 4 * kT * 16 : 0;
#define LAUNCH(ND, V, F)                                                                                        \
  AVD_CUDA(smem_attr(pass1_kernel<ND, V, F>, ring));  \
  pass1_kernel<ND, V, F><<<grid, kT, ring, c->stream>>>(                                                        \
      X, l, m, c->m_pad, c->l_pad, rpc, c->cfg.row_offset, c->qscale, c->qoff, seed32, kd, c->digits, c->dplan, \
      c->cand_key, c->cand_idx, c->cand_cnt, c->cand_cap, c->colsum_part, c->colmax_part, c->qsum_part,         \
      reinterpret_cast<double*>(c->qsq_part), c->qerr_part)
  if (c->nd == 2) {
    if (full) { if (vec) { LAUNCH(2, 4, true); } else { LAUNCH(2, 1, true); } }
    else { if (vec) { LAUNCH(2, 4, false); } else { LAUNCH(2, 1, false); } }
  } else {
    if (full) { if (vec) { LAUNCH(3, 4, true); } else { LAUNCH(3, 1, true); } }
    else { if (vec) { LAUNCH(3, 4, false); } else { LAUNCH(3, 1, false); } }
  }
#undef LAUNCH
  AVD_LAUNCHED(c);
  if (c->nd == 2)
    pass1_reduce_kernel<2><<<(unsigned)ceil_div(m, 32), 256, 0, c->stream>>>(
        m, r1, full ? 1 : 0, c->colsum_part, c->colmax_part, c->qsum_part, reinterpret_cast<const double*>(c->qsq_part),
        c->qerr_part, c->qscale, c->stats, c->colmax, c->qsum_local, c->qerr_local, c->ysq);
  else
    pass1_reduce_kernel<3><<<(unsigned)ceil_div(m, 32), 256, 0, c->stream>>>(
        m, r1, full ? 1 : 0, c->colsum_part, c->colmax_part, c->qsum_part, reinterpret_cast<const double*>(c->qsq_part),
        c->qerr_part, c->qscale, c->stats, c->colmax, c->qsum_local, c->qerr_local, c->ysq);
  AVD_LAUNCHED(c);
  if (full) {
    cand_publish_kernel<<<1, 1, 0, c->stream>>>(c->cand_cnt, c->cand_cap, c->cand_x);
    AVD_LAUNCHED(c);
  }
  return AVD_OK;
}

avd_status launch_finish(Ctx* c) {
  AVD_CUDA(cudaMemsetAsync(&c->dplan->nonfinite, 0, sizeof(int64_t), c->stream));
  AVD_CUDA(cudaMemsetAsync(&c->dplan->range_bits, 0, sizeof(int32_t), c->stream));
  finish_kernel<<<(unsigned)ceil_div(c->m_pad, 256), 256, 0, c->stream>>>(c->cfg.m, c->m_pad, c->cfg.l_global,
                                                                         c->plan.n_top, c->stats, c->mu, c->mu_hl,
                                                                         c->dplan, c->colmax, c->shift, c->nd);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
