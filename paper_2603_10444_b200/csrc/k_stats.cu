// k_stats.cu — K1: one HBM-streaming pass over X producing fp64 column sums (for
// mu = (1/l) X^T 1), sum x^2 (||X||_F^2), column max/min (the
// per-column scale of the Gram digit planes), the exact count of nonzero entries (|E_top| =
// min(n_top, #nonzero), R4) and a ROW-SAMPLED 4096-bin histogram of |x| float bits
// [30:19] that only seeds the candidate threshold b0 of K2 (exact counts come later, from the
// candidate list — k_select.cu); plus the "prepare" kernel that turns the (all-reduced) sums into
// mu, digit scales and b0.
#include <cfloat>
#include "common.cuh"

namespace avd {

namespace {

constexpr int kStatsThreads = 256;

__device__ __forceinline__ void hist_add(unsigned int* sh, uint32_t key, bool valid) {
  // warp-aggregated shared-memory histogram update (one atomic per distinct bin per warp)
  const uint32_t bin = valid ? (key >> 19) : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xFFFFFFFFu, bin);
  const int leader = __ffs(peers) - 1;
  if (valid && (int)(threadIdx.x & 31) == leader) atomicAdd(&sh[bin], (unsigned)__popc(peers));
}

template <int VEC>
__global__ void __launch_bounds__(kStatsThreads) stats_kernel(
    const float* __restrict__ X, int64_t l, int64_t m, int64_t rpc, int64_t row_offset, int sample,
    double* __restrict__ colsum_part, float* __restrict__ colmax_part, float* __restrict__ colmin_part,
    double* __restrict__ sq_part, unsigned long long* __restrict__ hist1, double* __restrict__ stats) {
  __shared__ unsigned int sh[kHistBins];
  __shared__ double sred[kStatsThreads / 32];
  __shared__ unsigned long long snz;
  __shared__ unsigned int snf;
  for (int b = threadIdx.x; b < kHistBins; b += kStatsThreads) sh[b] = 0;
  if (threadIdx.x == 0) { snf = 0; snz = 0; }
  __syncthreads();

  const int64_t c0 = ((int64_t)blockIdx.x * kStatsThreads + threadIdx.x) * VEC;
  const int64_t r0 = (int64_t)blockIdx.y * rpc;
  const int64_t r1 = min(l, r0 + rpc);
  const bool active = c0 < m;
  double s[VEC];
  float mx[VEC], mn[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { s[v] = 0.0; mx[v] = -FLT_MAX; mn[v] = FLT_MAX; }
  double sq = 0.0;
  unsigned int nonfin = 0, nz = 0;

  constexpr int U = 4;  // rows in flight per thread
  for (int64_t i = r0; i < r1; i += U) {
    float x[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = active && (i + u < r1);
      if constexpr (VEC == 4) {
        const float4 t = ok ? __ldcs(reinterpret_cast<const float4*>(X + (i + u) * m + c0))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        x[u][0] = t.x; x[u][1] = t.y; x[u][2] = t.z; x[u][3] = t.w;
      } else {
        x[u][0] = ok ? __ldcs(X + (i + u) * m + c0) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = active && (i + u < r1);
      const bool sampled = (((uint32_t)(row_offset + i + u)) & (uint32_t)(sample - 1)) == 0;  // warp-uniform; sample = 2^s
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float xv = x[u][v];
        const uint32_t key = __float_as_uint(xv) & 0x7FFFFFFFu;
        const bool fin = key < 0x7F800000u;
        if (ok) {
          mx[v] = fmaxf(mx[v], xv);
          mn[v] = fminf(mn[v], xv);
          nonfin += fin ? 0u : 1u;
          nz += (fin && key != 0) ? 1u : 0u;
        }
        if (sampled) hist_add(sh, key, ok && fin && key != 0);
      }
    }
    // fp64 accumulation of U-row fp32 partial sums (each partial rounds once, ~2^-24 relative)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      float ps = 0.f, pq = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = active && (i + u < r1);
        const float xv = ok ? x[u][v] : 0.f;
        ps += xv;
        pq = fmaf(xv, xv, pq);
      }
      s[v] += (double)ps;
      sq += (double)pq;
    }
  }
  if (active) {
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      if (c0 + v < m) {
        colsum_part[(int64_t)blockIdx.y * m + c0 + v] = s[v];
        colmax_part[(int64_t)blockIdx.y * m + c0 + v] = mx[v];
        colmin_part[(int64_t)blockIdx.y * m + c0 + v] = mn[v];
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
    nz += __shfl_xor_sync(0xFFFFFFFFu, nz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sred[threadIdx.x >> 5] = sq;
    atomicAdd(&snz, (unsigned long long)nz);
  }
  if (nonfin) atomicAdd(&snf, nonfin);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kStatsThreads / 32; ++w) t += sred[w];
    sq_part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    if (snf) atomicAdd(&stats[m + 1], (double)snf);
    if (snz) atomicAdd(&stats[m + 2], (double)snz);  // integer-valued doubles: exact, order-free
  }
  for (int b = threadIdx.x; b < kHistBins; b += kStatsThreads)
    if (sh[b]) atomicAdd(&hist1[b], (unsigned long long)sh[b]);
}

// Fixed-order reduction of the per-chunk partials -> stats[0..m) colsum, stats[m] sum x^2,
// colmax/colmin.
__global__ void stats_reduce_kernel(int64_t m, int r1, int nsq, const double* __restrict__ colsum_part,
                                    const float* __restrict__ colmax_part,
                                    const float* __restrict__ colmin_part,
                                    const double* __restrict__ sq_part, double* __restrict__ stats,
                                    float* __restrict__ colmax, float* __restrict__ colmin) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) {
    double s = 0.0;
    float mx = -FLT_MAX, mn = FLT_MAX;
    for (int r = 0; r < r1; ++r) {
      s += colsum_part[(int64_t)r * m + j];
      mx = fmaxf(mx, colmax_part[(int64_t)r * m + j]);
      mn = fminf(mn, colmin_part[(int64_t)r * m + j]);
    }
    stats[j] = s;
    colmax[j] = mx;
    colmin[j] = mn;
  }
  if (blockIdx.x == 0) {
    __shared__ double sh[256];
    double t = 0.0;
    for (int r = threadIdx.x; r < nsq; r += blockDim.x) t += sq_part[r];
    sh[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      double u = 0.0;
      for (int q = 0; q < (int)blockDim.x; ++q) u += sh[q];
      stats[m] = u;
    }
  }
}

// mu, digit-plane scale exponents, candidate threshold b0.
//  shift_j = B - e_j with e_j = ilogb(max_i |x_ij - mu_j|) + 1 and B = 7*nd - 1, so that
//  |(x - mu) * 2^shift| < 2^B and the dithered integer q fits nd balanced base-128 digits.
//  b0: the largest first-level bin whose sampled tail count, scaled by the sampling step,
//  covers 2 n_eff + 256 step (conservative; K6 verifies with exact counts over the candidates
//  and falls back to streaming X when they do not cover n_eff).
__global__ void prepare_kernel(int64_t m, int64_t m_pad, int64_t l_global, int nd, int64_t n_top, int sample,
                               const double* __restrict__ stats, const float* __restrict__ colmax,
                               const float* __restrict__ colmin, const unsigned long long* __restrict__ hist1,
                               double* __restrict__ mu, float* __restrict__ mu_hl, int32_t* __restrict__ shift,
                               DevPlan* __restrict__ dp) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m_pad) {
    int32_t sh = 0;
    float mh = 0.f, ml = 0.f;
    if (j < m) {
      const double mj = stats[j] / (double)l_global;
      mu[j] = mj;
      mh = (float)mj;
      ml = (float)(mj - (double)mh);
      const double a = fmax((double)colmax[j] - mj, mj - (double)colmin[j]);
      if (a > 0.0 && a < 1e300) sh = (7 * nd - 1) - (ilogb(a) + 1);
    }
    shift[j] = sh;
    mu_hl[j] = mh;
    mu_hl[m_pad + j] = ml;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const long long nonzero = (long long)stats[m + 2];
    const long long n_eff = min((long long)n_top, nonzero);
    const unsigned long long need = 2ull * (unsigned long long)n_eff + 256ull * (unsigned long long)sample;
    constexpr int per = kHistBins / 32;
    const int hi = kHistBins - 1 - lane * per;  // lane covers bins (hi-per, hi]
    unsigned long long mine = 0;
    for (int b = hi; b > hi - per; --b) mine += hist1[b] * (unsigned long long)sample;
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
        cum += hist1[b] * (unsigned long long)sample;
        if (cum >= need) break;
      }
      b0 = b;
    }
    // lowest lane holding a crossing wins; none -> every nonzero entry is a candidate (b0 = 0)
    for (int o = 16; o > 0; o >>= 1) b0 = max(b0, __shfl_xor_sync(0xFFFFFFFFu, b0, o));
    if (lane == 0) {
      dp->n_eff = n_eff;
      dp->empty = n_eff == 0 ? 1 : 0;
      dp->b0 = b0 < 0 ? 0 : b0;
      dp->b1 = 0;
      dp->b2 = 0;
      dp->cnt_gt = 0;
      dp->cand_count = 0;
      dp->nonfinite = (long long)stats[m + 1];
    }
  }
}

}  // namespace

int stats_sample_step(int64_t l_global) {
  const int64_t want = std::max<int64_t>(1, std::min<int64_t>(16, l_global / 4096));
  int s = 1;
  while (s * 2 <= want) s *= 2;  // power of two: the kernel tests row & (s - 1)
  return s;
}

avd_status launch_stats(Ctx* c, const float* X) {
  const int64_t m = c->cfg.m, l = c->cfg.l_local;
  const bool vec = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int VEC = vec ? 4 : 1;
  const int ncb = (int)ceil_div(m, (int64_t)kStatsThreads * VEC);
  const int64_t rpc = round_up(ceil_div(l, c->r1), 4);
  const int sample = stats_sample_step(c->cfg.l_global);
  AVD_CUDA(cudaMemsetAsync(c->hist1, 0, sizeof(unsigned long long) * kHistBins, c->stream));
  AVD_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(double) * (m + 3), c->stream));
  dim3 grid(ncb, c->r1);
  if (vec)
    stats_kernel<4><<<grid, kStatsThreads, 0, c->stream>>>(X, l, m, rpc, c->cfg.row_offset, sample, c->colsum_part,
                                                           c->colmax_part, c->colmin_part, c->sq_part, c->hist1, c->stats);
  else
    stats_kernel<1><<<grid, kStatsThreads, 0, c->stream>>>(X, l, m, rpc, c->cfg.row_offset, sample, c->colsum_part,
                                                           c->colmax_part, c->colmin_part, c->sq_part, c->hist1, c->stats);
  AVD_LAUNCHED(c);
  stats_reduce_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, c->stream>>>(
      m, c->r1, c->r1 * ncb, c->colsum_part, c->colmax_part, c->colmin_part, c->sq_part, c->stats,
      c->colmax, c->colmin);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_prepare(Ctx* c) {
  prepare_kernel<<<(unsigned)ceil_div(c->m_pad, 256), 256, 0, c->stream>>>(
      c->cfg.m, c->m_pad, c->cfg.l_global, c->nd, c->plan.n_top, stats_sample_step(c->cfg.l_global), c->stats,
      c->colmax, c->colmin, c->hist1, c->mu, c->mu_hl, c->shift, c->dplan);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
