// k_stats.cu — K1: one HBM-streaming pass over X producing fp64 column sums (for
// mu = (1/l) X^T 1), sum x^2 (||X||_F^2), column max/min (the
// per-column scale of the Gram digit planes) and a 4096-bin histogram of |x| float bits
// [30:19] (first radix level of the top-0.1% threshold); plus the
// "prepare" kernel that turns the (all-reduced) sums into mu, digit scales and the first
// threshold bin.
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
    const float* __restrict__ X, int64_t l, int64_t m, int64_t rpc, double* __restrict__ colsum_part,
    float* __restrict__ colmax_part, float* __restrict__ colmin_part, double* __restrict__ sq_part,
    unsigned long long* __restrict__ hist1, double* __restrict__ stats) {
  __shared__ unsigned int sh[kHistBins];
  __shared__ double sred[kStatsThreads / 32];
  __shared__ unsigned int snf;
  for (int b = threadIdx.x; b < kHistBins; b += kStatsThreads) sh[b] = 0;
  if (threadIdx.x == 0) snf = 0;
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
  unsigned int nonfin = 0;

  constexpr int U = 4;  // rows in flight per thread
  for (int64_t i = r0; i < r1; i += U) {
    float x[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = active && (i + u < r1);
      if (VEC == 4) {
        float4 t = ok ? __ldcs(reinterpret_cast<const float4*>(X + (i + u) * m + c0))
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        x[u][0] = t.x; x[u][VEC > 1 ? 1 : 0] = t.y; x[u][VEC > 2 ? 2 : 0] = t.z; x[u][VEC > 3 ? 3 : 0] = t.w;
      } else {
        x[u][0] = ok ? __ldcs(X + (i + u) * m + c0) : 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = active && (i + u < r1);
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const float xv = x[u][v];
        const uint32_t key = __float_as_uint(xv) & 0x7FFFFFFFu;
        const bool fin = key < 0x7F800000u;
        if (ok) {
          const double d = (double)xv;
          s[v] += d;
          sq = fma(d, d, sq);
          mx[v] = fmaxf(mx[v], xv);
          mn[v] = fminf(mn[v], xv);
          nonfin += fin ? 0u : 1u;
        }
        hist_add(sh, key, ok && fin && key != 0);
      }
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
  // block reduction of sum x^2 in a fixed order
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = sq;
  if (nonfin) atomicAdd(&snf, nonfin);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kStatsThreads / 32; ++w) t += sred[w];
    sq_part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
    if (snf) atomicAdd(&stats[m + 1], (double)snf);
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
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < nsq; ++r) t += sq_part[r];
    stats[m] = t;
  }
}

// mu, digit-plane scale exponents, first-level threshold bin.
//  shift_j = B - e_j with e_j = ilogb(max_i |x_ij - mu_j|) + 1 and B = 7*nd - 1, so that
//  |(x - mu) * 2^shift| < 2^B and the dithered integer q fits nd balanced base-128 digits.
__global__ void prepare_kernel(int64_t m, int64_t m_pad, int64_t l_global, int nd,
                               int64_t n_top, const double* __restrict__ stats,
                               const float* __restrict__ colmax, const float* __restrict__ colmin,
                               const unsigned long long* __restrict__ hist1, double* __restrict__ mu,
                               int32_t* __restrict__ shift, DevPlan* __restrict__ dp) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m_pad) {
    int32_t sh = 0;
    if (j < m) {
      const double mj = stats[j] / (double)l_global;
      mu[j] = mj;
      const double a = fmax((double)colmax[j] - mj, mj - (double)colmin[j]);
      if (a > 0.0 && a < 1e300) sh = (7 * nd - 1) - (ilogb(a) + 1);
    }
    shift[j] = sh;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    // first-level bin b1: count(bins > b1) < n_eff <= count(bins >= b1); scanned from the top
    const int lane = threadIdx.x;
    constexpr int per = kHistBins / 32;
    const int hi = kHistBins - 1 - lane * per;  // lane covers bins (hi-per, hi]
    unsigned long long mine = 0;
    for (int b = hi; b > hi - per; --b) mine += hist1[b];
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    const unsigned long long total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const long long n_eff = (long long)min((unsigned long long)n_top, total);
    const unsigned long long excl = incl - mine;
    const bool crosses = n_eff > 0 && excl < (unsigned long long)n_eff && incl >= (unsigned long long)n_eff;
    if (crosses) {
      unsigned long long cum = excl;
      int b = hi;
      for (; b > hi - per; --b) {
        if (cum + hist1[b] >= (unsigned long long)n_eff) break;
        cum += hist1[b];
      }
      dp->b1 = b;
      dp->cnt_gt = (long long)cum;
    }
    if (lane == 0) {
      dp->n_eff = n_eff;
      dp->empty = n_eff == 0 ? 1 : 0;
      if (n_eff == 0) { dp->b1 = kHistBins; dp->cnt_gt = 0; }
      dp->cand_count = 0;
      dp->nonfinite = (long long)stats[m + 1];
    }
  }
}

}  // namespace

avd_status launch_stats(Ctx* c, const float* X) {
  const int64_t m = c->cfg.m, l = c->cfg.l_local;
  const bool vec = (m % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int VEC = vec ? 4 : 1;
  const int ncb = (int)ceil_div(m, (int64_t)kStatsThreads * VEC);
  const int64_t rpc = round_up(ceil_div(l, c->r1), 4);
  AVD_CUDA(cudaMemsetAsync(c->hist1, 0, sizeof(unsigned long long) * kHistBins, c->stream));
  AVD_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(double) * (m + 2), c->stream));
  dim3 grid(ncb, c->r1);
  if (vec)
    stats_kernel<4><<<grid, kStatsThreads, 0, c->stream>>>(X, l, m, rpc, c->colsum_part, c->colmax_part,
                                                           c->colmin_part, c->sq_part, c->hist1, c->stats);
  else
    stats_kernel<1><<<grid, kStatsThreads, 0, c->stream>>>(X, l, m, rpc, c->colsum_part, c->colmax_part,
                                                           c->colmin_part, c->sq_part, c->hist1, c->stats);
  AVD_LAUNCHED(c);
  stats_reduce_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, c->stream>>>(
      m, c->r1, c->r1 * ncb, c->colsum_part, c->colmax_part, c->colmin_part, c->sq_part, c->stats,
      c->colmax, c->colmin);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_prepare(Ctx* c) {
  prepare_kernel<<<(unsigned)ceil_div(c->m_pad, 256), 256, 0, c->stream>>>(
      c->cfg.m, c->m_pad, c->cfg.l_global, c->nd, c->plan.n_top, c->stats, c->colmax, c->colmin,
      c->hist1, c->mu, c->shift, c->dplan);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
