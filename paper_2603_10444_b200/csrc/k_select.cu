// k_select.cu — K6: exact top-0.1% set E_top by |X_ij|, ties broken by the
// smaller global linear index i*m+j, zeros excluded (R3, R4); K7: rho gather
// (PAPER.md:23-27).
//
// Keys are the 31-bit magnitude bit patterns of the fp32 entries (ordering of |x| == ordering of
// the bits).  Radix levels: bits [30:19] (hist1, K1) -> [18:7] (hist2) -> [6:0] (hist3) give
// the exact threshold key T, count_gt(T) and the tie quota q = n_eff - count_gt(T).  Entries
// with key > T and the first q entries with key == T (in linear order) form E_top.  They are
// marked in two bitmaps over this rank's linear index range and emitted in ascending order by
// a two-level ordered compaction, so the output needs no sort and is deterministic.
// Rank r takes the ties left after ranks < r (rows are sharded in rank order).
// The histogram and mark passes read the K2 candidate list (entries with key>>19 >= b1), or,
// if it overflowed its capacity, stream X directly.
#include <cstring>
#include <vector>
#include "common.cuh"

namespace avd {

namespace {

constexpr int kSelThreads = 256;
constexpr int kWordsPerBlk = 1024;  // bitmap words per compaction block

template <bool FROM_X>
__device__ __forceinline__ bool fetch(int64_t t, const uint32_t* __restrict__ ckey, const uint64_t* __restrict__ cidx,
                                      const float* __restrict__ X, int64_t base, uint32_t& key, uint64_t& lidx) {
  if (FROM_X) {
    const float x = __ldg(X + t);
    key = __float_as_uint(x) & 0x7FFFFFFFu;
    lidx = (uint64_t)t;
    return key != 0 && key < 0x7F800000u;
  } else {
    key = ckey[t];
    if (key == 0) return false;  // a hole of a K2 slot block
    lidx = cidx[t] - (uint64_t)base;
    return true;
  }
}

// radix level 0: bits [30:19] of every candidate (exact counts);
// level 1: bits [18:7] over key>>19 == b1 ; level 2: bits [6:0] over key>>7 == (b1, b2)
template <bool FROM_X>
__global__ void __launch_bounds__(kSelThreads) hist_kernel(int level, int64_t n, const uint32_t* __restrict__ ckey,
                                                           const uint64_t* __restrict__ cidx, const float* __restrict__ X,
                                                           const DevPlan* __restrict__ dp, unsigned long long* __restrict__ out,
                                                           const unsigned long long* __restrict__ n_dev = nullptr,
                                                           int64_t n_cap = 0) {
  __shared__ unsigned int sh[kHistBins];
  if (n_dev) n = min((int64_t)*n_dev, n_cap);  // count read on the device (speculative level 0)
  const int nb = level < 2 ? kHistBins : kHist3Bins;
  for (int b = threadIdx.x; b < nb; b += kSelThreads) sh[b] = 0;
  __syncthreads();
  const uint32_t pre = level == 0 ? 0u : (level == 1 ? (uint32_t)dp->b1 : (((uint32_t)dp->b1 << 12) | (uint32_t)dp->b2));
  const int shiftp = level == 0 ? 31 : (level == 1 ? 19 : 7);
  for (int64_t t = (int64_t)blockIdx.x * kSelThreads + threadIdx.x; t < n; t += (int64_t)gridDim.x * kSelThreads) {
    uint32_t key;
    uint64_t li;
    if (!fetch<FROM_X>(t, ckey, cidx, X, 0, key, li)) continue;
    if ((key >> shiftp) != pre) continue;
    const uint32_t bin = level == 0 ? (key >> 19) : (level == 1 ? ((key >> 7) & 0xFFFu) : (key & 0x7Fu));
    atomicAdd(&sh[bin], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += kSelThreads)
    if (sh[b]) atomicAdd(&out[b], (unsigned long long)sh[b]);
}

// Find the bin of radix level `level` that contains the n_eff-th largest key (one warp).
// Level 0 first sets |E_top| = n_eff = min(n_top, #counted keys): streaming X the level-0
// histogram counts every nonzero finite entry exactly; the candidate list is only used when it
// holds >= n_top entries, so there n_eff = n_top (R4).
__global__ void find_bin_kernel(int level, const unsigned long long* __restrict__ h, int64_t n_top,
                                DevPlan* __restrict__ dp) {
  const int lane = threadIdx.x;
  const int nb = level < 2 ? kHistBins : kHist3Bins;
  const int per = nb / 32;
  const int hi = nb - 1 - lane * per;
  // the lane's `per` bins (hi-per, hi] as 16-byte loads, 8 in flight (a latency-bound single warp)
  unsigned long long mine = 0;
  {
    const ulonglong2* hv = reinterpret_cast<const ulonglong2*>(h + (hi - per + 1));
#pragma unroll 8
    for (int t = 0; t < per / 2; ++t) {
      const ulonglong2 v = __ldg(hv + t);
      mine += v.x + v.y;
    }
  }
  unsigned long long incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  const unsigned long long excl = incl - mine;
  if (level == 0) {
    const unsigned long long total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const long long n_eff = min((long long)n_top, (long long)total);
    __syncwarp();
    if (lane == 0) {
      dp->n_eff = n_eff;
      dp->empty = n_eff == 0 ? 1 : 0;
      dp->cnt_gt = 0;
    }
    __syncwarp();
  }
  if (dp->empty) return;
  const long long need = dp->n_eff - dp->cnt_gt;  // rank inside the current prefix (>= 1)
  if (excl < (unsigned long long)need && incl >= (unsigned long long)need) {
    unsigned long long cum = excl;
    int b = hi;
    for (; b > hi - per; --b) {
      if (cum + h[b] >= (unsigned long long)need) break;
      cum += h[b];
    }
    if (level == 0) {
      dp->b1 = b;
      dp->cnt_gt = (long long)cum;
    } else if (level == 1) {
      dp->b2 = b;
      dp->cnt_gt = dp->cnt_gt + (long long)cum;
    } else {
      dp->T = ((uint32_t)dp->b1 << 19) | ((uint32_t)dp->b2 << 7) | (uint32_t)b;
      dp->cnt_gt_T = dp->cnt_gt + (long long)cum;
      dp->q = dp->n_eff - dp->cnt_gt_T;
    }
  }
}

// mark entries with key > T (sel) and key == T (tie); count both for this rank
template <bool FROM_X>
__global__ void __launch_bounds__(kSelThreads) mark_kernel(int64_t n, const uint32_t* __restrict__ ckey,
                                                           const uint64_t* __restrict__ cidx, const float* __restrict__ X,
                                                           int64_t base, const DevPlan* __restrict__ dp,
                                                           uint32_t* __restrict__ bm_sel, uint32_t* __restrict__ bm_tie,
                                                           unsigned long long* __restrict__ counts,
                                                           unsigned long long* __restrict__ blk, int64_t nblk) {
  __shared__ unsigned int c_sel, c_tie;
  if (threadIdx.x == 0) { c_sel = 0; c_tie = 0; }
  __syncthreads();
  const uint32_t T = dp->T;
  const bool empty = dp->empty != 0;
  unsigned int ns = 0, nt = 0;
  if (!empty) {
    for (int64_t t = (int64_t)blockIdx.x * kSelThreads + threadIdx.x; t < n; t += (int64_t)gridDim.x * kSelThreads) {
      uint32_t key;
      uint64_t li;
      if (!fetch<FROM_X>(t, ckey, cidx, X, base, key, li)) continue;
      // + the per-compaction-block counts the ordered emit scans (no separate counting pass)
      const int64_t bk = (int64_t)(li >> 5) / kWordsPerBlk;
      if (key > T) {
        atomicOr(&bm_sel[li >> 5], 1u << (li & 31));
        atomicAdd(&blk[bk], 1ull);
        ++ns;
      } else if (key == T) {
        atomicOr(&bm_tie[li >> 5], 1u << (li & 31));
        atomicAdd(&blk[nblk + bk], 1ull);
        ++nt;
      }
    }
  }
  if (ns) atomicAdd(&c_sel, ns);
  if (nt) atomicAdd(&c_tie, nt);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (c_sel) atomicAdd(&counts[0], (unsigned long long)c_sel);
    if (c_tie) atomicAdd(&counts[1], (unsigned long long)c_tie);
  }
}

// counts[0..1] (this rank) -> ties[rank] (sel) and ties[world + rank] (tie) for the exchange
__global__ void publish_counts_kernel(const unsigned long long* __restrict__ counts, long long* __restrict__ ties,
                                      int world, int rank) {
  const int t = threadIdx.x;
  if (t < 2 * world) ties[t] = 0;
  __syncthreads();
  if (t == 0) { ties[rank] = (long long)counts[0]; ties[world + rank] = (long long)counts[1]; }
}

// exclusive scan of block counts (one CTA); quota / offset come from avd_tie_quota (host)
// block-wide exclusive scan helpers (warp shuffles + one smem pass)
template <typename T, int NT>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NT / 32 ? warp_tot[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < NT / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == NT / 32 - 1) warp_tot[NT / 32] = wi;
  }
  __syncthreads();
  total = warp_tot[NT / 32];
  const T r = warp_tot[warp] + incl - v;
  __syncthreads();
  return r;
}

// exclusive scan of the per-block (sel, tie) counts in one CTA (each thread owns a contiguous
// run of blocks); quota / offset come from avd_tie_quota (host)
// ties_dev != nullptr (one rank): the tie quota is taken on the device — every tie of the threshold
// key up to q (clamped to the ties held), offset 0 — with no host round trip
__global__ void __launch_bounds__(1024) blk_scan_kernel(int64_t* __restrict__ blk, int64_t nblk, int64_t quota,
                                                        int64_t offset, int64_t ties_local, DevPlan* __restrict__ dp,
                                                        const long long* __restrict__ ties_dev) {
  if (ties_dev) {
    ties_local = ties_dev[1];
    quota = dp->empty ? 0 : max((int64_t)0, min((int64_t)dp->q, ties_local));
    offset = 0;
  }
  __shared__ int64_t wt[1024 / 32 + 1];
  const int64_t per = (nblk + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = min(nblk, b0 + per);
  int64_t sel_total = 0;
  for (int which = 0; which < 2; ++which) {
    int64_t* a = blk + which * nblk;
    // the run is read in batches of 8 independent loads (one latency per batch, not per block)
    int64_t run = 0;
    int64_t i = b0;
    for (; i + 8 <= b1; i += 8) {
      int64_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a[i + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) run += v[u];
    }
    for (; i < b1; ++i) run += a[i];
    int64_t total;
    int64_t acc = block_exclusive_scan<int64_t, 1024>(run, wt, total);
    for (i = b0; i + 8 <= b1; i += 8) {
      int64_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a[i + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) { a[i + u] = acc; acc += v[u]; }
    }
    for (; i < b1; ++i) {
      const int64_t v = a[i];
      a[i] = acc;
      acc += v;
    }
    if (which == 0) sel_total = total;
  }
  if (threadIdx.x == 0) {
    dp->ties_local = ties_local;
    dp->quota = quota;
    dp->sel_local = sel_total + quota;
    dp->top_offset = offset;
  }
}

__global__ void __launch_bounds__(kSelThreads) emit_kernel(const uint32_t* __restrict__ bs, const uint32_t* __restrict__ bt,
                                                           int64_t nwords, int64_t nblk, const int64_t* __restrict__ blk,
                                                           const DevPlan* __restrict__ dp, int64_t base_idx,
                                                           int64_t* __restrict__ out) {
  __shared__ int ps[kSelThreads / 32 + 1], pt[kSelThreads / 32 + 1];
  const int64_t w0 = (int64_t)blockIdx.x * kWordsPerBlk;
  const int64_t quota = dp->quota;
  int64_t sel_before = blk[blockIdx.x], tie_before = blk[nblk + blockIdx.x];
  constexpr int WPT = kWordsPerBlk / kSelThreads;  // 4 consecutive words per thread
  uint32_t ws[WPT], wt[WPT];
  int a = 0, b = 0;
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t w = w0 + threadIdx.x * WPT + q;
    ws[q] = w < nwords ? bs[w] : 0u;
    wt[q] = w < nwords ? bt[w] : 0u;
    a += __popc(ws[q]);
    b += __popc(wt[q]);
  }
  int tot;
  const int ea = block_exclusive_scan<int, kSelThreads>(a, ps, tot);
  const int eb = block_exclusive_scan<int, kSelThreads>(b, pt, tot);
  int64_t sb4 = sel_before + ea;
  int64_t tb4 = tie_before + eb;
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const int64_t w = w0 + threadIdx.x * WPT + q;
    uint32_t s = ws[q], t = wt[q];
    while (s | t) {
      const uint32_t ls = s & (0u - s), lt = t & (0u - t);
      // next set bit in linear order among both masks
      const bool take_sel = ls && (!lt || ls < lt);
      const uint32_t bit = take_sel ? ls : lt;
      const int pos_in_word = __ffs(bit) - 1;
      if (take_sel) {
        out[sb4 + min(tb4, quota)] = base_idx + w * 32 + pos_in_word;
        ++sb4;
        s &= s - 1;
      } else {
        if (tb4 < quota) out[sb4 + tb4] = base_idx + w * 32 + pos_in_word;
        ++tb4;
        t &= t - 1;
      }
    }
  }
}

// rho per selected entry + per-CTA aggregate partials
__global__ void __launch_bounds__(kSelThreads) gather_kernel(const int64_t* __restrict__ top_idx, const DevPlan* __restrict__ dp,
                                                             const float* __restrict__ X, int64_t m, int64_t row_offset,
                                                             const double* __restrict__ mu, const float* __restrict__ P,
                                                             const double* __restrict__ V, int k, int k_pad,
                                                             double* __restrict__ rho, double* __restrict__ agg_part) {
  __shared__ double red[kSelThreads / 32][8];
  const int64_t n = dp->sel_local;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t t = (int64_t)blockIdx.x * kSelThreads + threadIdx.x; t < n; t += (int64_t)gridDim.x * kSelThreads) {
    const int64_t g = top_idx[t];
    const int64_t i = g / m - row_offset, j = g % m;
    const double x = (double)X[i * m + j];
    const double M = mu[j];
    const double xc = x - M;
    double S = 0.0;
    for (int r = 0; r < k; ++r) S = fma((double)P[i * k_pad + r], V[j * k + r], S);
    const double T = xc - S;
    const double x2 = x * x;
    const double rm = M * M / x2, rs = S * S / x2, rt = T * T / x2;
    const double cr = 1.0 - (rm + rs + rt);
    rho[t * 4 + 0] = rm; rho[t * 4 + 1] = rs; rho[t * 4 + 2] = rt; rho[t * 4 + 3] = cr;
    acc[0] += rm; acc[1] += rs; acc[2] += rt; acc[3] += cr;
    acc[4] += M * M; acc[5] += S * S; acc[6] += T * T; acc[7] += x2;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xFFFFFFFFu, acc[q], o);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) red[threadIdx.x >> 5][q] = acc[q];
  __syncthreads();
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (int w = 0; w < kSelThreads / 32; ++w) s += red[w][threadIdx.x];
    agg_part[(int64_t)blockIdx.x * 8 + threadIdx.x] = s;
  }
}

// fixed-order sum of the per-CTA partials: 32 lanes stride the partials of each of the 8 sums,
// then a fixed shuffle tree (deterministic)
__global__ void agg_reduce_kernel(const double* __restrict__ part, int nparts, double* __restrict__ agg) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp w: sum w
  double s = 0.0;
  for (int q = lane; q < nparts; q += 32) s += part[(int64_t)q * 8 + w];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if (lane == 0) agg[w] = s;
}

}  // namespace

// level 0: radix level 0 histogram ; level 1: find b1, level-1 histogram ;
// level 2: find b2, level-2 histogram ; level 3: find T, mark, publish per-rank counts
avd_status launch_select(Ctx* c, const float* X, int level, int rank) {
  const bool fromX = c->cand_overflow;
  const int64_t n = fromX ? c->cfg.l_local * c->cfg.m : c->hplan.cand_count;
  const int64_t base = c->cfg.row_offset * c->cfg.m;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kSelThreads), 4LL * c->num_sms));
  if (level <= 2) {
    unsigned long long* h = level == 0 ? c->hist0 : (level == 1 ? c->hist2 : c->hist3);
    if (level > 0) {
      find_bin_kernel<<<1, 32, 0, c->stream>>>(level - 1, level == 1 ? c->hist0 : c->hist2, c->plan.n_top, c->dplan);
      AVD_LAUNCHED(c);
    }
    AVD_CUDA(cudaMemsetAsync(h, 0, sizeof(unsigned long long) * (level < 2 ? kHistBins : kHist3Bins), c->stream));
    if (fromX) hist_kernel<true><<<grid, kSelThreads, 0, c->stream>>>(level, n, nullptr, nullptr, X, c->dplan, h);
    else hist_kernel<false><<<grid, kSelThreads, 0, c->stream>>>(level, n, c->cand_key, c->cand_idx, nullptr, c->dplan, h);
    AVD_LAUNCHED(c);
  } else {
    find_bin_kernel<<<1, 32, 0, c->stream>>>(2, c->hist3, c->plan.n_top, c->dplan);
    AVD_LAUNCHED(c);
    AVD_CUDA(cudaMemsetAsync(c->bm_sel, 0, sizeof(uint32_t) * c->nwords, c->stream));
    AVD_CUDA(cudaMemsetAsync(c->bm_tie, 0, sizeof(uint32_t) * c->nwords, c->stream));
    unsigned long long* counts = reinterpret_cast<unsigned long long*>(c->blk_cnt + 2 * c->nblk);
    AVD_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), c->stream));
    unsigned long long* blk = reinterpret_cast<unsigned long long*>(c->blk_cnt);
    AVD_CUDA(cudaMemsetAsync(blk, 0, 2 * sizeof(unsigned long long) * c->nblk, c->stream));
    if (fromX)
      mark_kernel<true><<<grid, kSelThreads, 0, c->stream>>>(n, nullptr, nullptr, X, base, c->dplan, c->bm_sel,
                                                             c->bm_tie, counts, blk, c->nblk);
    else
      mark_kernel<false><<<grid, kSelThreads, 0, c->stream>>>(n, c->cand_key, c->cand_idx, nullptr, base, c->dplan,
                                                              c->bm_sel, c->bm_tie, counts, blk, c->nblk);
    AVD_LAUNCHED(c);
    publish_counts_kernel<<<1, 256, 0, c->stream>>>(counts, c->ties, c->cfg.world, rank);
    AVD_LAUNCHED(c);
  }
  return AVD_OK;
}

// Level-0 histogram over the candidate list with the count read on the device, queued before the
// host learns whether the list is usable (avd_stage_select redoes level 0 from X if it is not).
avd_status launch_select0_speculative(Ctx* c) {
  AVD_CUDA(cudaMemsetAsync(c->hist0, 0, sizeof(unsigned long long) * kHistBins, c->stream));
  hist_kernel<false><<<(unsigned)(4 * c->num_sms), kSelThreads, 0, c->stream>>>(
      0, 0, c->cand_key, c->cand_idx, nullptr, c->dplan, c->hist0, c->cand_cnt, c->cand_cap);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_gather(Ctx* c, const float* X, int rank, int64_t* top_idx, double* rho) {
  // exchanged per-rank counts -> this rank's tie quota and global offset (host integer logic)
  const int world = c->cfg.world;
  // both land in the pinned scratch (pageable D2H copies cost ~10 us each)
  if (world == 1) {  // the quota is taken on the device (no host round trip)
    blk_scan_kernel<<<1, 1024, 0, c->stream>>>(c->blk_cnt, c->nblk, 0, 0, 0, c->dplan,
                                               reinterpret_cast<const long long*>(c->ties));
    AVD_LAUNCHED(c);
  } else {
    long long* hs = reinterpret_cast<long long*>(c->eig_host);
    AVD_CUDA(cudaMemcpyAsync(hs, c->ties, sizeof(long long) * 2 * world, cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaMemcpyAsync(hs + 2 * world, c->dplan, sizeof(DevPlan), cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<long long> tc(hs, hs + 2 * world);
    std::memcpy(&c->hplan, hs + 2 * world, sizeof(DevPlan));
    std::vector<int64_t> sel(world), tie(world);
    for (int r = 0; r < world; ++r) { sel[r] = tc[r]; tie[r] = tc[world + r]; }
    int64_t quota = 0, offset = 0;
    AVD_TRY(avd_tie_quota(sel.data(), tie.data(), world, rank, c->hplan.empty ? 0 : c->hplan.q, &quota, &offset));
    // per-block (sel, tie) counts were accumulated by mark_kernel
    blk_scan_kernel<<<1, 1024, 0, c->stream>>>(c->blk_cnt, c->nblk, quota, offset, tie[rank], c->dplan, nullptr);
    AVD_LAUNCHED(c);
  }
  emit_kernel<<<(unsigned)c->nblk, kSelThreads, 0, c->stream>>>(c->bm_sel, c->bm_tie, c->nwords, c->nblk, c->blk_cnt,
                                                                 c->dplan, c->cfg.row_offset * c->cfg.m, top_idx);
  AVD_LAUNCHED(c);
  gather_kernel<<<(unsigned)c->n_gather_ctas, kSelThreads, 0, c->stream>>>(top_idx, c->dplan, X, c->cfg.m, c->cfg.row_offset,
                                                                           c->mu, c->P, c->V, c->k, c->k_pad, rho, c->agg_part);
  AVD_LAUNCHED(c);
  agg_reduce_kernel<<<1, 256, 0, c->stream>>>(c->agg_part, c->n_gather_ctas, c->agg);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
