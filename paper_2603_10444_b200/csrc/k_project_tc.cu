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

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// fp64 V (m x k, row-major) -> Vt_hl [2*KP][m_pad32] (hi rows then lo rows) and
// V_hl [2][m_pad128][KP32] (hi plane then lo plane); padding is zero.
// fp64 V (m x k, row-major) -> Vt_hl [2*KP][m_pad32] (hi rows then lo rows) and
// V_hl [2][m_pad128][KP32] (hi plane then lo plane); padding is zero.  Column k of Vt_hl (K5's B
// operand only) carries the mean direction mu / ||mu||, so P[:, k] = xc_i . mu_hat and
// p_i = x_i . mu_hat = P[i][k] + ||mu|| come with the projection for free; V_hl
// (K8's B operand) keeps a zero there, so the spike S = P V_k^T is unaffected.
__global__ void split_v_kernel(const double* __restrict__ V, const double* __restrict__ mu,
                               const double* __restrict__ diag, int64_t m, int k, int KP, int KP32, int64_t m_pad32,
                               int64_t m_pad128, float* __restrict__ Vt_hl, float* __restrict__ V_hl) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m_pad128 * KP32) return;
  const int64_t j = t / KP32;
  const int r = (int)(t % KP32);
  const float v = (j < m && r < k) ? (float)V[j * k + r] : 0.f;
  const float hi = rna_tf32(v), lo = rna_tf32(v - hi);
  V_hl[j * KP32 + r] = hi;
  V_hl[(m_pad128 + j) * KP32 + r] = lo;
  if (r < KP && j < m_pad32) {
    float vt = v;
    if (r == k) vt = (j < m && diag[0] > 0.0) ? (float)(mu[j] / diag[0]) : 0.f;
    const float th = rna_tf32(vt), tl = rna_tf32(vt - th);
    Vt_hl[(int64_t)r * m_pad32 + j] = th;
    Vt_hl[(int64_t)(KP + r) * m_pad32 + j] = tl;
  }
}

// ======================================================================= K5
template <int KP, int NS>
__global__ void __launch_bounds__(kPThreads, 1) proj_tc_kernel(
    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmVt, int64_t l_local, int64_t m,
    const float* __restrict__ mu_hl, int64_t m_pad, float* __restrict__ P, float* __restrict__ P_hl, int64_t l_pad,
    double* __restrict__ en_part, double* __restrict__ colsumP_part) {
  constexpr int KP32 = (KP + 31) / 32 * 32;
  constexpr int NSLOT_MAX = (512 / KP) < 8 ? (512 / KP) : 8;
  constexpr uint32_t kVtBytes = 2 * KP * 128;
  constexpr uint32_t kStage = 2 * kTile + ((kVtBytes + 1023) / 1024) * 1024;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[NS], conv_bar[NS], empty_bar[NS], tfull_bar, tempty_bar;
  __shared__ uint32_t tmem_sh;
  __shared__ double colsum_w[8][KP];
  __shared__ double sq_w[8];

  const uint32_t warp = warp_id(), lane = lane_id();
  const int64_t nrb = ceil_div(l_local, 128);
  const int NC = (int)((m + 31) / 32);
  const int nslot = NC < NSLOT_MAX ? NC : NSLOT_MAX;  // every slot receives >= 1 chunk

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&conv_bar[s], 8); mbar_init(&empty_bar[s], 1); }
    mbar_init(&tfull_bar, 1);
    mbar_init(&tempty_bar, 8);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) { tma_prefetch(&tmX); tma_prefetch(&tmVt); }
  if (warp == 1) tmem_alloc<512>(&tmem_sh);
  if (warp >= 2) {
    for (int r = lane; r < KP; r += 32) colsum_w[warp - 2][r] = 0.0;
    if (lane == 0) sq_w[warp - 2] = 0.0;
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
          mbar_arrive_expect_tx(&full_bar[s], kTile + kVtBytes);
          tma_load_2d(st, &tmX, &full_bar[s], c * 32, (int32_t)(rb * 128));
          tma_load_2d(st + 2 * kTile, &tmVt, &full_bar[s], c * 32, 0);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_tf32(128, KP, 0, 0);
    uint32_t it = 0, ui = 0;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
      mbar_wait(&tempty_bar, (ui & 1) ^ 1);
      tc_fence_after();
      for (int c = 0; c < NC; ++c, ++it) {
        const uint32_t s = it % NS, r = it / NS;
        mbar_wait(&full_bar[s], r & 1);
        mbar_wait(&conv_bar[s], r & 1);
        tc_fence_after();
        const int slot = (int)((int64_t)c * nslot / NC);
        const bool slot_first = (c == 0) || ((int)((int64_t)(c - 1) * nslot / NC) != slot);
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + s * kStage);
          const uint32_t d = tmem + slot * KP;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ahi = smem_desc(base + kk * 32, 16, 1024, 2);
            const uint64_t alo = smem_desc(base + kTile + kk * 32, 16, 1024, 2);
            const uint64_t bhi = smem_desc(base + 2 * kTile + kk * 32, 16, 1024, 2);
            const uint64_t blo = smem_desc(base + 2 * kTile + KP * 128 + kk * 32, 16, 1024, 2);
            mma_tf32(d, ahi, bhi, idesc, (slot_first && kk == 0) ? 0u : 1u);
            mma_tf32(d, ahi, blo, idesc, 1u);
            mma_tf32(d, alo, bhi, idesc, 1u);
          }
          mma_commit(&empty_bar[s]);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&tfull_bar);
      __syncwarp();
    }
  } else {
    // ================= converter + epilogue warps (8 warps, two per TMEM lane quadrant)
    const int ew = warp - 2;              // 0..7
    const uint32_t q = warp & 3;          // TMEM lane quadrant
    const int half = ew >> 2;             // epilogue column half
    const int ct = threadIdx.x - 64;      // 0..255 converter thread
    const int g = (ct & 7) ^ ((ct >> 3) & 7);  // logical 4-column group of this thread (SW128)
    const int rbase = ct >> 3;            // rows rbase + 32 u, u < 4
    double sq = 0.0;
    uint32_t it = 0, ui = 0;
    float4 mh4 = __ldg(reinterpret_cast<const float4*>(mu_hl + g * 4));
    float4 ml4 = __ldg(reinterpret_cast<const float4*>(mu_hl + m_pad + g * 4));
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x, ++ui) {
      const int64_t row0 = rb * 128;
      for (int c = 0; c < NC; ++c, ++it) {
        const uint32_t s = it % NS, r = it / NS;
        const int64_t col = (int64_t)c * 32 + g * 4;
        const float mh[4] = {mh4.x, mh4.y, mh4.z, mh4.w}, ml[4] = {ml4.x, ml4.y, ml4.z, ml4.w};
        {  // prefetch mu of the next chunk (mu depends on the column only)
          const int64_t ncol = (int64_t)(c + 1 < NC ? c + 1 : 0) * 32 + g * 4;
          mh4 = __ldg(reinterpret_cast<const float4*>(mu_hl + ncol));
          ml4 = __ldg(reinterpret_cast<const float4*>(mu_hl + m_pad + ncol));
        }
        bool cok[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) cok[e] = col + e < m;
        mbar_wait(&full_bar[s], r & 1);
        uint8_t* st = smem + s * kStage;
        const float4* xs = reinterpret_cast<const float4*>(st);
        float4* hs = reinterpret_cast<float4*>(st);          // hi overwrites x in place
        float4* ls = reinterpret_cast<float4*>(st + kTile);
        float s32u[4];  // one partial per u: four short FFMA chains instead of one of 16
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float s32 = 0.f;
          const int ch = ct + 256 * u;  // 16-byte chunk index in the tile
          const bool rok = row0 + rbase + 32 * u < l_local;
          const float4 x = xs[ch];
          const float xv[4] = {x.x, x.y, x.z, x.w};
          float hv[4], lv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // fp32 centring with mu = hi + lo: (x - mu_hi) is exact or correctly rounded
            const float xc = (rok && cok[e]) ? (xv[e] - mh[e]) - ml[e] : 0.f;
            s32 = fmaf(xc, xc, s32);
            hv[e] = rna_tf32(xc);
            lv[e] = rna_tf32(xc - hv[e]);
          }
          hs[ch] = make_float4(hv[0], hv[1], hv[2], hv[3]);
          ls[ch] = make_float4(lv[0], lv[1], lv[2], lv[3]);
          s32u[u] = s32;
        }
        const float s32 = (s32u[0] + s32u[1]) + (s32u[2] + s32u[3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv_bar[s]);
        sq += (double)s32;  // off the MMA's critical path (after the stage is handed over)
      }
      // ---- epilogue: P row = sum of slots (this warp: half of the KP columns)
      mbar_wait(&tfull_bar, ui & 1);
      tc_fence_after();
      const int64_t row = row0 + q * 32 + lane;
      const bool rok = row < l_local;
      const uint32_t tb = tmem + ((q * 32) << 16);
#pragma unroll 1
      for (int c0 = half * (KP / 2); c0 < (half + 1) * (KP / 2); c0 += 8) {
        float pv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) pv[t] = 0.f;
        for (int sl = 0; sl < nslot; ++sl) {
          uint32_t rv[8];
          tmem_ld8(tb + sl * KP + c0, rv);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 8; ++t) pv[t] += __uint_as_float(rv[t]);
        }
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
      if (lane == 0) mbar_arrive(&tempty_bar);
    }
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o);
    if (lane == 0) sq_w[ew] = sq;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < KP) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += colsum_w[w][threadIdx.x];
    colsumP_part[(int64_t)blockIdx.x * KP + threadIdx.x] = t;
  }
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sq_w[w];
    en_part[(int64_t)blockIdx.x * 4 + 3] = t;
  }
  if (warp == 1) tmem_dealloc<512>(tmem);
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
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
#pragma unroll
          for (int t = 0; t < 16; t += 2) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const bool ok = rok && j0 + t + e < m;
              const float xc = (xv[t + e] - mh[t + e]) - ml[t + e];
              const float S = ok ? __uint_as_float(rv[t + e]) : 0.f;
              const float T = ok ? xc - S : 0.f;
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

template <int KP>
avd_status launch_k5(Ctx* c, const CUtensorMap& tmX, const CUtensorMap& tmVt, int grid) {
  constexpr uint32_t kStage = 2 * kTile + ((2 * KP * 128 + 1023) / 1024) * 1024;
  constexpr int NS = (220 * 1024) / kStage;  // 5 stages in flight
  const size_t smem = NS * kStage + 1024;
  AVD_CUDA(smem_attr(proj_tc_kernel<KP, NS>, (int)smem));
  proj_tc_kernel<KP, NS><<<grid, kPThreads, smem, c->stream>>>(tmX, tmVt, c->cfg.l_local, c->cfg.m, c->mu_hl,
                                                               c->m_pad, c->P, c->P_hl, c->l_pad, c->en_part,
                                                               c->colsumP_part);
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

// V_k -> hi/lo operand copies (once per solve)
avd_status launch_split_v(Ctx* c) {
  const int KP32 = (c->k_pad + 31) / 32 * 32;
  const int64_t n = c->m_pad * KP32;
  split_v_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c->stream>>>(c->V, c->mu, c->diag, c->cfg.m, c->k, c->k_pad,
                                                                    KP32, c->m_pad32, c->m_pad, c->Vt_hl, c->V_hl);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_project_tc(Ctx* c, const float* X) {
  const int KP = c->k_pad;
  const int KP32 = (KP + 31) / 32 * 32;
  const int64_t nrb = ceil_div(c->cfg.l_local, 128);
  const int grid = (int)std::min<int64_t>(nrb, c->num_sms);
  CUtensorMap tmX, tmVt, tmP, tmV;
  if (encode2d(&tmX, X, c->cfg.m, c->cfg.l_local, c->cfg.m * 4, 32, 128) != CUDA_SUCCESS ||
      encode2d(&tmVt, c->Vt_hl, c->m_pad32, 2 * KP, c->m_pad32 * 4, 32, 2 * KP) != CUDA_SUCCESS ||
      encode2d(&tmP, c->P_hl, KP32, 2 * c->l_pad, KP32 * 4, 32, 128) != CUDA_SUCCESS ||
      encode2d(&tmV, c->V_hl, KP32, 2 * c->m_pad, KP32 * 4, 32, 32) != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (projection maps)");
    return AVD_ECUDA;
  }
  AVD_CUDA(cudaMemsetAsync(c->en_part, 0, sizeof(double) * 4 * c->n_proj_ctas, c->stream));
  AVD_CUDA(cudaMemsetAsync(c->colsumP_part, 0, sizeof(double) * KP * c->n_proj_ctas, c->stream));
  AVD_TRY(launch_split_v(c));
  switch (KP) {
    case 16: AVD_TRY(launch_k5<16>(c, tmX, tmVt, grid)); break;
    case 32: AVD_TRY(launch_k5<32>(c, tmX, tmVt, grid)); break;
    case 48: AVD_TRY(launch_k5<48>(c, tmX, tmVt, grid)); break;
    case 64: AVD_TRY(launch_k5<64>(c, tmX, tmVt, grid)); break;
    case 80: AVD_TRY(launch_k5<80>(c, tmX, tmVt, grid)); break;
    case 96: AVD_TRY(launch_k5<96>(c, tmX, tmVt, grid)); break;
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
