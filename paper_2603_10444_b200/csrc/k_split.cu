// k_split.cu — K2: centring X_c = X - 1 mu^T fused with the operand encoding of
// the Gram and the top-set candidate pass.
//   * every centred entry x_c is scaled by the column's power of two 2^shift_j and rounded with
//     a deterministic dither u ~ U[0,1): q = floor(x_c 2^shift_j + u)  (|q| <= 2^(7 nd - 1));
//     q is written as nd balanced base-128 int8 digits into TRANSPOSED planes
//     D_d[j][i] (K-major operands of the tcgen05 kind::i8 Gram);
//   * entries whose |x| bit pattern falls in a first-level bin >= b0 are appended as
//     (key, global linear index) candidates of E_top.
// One read of X (4 B/entry), nd bytes written per entry.
#include <cudaTypedefs.h>
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // k_gram.cu

namespace {

constexpr int kSplitRows = 128;   // rows i per CTA tile (= one 128-byte digit row)
constexpr int kSplitCols = 64;    // columns j per CTA tile
constexpr int kSplitThreads = 256;
constexpr int kSW = 33;           // padded smem row stride in 32-bit words

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}

template <int ND, bool VEC>
__global__ void __launch_bounds__(kSplitThreads) split_kernel(
    const __grid_constant__ CUtensorMap tmX, const float* __restrict__ X, int64_t l_local, int64_t m, int64_t m_pad, int64_t l_pad,
    int64_t row_offset, const float* __restrict__ mu_hl, const int32_t* __restrict__ shift,
    uint32_t seed32, int8_t* __restrict__ digits, const DevPlan* __restrict__ dp,
    uint32_t* __restrict__ cand_key, uint64_t* __restrict__ cand_idx,
    unsigned long long* __restrict__ cand_cnt, int64_t cand_cap) {
  extern __shared__ __align__(128) float sX_raw[];  // [kSplitRows][kSplitCols] tile of X
  float* sX = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sX_raw) + 127) & ~uintptr_t(127));
  __shared__ uint32_t sD[ND][kSplitCols * kSW];
  __shared__ uint32_t srow[kSplitRows];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i0 = (int64_t)blockIdx.x * kSplitRows;
  const int64_t j0 = (int64_t)blockIdx.y * kSplitCols;
  // ---- stage the whole 128 x 64 tile asynchronously (32 KB in flight per CTA): one TMA
  //      (out-of-range rows / columns zero-filled), or per-thread cp.async when m % 4 != 0
  __shared__ __align__(8) uint64_t tbar;
  if (VEC) {
    if (threadIdx.x == 0) {
      sm100::mbar_init(&tbar, 1);
      sm100::fence_mbar_init();
      sm100::mbar_arrive_expect_tx(&tbar, kSplitRows * kSplitCols * 4);
      sm100::tma_load_2d(sX, &tmX, &tbar, (int32_t)j0, (int32_t)i0);
    }
  } else {
    for (int id = threadIdx.x; id < kSplitRows * kSplitCols; id += kSplitThreads) {
      const int r = id / kSplitCols, cc = id % kSplitCols;
      const int64_t gi = i0 + r, gj = j0 + cc;
      const bool v = gi < l_local && gj < m;
      cp_async4(sX + r * kSplitCols + cc, v ? (const void*)(X + gi * m + gj) : (const void*)X, v);
    }
  }
  if (!VEC) asm volatile("cp.async.commit_group;" ::: "memory");
  const int jl = (warp & 1) * 32 + lane;
  const int64_t j = j0 + jl;
  const int rg = warp >> 1;  // 32-row group
  if (threadIdx.x < kSplitRows)
    srow[threadIdx.x] = mix32((uint32_t)(row_offset + i0 + threadIdx.x) * 0x9E3779B1u ^ seed32);
  const uint32_t b0 = (uint32_t)dp->b0;
  // candidate test as one unsigned compare: key in [max(1, b0 << 19), 0x7F800000)
  const uint32_t klo = max(1u, b0 << 19);
  const uint32_t kspan = 0x7F800000u - klo;
  const int rows_here = (l_local - i0) < kSplitRows ? (int)(l_local - i0) : kSplitRows;  // valid rows of this tile
  const bool colok = j < m;
  // mu = hi + lo (fp32 pair); 2^shift as an exact fp32 power of two (shift clamped to the normal
  // range: columns with max|xc| < 2^-100 quantise to zero)
  const float mh = colok ? mu_hl[j] : 0.f, ml = colok ? mu_hl[m_pad + j] : 0.f;
  const int sh = colok ? shift[j] : 0;
  const float scale = (colok && sh <= 126 && sh >= -126) ? __int_as_float((sh + 127) << 23) : 0.f;
  const uint32_t colh = mix32((uint32_t)j ^ 0x68E31DA4u);
  if (VEC) {
    __syncthreads();  // barrier initialised before anyone waits on it
    sm100::mbar_wait(&tbar, 0);
  } else {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }

#pragma unroll 1
  for (int t = 0; t < 8; ++t) {
    float xs[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) xs[u] = sX[(rg * 32 + t * 4 + u) * kSplitCols + jl];
    uint32_t packed[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) packed[d] = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int rl = rg * 32 + t * 4 + u;
      const bool ok = colok && rl < rows_here;
      const float x = xs[u];
      const uint32_t key = __float_as_uint(x) & 0x7FFFFFFFu;
      // ---- candidate append (warp aggregated)
      const bool cand = ok && (key - klo) < kspan;
      const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, cand);
      if (ballot) {
        const int ldr = __ffs(ballot) - 1;
        unsigned long long base = 0;
        if (lane == ldr) base = atomicAdd(cand_cnt, (unsigned long long)__popc(ballot));
        base = __shfl_sync(0xFFFFFFFFu, base, ldr);
        if (cand) {
          const unsigned long long pos = base + __popc(ballot & ((1u << lane) - 1u));
          if (pos < (unsigned long long)cand_cap) {
            cand_key[pos] = key;
            cand_idx[pos] = (uint64_t)(row_offset + i0 + rl) * (uint64_t)m + (uint64_t)j;
          }
        }
      }
      // ---- dithered fixed-point digits of the centred entry: q = floor(xc 2^shift + u)
      if (ok) {
        const float y = ((x - mh) - ml) * scale;     // exact power-of-two scaling, |y| < 2^(7nd-1)
        const uint32_t h = (srow[rl] ^ colh) * 0x9E3779B1u;  // row/column hashes are mix32-ed
        // u in [0, 1 - ulp(2^(7nd-1))]: the clamp keeps fl(y + u) < y + 1 for integer y (exact data
        // stays exact); it moves probability <= 2^-10 (nd=2) / 2^-3 (nd=3) of u to the clamp value
        constexpr float kDithMax = ND == 2 ? 1.0f - 0x1p-10f : 1.0f - 0x1p-3f;
        const float dith = fminf(__uint_as_float(0x3F800000u | (h >> 9)) - 1.0f, kDithMax);
        int32_t q = __float2int_rd(y + dith);        // RN sum then floor: dithered rounding
        // balanced base-128 digits, most significant first
        int32_t dg[ND];
#pragma unroll
        for (int d = ND - 1; d >= 1; --d) {
          const int32_t hi = (q + 64) >> 7;
          dg[d] = q - (hi << 7);                      // in [-64, 63]
          q = hi;
        }
        dg[0] = q;
#pragma unroll
        for (int d = 0; d < ND; ++d) packed[d] = __byte_perm(packed[d], (uint32_t)dg[d], u == 0 ? 0x3214 : (u == 1 ? 0x3240 : (u == 2 ? 0x3410 : 0x4210)));
      }
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) sD[d][jl * kSW + rg * 8 + t] = packed[d];
  }
  __syncthreads();
  // write-out: plane d, row j0+jr, 32 words (128 rows of i) per row -> one 128 B line per warp
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    for (int jr = warp; jr < kSplitCols; jr += kSplitThreads / 32) {
      const uint32_t w = sD[d][jr * kSW + lane];
      uint32_t* dst = reinterpret_cast<uint32_t*>(digits + ((int64_t)d * m_pad + j0 + jr) * l_pad + i0);
      __stcs(dst + lane, w);
    }
  }
}

// exchange slot for the global candidate decision: [count, overflowed]
__global__ void cand_publish_kernel(const unsigned long long* __restrict__ cnt, int64_t cap,
                                    long long* __restrict__ out) {
  out[0] = (long long)*cnt;
  out[1] = (long long)(*cnt > (unsigned long long)cap ? 1 : 0);
}

}  // namespace

avd_status launch_split(Ctx* c, const float* X) {
  AVD_CUDA(cudaMemsetAsync(c->cand_cnt, 0, sizeof(unsigned long long), c->stream));
  dim3 grid((unsigned)(c->l_pad / kSplitRows), (unsigned)(c->m_pad / kSplitCols));
  const uint32_t seed32 = (uint32_t)(c->cfg.seed * 0x9E3779B97F4A7C15ull >> 32) ^ 0xA5A5A5A5u;
  const bool vec = (c->cfg.m % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const size_t sm = sizeof(float) * kSplitRows * kSplitCols + 128;
  CUtensorMap tmX{};
  if (vec) {
    uint64_t dims[2] = {(uint64_t)c->cfg.m, (uint64_t)c->cfg.l_local};
    uint64_t strides[1] = {(uint64_t)c->cfg.m * 4};
    uint32_t box[2] = {kSplitCols, kSplitRows};
    uint32_t es[2] = {1, 1};
    if (tma_encode_fn()(&tmX, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (split)");
      return AVD_ECUDA;
    }
  }
#define LAUNCH(ND, V)                                                                                         \
  do {                                                                                                        \
    AVD_CUDA(cudaFuncSetAttribute(split_kernel<ND, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    split_kernel<ND, V><<<grid, kSplitThreads, sm, c->stream>>>(                                              \
        tmX, X, c->cfg.l_local, c->cfg.m, c->m_pad, c->l_pad, c->cfg.row_offset, c->mu_hl, c->shift, seed32,       \
        c->digits, c->dplan, c->cand_key, c->cand_idx, c->cand_cnt, c->cand_cap);                             \
  } while (0)
  if (c->nd == 2) { if (vec) LAUNCH(2, true); else LAUNCH(2, false); }
  else { if (vec) LAUNCH(3, true); else LAUNCH(3, false); }
#undef LAUNCH
  AVD_LAUNCHED(c);
  cand_publish_kernel<<<1, 1, 0, c->stream>>>(c->cand_cnt, c->cand_cap, c->cand_x);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
