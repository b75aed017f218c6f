// k_eig_i8.cu — the power-step products of K4 on the int8 tensor cores.
//
// The subspace iteration (k_eig.cu) applies G twice per step: Z = G Q, Y = G Z.  These products
// only steer the subspace (every reported quantity comes from the fp64 Rayleigh-Ritz product with
// the exact G), so they take G and the block in fixed point:
//   G_ab = s_a z_ab,  |z_ab| < 2^26, four balanced base-128 digits per row a (s_a = 2^(e_a - 26),
//          e_a from the row's largest |G_ab|) — once per solve (gdig_kernel);
//   Q_br = t_r w_br,  |w_br| < 2^19, three digits per column r (t_r from the column's largest
//          |Q_br|) — per product (qdig_kernel);
// and tcgen05.mma kind::i8 accumulates every digit product exactly in int32 TMEM, by weight class
// c = d_G + d_Q (weight 128^(5 - c)); the classes c <= 3 are kept (the dropped ones weigh <= 2^-28
// of the leading class).  The operator error is ~2^-27 of each row's largest entry (the converged
// subspace moves by that much), the block's 2^-20 only perturbs each step's input, which the next
// steps damp.  Split-K over the 128-byte K chunks fills the GPU: per (128-row block, K slice) CTA
// the epilogue combines the classes in fp64, scales by s_a t_r and stores a partial; the last CTA
// of a row block (acq_rel ticket) sums the slices in slice order — deterministic — and writes Y
// (fp64), its fp32 mirror and the per-column max |Y| the next product's digits need.
#include <cudaTypedefs.h>
#include "common.cuh"
#include "sm100.cuh"

namespace avd {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // k_gram.cu

namespace {
using namespace sm100;

constexpr int kG8Threads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (one per TMEM lane quadrant)
constexpr int kGDig = 4, kQDig = 3, kNCls = 4;

__device__ __forceinline__ unsigned ticket_acq_rel8(unsigned* t) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
  return old;
}

// balanced base-128 digits of z (|z| < 64 * (128^n - 1) / 127 * 128 ... ), most significant first
template <int N>
__device__ __forceinline__ void digits_of(long long z, int8_t (&d)[N]) {
  long long off = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) off = off * 128 + 64;
  const long long zz = z + off;
#pragma unroll
  for (int i = 0; i < N; ++i) d[i] = (int8_t)(((zz >> (7 * (N - 1 - i))) & 127) - 64);
}

// G (fp64, ld m_pad) -> Gd [4][m_pad][m_pad] int8, sG[a] = 2^(e_a - 26); one CTA per row a
__global__ void __launch_bounds__(256) gdig_kernel(const double* __restrict__ G, int64_t m, int64_t m_pad,
                                                   int8_t* __restrict__ Gd, double* __restrict__ sG) {
  __shared__ double sh[256];
  const int64_t a = blockIdx.x;
  const double* row = G + a * m_pad;
  double mx = 0.0;
  if (a < m)
    for (int64_t b = threadIdx.x; b < m; b += 256) mx = fmax(mx, fabs(row[b]));
  sh[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  const double gmax = sh[0];
  const int e = (gmax > 0.0 && gmax < 1e300) ? ilogb(gmax) + 1 : 0;
  if (threadIdx.x == 0) sG[a] = ldexp(1.0, e - 26);
  const int64_t plane = m_pad * m_pad;
  for (int64_t b = threadIdx.x; b < m_pad; b += 256) {
    const long long z = (a < m && b < m && gmax > 0.0) ? llrint(ldexp(row[b], 26 - e)) : 0ll;
    int8_t d[kGDig];
    digits_of<kGDig>(z, d);
#pragma unroll
    for (int i = 0; i < kGDig; ++i) Gd[i * plane + a * m_pad + b] = d[i];
  }
}

// Q (fp64, m x p row-major) -> Qd [3][p][m_pad] int8 (transposed: K-major B operand) with
// tQ[r] = 2^(e_r - 19) from the column max.  Two coalesced kernels: per 64-row tile column maxima
// (atomicMax on the bit patterns of |.|: order-free, deterministic), then per 128-row tile the
// digits, written transposed through shared memory.
constexpr int kQdTile = 64;
__global__ void __launch_bounds__(256) qmax_kernel(const double* __restrict__ Q, int64_t m, int p,
                                                   unsigned long long* __restrict__ qmax) {
  extern __shared__ double tq[];  // [kQdTile][p]
  const int64_t b0 = (int64_t)blockIdx.x * kQdTile;
  const int rows = (int)(m - b0 < kQdTile ? m - b0 : kQdTile);
  for (int t = threadIdx.x; t < rows * p; t += 256) tq[t] = fabs(Q[b0 * p + t]);
  __syncthreads();
  for (int r = threadIdx.x; r < p; r += 256) {
    double mx = 0.0;
    for (int i = 0; i < rows; ++i) mx = fmax(mx, tq[i * p + r]);
    atomicMax(qmax + r, (unsigned long long)__double_as_longlong(mx));
  }
}
constexpr int kQdRows = 32;  // rows per CTA of the digit kernel
__global__ void __launch_bounds__(256) qdig_kernel(const double* __restrict__ Q, int64_t m, int64_t m_pad, int p,
                                                   const unsigned long long* __restrict__ qmax,
                                                   int8_t* __restrict__ Qd, double* __restrict__ tQ) {
  extern __shared__ double tq[];  // [kQdRows][p] + [p] scales
  double* sc = tq + kQdRows * p;
  const int64_t b0 = (int64_t)blockIdx.x * kQdRows;
  const int rows = (int)(m - b0 <= 0 ? 0 : (m - b0 < kQdRows ? m - b0 : kQdRows));
  for (int t = threadIdx.x; t < kQdRows * p; t += 256) tq[t] = t < rows * p ? Q[b0 * p + t] : 0.0;
  for (int r = threadIdx.x; r < p; r += 256) {
    const double mx = __longlong_as_double((long long)qmax[r]);
    const int e = (mx > 0.0 && mx < 1e300) ? ilogb(mx) + 1 : 0;
    sc[r] = mx > 0.0 ? ldexp(1.0, 19 - e) : 0.0;
    if (blockIdx.x == 0) tQ[r] = ldexp(1.0, e - 19);
  }
  __syncthreads();
  const int64_t plane = (int64_t)p * m_pad;
  for (int t = threadIdx.x; t < kQdRows * p; t += 256) {
    const int r = t / kQdRows, i = t % kQdRows;  // consecutive threads: consecutive rows of column r
    const long long z = llrint(tq[i * p + r] * sc[r]);
    int8_t d[kQDig];
    digits_of<kQDig>(z, d);
#pragma unroll
    for (int di = 0; di < kQDig; ++di) Qd[di * plane + (int64_t)r * m_pad + b0 + i] = d[di];
  }
}

__host__ __device__ constexpr uint32_t idesc_i8k2(uint32_t M, uint32_t N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8k2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int P>
constexpr uint32_t tmem_cols() {
  return kNCls * P <= 128 ? 128 : (kNCls * P <= 256 ? 256 : 512);
}

// CTA = (row block rb0 + blockIdx.x / KS, K slice blockIdx.x % KS): 128 rows of Y, all P columns.
// The tensor maps live in GLOBAL memory (64-B aligned workspace slots): the kernel runs inside the
// eigensolver's conditional graph bodies, whose kernel parameters the device itself launches, so
// a __grid_constant__ map in parameter space is not a valid TMA descriptor address there.
template <int P, int NS>
__global__ void __launch_bounds__(kG8Threads, 1) gemm_i8_kernel(
    const CUtensorMap* __restrict__ tmGp, const CUtensorMap* __restrict__ tmQp, int64_t m, int64_t m_pad,
    int KS, int rb0, const double* __restrict__ sG, const double* __restrict__ tQ, double* __restrict__ part,
    unsigned* __restrict__ tickets, double* __restrict__ Y, float* __restrict__ Y32, double* __restrict__ colmax,
    const int* __restrict__ skip) {
  if (skip && *skip) return;  // device-side gate (eigensolver graph: Z comes from the RR check)
  constexpr uint32_t kA = 128 * 128;
  constexpr uint32_t kB = P * 128;
  constexpr uint32_t kStage = ((kGDig * kA + kQDig * kB + 1023) / 1024) * 1024;
  constexpr uint32_t kCols = tmem_cols<P>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[NS], empty_bar[NS], tfull_bar;
  __shared__ uint32_t tmem_sh;
  __shared__ unsigned last_sh;
  __shared__ double s_t[P];

  const uint32_t warp = warp_id(), lane = lane_id();
  const int rb = rb0 + (int)(blockIdx.x / KS), ks = (int)(blockIdx.x % KS);
  const int NKC = (int)(m_pad / 128);
  const int kc0 = (int)((int64_t)NKC * ks / KS), kc1 = (int)((int64_t)NKC * (ks + 1) / KS);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full_bar[s], 1); mbar_init(&empty_bar[s], 1); }
    mbar_init(&tfull_bar, 1);
    fence_mbar_init();
  }
  const CUtensorMap* tmG = tmGp;
  const CUtensorMap* tmQ = tmQp;
  if (warp == 0 && lane == 0) { tma_prefetch(tmG); tma_prefetch(tmQ); }
  if (warp == 1) tmem_alloc<kCols>(&tmem_sh);
  for (int r = threadIdx.x; r < P; r += blockDim.x) s_t[r] = tQ[r];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_sh;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int kc = kc0; kc < kc1; ++kc, ++it) {
        const uint32_t s = it % NS, r = it / NS;
        mbar_wait(&empty_bar[s], (r & 1) ^ 1);
        uint8_t* st = smem + s * kStage;
        mbar_arrive_expect_tx(&full_bar[s], kGDig * kA + kQDig * kB);
#pragma unroll
        for (int d = 0; d < kGDig; ++d)
          tma_load_2d(st + d * kA, tmG, &full_bar[s], kc * 128, (int32_t)(d * m_pad + (int64_t)rb * 128));
#pragma unroll
        for (int d = 0; d < kQDig; ++d)
          tma_load_2d(st + kGDig * kA + d * kB, tmQ, &full_bar[s], kc * 128, d * P);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_i8k2(128, P);
    uint32_t it = 0;
    for (int kc = kc0; kc < kc1; ++kc, ++it) {
      const uint32_t s = it % NS, r = it / NS;
      mbar_wait(&full_bar[s], r & 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t base = smem_u32(smem + s * kStage);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
          for (int dg = 0; dg < kGDig; ++dg) {
            const uint64_t a = smem_desc(base + dg * kA + kk * 32, 16, 1024, 2);
#pragma unroll
            for (int dq = 0; dq < kQDig; ++dq) {
              if (dg + dq >= kNCls) continue;  // dropped class (<= 2^-28 of the leading weight)
              const uint64_t bq = smem_desc(base + kGDig * kA + dq * kB + kk * 32, 16, 1024, 2);
              // the class's first product in this loop order: the smallest d_G with d_Q < kQDig
              const bool first = kc == kc0 && kk == 0 && (dg == 0 || dq == kQDig - 1);
              mma_i8k2(tmem + (dg + dq) * P, a, bq, idesc, first ? 0u : 1u);
            }
          }
        }
        mma_commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(&tfull_bar);
    __syncwarp();
  } else {
    // epilogue: warp q = TMEM lane quadrant, thread = row rb*128 + 32q + lane, all P columns
    const uint32_t q = warp & 3;
    const int64_t row = (int64_t)rb * 128 + q * 32 + lane;
    mbar_wait(&tfull_bar, 0);
    tc_fence_after();
    const double sa = row < m ? sG[row] : 0.0;
    double* dst = part + (((int64_t)(rb - rb0) * KS + ks) * 128 + q * 32 + lane) * P;
    const uint32_t tb = tmem + ((q * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < P; c0 += 8) {
      double acc[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] = 0.0;
#pragma unroll
      for (int cl = 0; cl < kNCls; ++cl) {
        uint32_t rv[8];
        tmem_ld8(tb + cl * P + c0, rv);
        tmem_ld_wait();
        const double wgt = (double)(1ll << (7 * (kGDig + kQDig - 2 - cl)));  // 128^(5 - c)
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = fma((double)(int)rv[t], wgt, acc[t]);
      }
#pragma unroll
      for (int t = 0; t < 8; t += 2)
        *reinterpret_cast<double2*>(dst + c0 + t) =
            make_double2(acc[t] * sa * s_t[c0 + t], acc[t + 1] * sa * s_t[c0 + t + 1]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kCols>(tmem);
  // the row block's last CTA: fixed-order sum of the KS partials, Y, Y32, column max |Y|
  if (threadIdx.x == 0) {
    __threadfence();
    last_sh = (ticket_acq_rel8(&tickets[rb]) == (unsigned)(KS - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!last_sh) return;
  const double* base = part + (int64_t)(rb - rb0) * KS * 128 * P;
  for (int e = threadIdx.x; e < 128 * P; e += blockDim.x) {
    double s0 = 0.0;
    int kq = 0;
    for (; kq + 4 <= KS; kq += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcg(base + (int64_t)(kq + u) * 128 * P + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) s0 += v[u];
    }
    for (; kq < KS; ++kq) s0 += __ldcg(base + (int64_t)kq * 128 * P + e);
    const int64_t row = (int64_t)rb * 128 + e / P;
    const int r = e % P;
    if (row < m) {
      Y[row * P + r] = s0;
      if (Y32) Y32[row * P + r] = (float)s0;
      if (colmax)  // |s0| >= 0: the double's bit pattern orders like an integer
        atomicMax(reinterpret_cast<unsigned long long*>(colmax + r), (unsigned long long)__double_as_longlong(fabs(s0)));
    }
  }
  if (threadIdx.x == 0) tickets[rb] = 0u;  // re-armed for the next launch (stream-ordered)
}

}  // namespace

// ---------------------------------------------------------------- host side
bool eig_i8_enabled(const Ctx* c) {
  static const bool off = [] { const char* e = std::getenv("AVD_EIG_SIMT"); return e && e[0] == '1'; }();
  // small m (c1, c2): the SIMT product's latency beats the digit conversions' fixed cost
  return !off && !c->gram_free && c->p <= 112 && c->gd != nullptr && c->cfg.m >= 3072;
}

// stage bytes and ring depth of one instantiation (<= ~200 KB of dynamic shared memory)
template <int P>
constexpr int g8_stages() {
  constexpr uint32_t kStage = ((kGDig * 128 * 128 + kQDig * P * 128 + 1023) / 1024) * 1024;
  return (int)((200u * 1024u) / kStage) > 4 ? 4 : (int)((200u * 1024u) / kStage);
}

void gemm_i8_geometry(int64_t m_pad, int num_sms, int64_t r0, int64_t r1, int* RB, int* KS, int* rb0) {
  *rb0 = 0;
  *RB = (int)(m_pad / 128);
  if (r1 > r0) { *rb0 = (int)(r0 / 128); *RB = (int)ceil_div(r1 - r0, 128); }
  const int NKC = (int)(m_pad / 128);
  *KS = (int)std::max<int64_t>(1, std::min<int64_t>(NKC, num_sms / std::max(1, *RB)));
}
size_t gemm_i8_part_bytes(int64_t m_pad, int p, int num_sms) {
  int RB, KS, rb0;
  gemm_i8_geometry(m_pad, num_sms, 0, 0, &RB, &KS, &rb0);
  return sizeof(double) * (size_t)std::max<int64_t>((int64_t)RB * KS, num_sms) * 128 * p;
}

avd_status eig_i8_prepare(Ctx* c) {  // once per solve: G -> digits; the tensor maps
  gdig_kernel<<<(unsigned)c->m_pad, 256, 0, c->stream>>>(c->G, c->cfg.m, c->m_pad, c->gd, c->gsc);
  AVD_LAUNCHED(c);
  if (!c->tm_gd_ready) {
    uint64_t gdims[2] = {(uint64_t)c->m_pad, (uint64_t)(kGDig * c->m_pad)};
    uint64_t gstr[1] = {(uint64_t)c->m_pad};
    uint32_t gbox[2] = {128, 128}, es[2] = {1, 1};
    uint64_t qdims[2] = {(uint64_t)c->m_pad, (uint64_t)(kQDig * c->p)};
    uint64_t qstr[1] = {(uint64_t)c->m_pad};
    uint32_t qbox[2] = {128, (uint32_t)c->p};
    if (tma_encode_fn()(&c->tm_gd, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->gd, gdims, gstr, gbox, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        tma_encode_fn()(&c->tm_qd, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, c->qd, qdims, qstr, qbox, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (eigensolver int8 maps)");
      return AVD_ECUDA;
    }
    AVD_CUDA(cudaMemcpyAsync(c->tm_dev, &c->tm_gd, sizeof(CUtensorMap), cudaMemcpyHostToDevice, c->stream));
    AVD_CUDA(cudaMemcpyAsync(c->tm_dev + 1, &c->tm_qd, sizeof(CUtensorMap), cudaMemcpyHostToDevice, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));  // (once per context: the host copies must outlive the call)
    c->tm_gd_ready = true;
  }
  return AVD_OK;
}

// Y = G In (In fp64 m x p; Y fp64 + optional fp32 mirror); rows [r0, r1) only when r1 > r0
avd_status gemm_i8(Ctx* c, const double* In, double* Y, float* Y32, const int* skip, int64_t r0, int64_t r1) {
  const int p = c->p;
  unsigned long long* qmax = reinterpret_cast<unsigned long long*>(c->qsc + kMaxP);
  AVD_CUDA(cudaMemsetAsync(qmax, 0, sizeof(unsigned long long) * p, c->stream));
  qmax_kernel<<<(unsigned)ceil_div(c->cfg.m, kQdTile), 256, sizeof(double) * kQdTile * p, c->stream>>>(
      In, c->cfg.m, p, qmax);
  AVD_LAUNCHED(c);
  qdig_kernel<<<(unsigned)(c->m_pad / kQdRows), 256, sizeof(double) * (kQdRows + 1) * p, c->stream>>>(
      In, c->cfg.m, c->m_pad, p, qmax, c->qd, c->qsc);
  AVD_LAUNCHED(c);
  double* out_colmax = nullptr;
  int RB, KS, rb0;
  gemm_i8_geometry(c->m_pad, c->num_sms, r0, r1, &RB, &KS, &rb0);
  unsigned* tickets = c->g8_tickets;
  switch (p) {
#define CASE(PP)                                                                                             \
  case PP: {                                                                                                 \
    constexpr int NS = g8_stages<PP>();                                                                      \
    constexpr uint32_t kStage = ((kGDig * 128 * 128 + kQDig * PP * 128 + 1023) / 1024) * 1024;               \
    const size_t smem = (size_t)NS * kStage + 1024;                                                          \
    AVD_CUDA(smem_attr(gemm_i8_kernel<PP, NS>, (int)smem));                                                  \
    gemm_i8_kernel<PP, NS><<<RB * KS, kG8Threads, smem, c->stream>>>(c->tm_dev, c->tm_dev + 1, c->cfg.m, c->m_pad, KS, \
                                                                     rb0, c->gsc, c->qsc, c->g8_part, tickets, \
                                                                     Y, Y32, out_colmax, skip);                \
    break;                                                                                                   \
  }
    CASE(16) CASE(32) CASE(48) CASE(64) CASE(80) CASE(96) CASE(112)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
