// k_project.cu — K5 + K8 fused, one CTA per block of 32 rows:
//   phase 1 (K5): P_i = xc_i V_k  (row projections; spike_i = P_i V_k^T)
//   phase 2 (K8): spike_ij = P_i . V_j, tail_ij = xc_ij - spike_ij and the
//                 elementwise energies sum spike^2, sum tail^2, sum spike*tail, sum xc^2
//                 (checked against the closed forms of PAPER.md:15-17), plus column sums of P
//                 (column means of spike = (1/l) (1^T P) V^T, "zero column means").
// X is read from HBM in phase 1 and from L2 in phase 2 (the 32-row block is L2-resident).
#include "common.cuh"

namespace avd {

namespace {

constexpr int kRB = 32;   // rows per CTA
constexpr int kCK = 64;   // columns per chunk
constexpr int kProjThreads = 256;

template <int KPC>  // k_pad / 16
__global__ void __launch_bounds__(kProjThreads) project_kernel(
    const float* __restrict__ X, int64_t l_local, int64_t m, const double* __restrict__ mu,
    const float* __restrict__ V32, float* __restrict__ P, double* __restrict__ en_part,
    double* __restrict__ colsumP_part) {
  constexpr int KP = KPC * 16;
  __shared__ float xs[kCK][kRB + 1];   // xc transposed [col][row]
  __shared__ float vs[kCK][KP];        // V rows of the chunk
  __shared__ float ps[kRB][KP + 1];    // P of the block
  __shared__ double red[kProjThreads / 32][4];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // phase 1: rows 2ty, 2ty+1 ; cols tx + 16c
  const int64_t r0 = (int64_t)blockIdx.x * kRB;

  auto load_chunk = [&](int64_t j0) {
    // X tile kRB x kCK -> xs (centred, transposed); 256 threads x 8 elements
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int t = tid + e * kProjThreads;
      const int rr = t / kCK, cc = t % kCK;
      const int64_t i = r0 + rr, j = j0 + cc;
      float v = 0.f;
      if (i < l_local && j < m) v = (float)((double)__ldg(X + i * m + j) - mu[j]);
      xs[cc][rr] = v;
    }
    for (int t = tid; t < kCK * KP; t += kProjThreads) {
      const int cc = t / KP, rcol = t % KP;
      const int64_t j = j0 + cc;
      vs[cc][rcol] = (j < m) ? V32[j * KP + rcol] : 0.f;
    }
  };

  // ---------------- phase 1: P = Xc V
  float acc[2][KPC];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < KPC; ++c) acc[a][c] = 0.f;
  for (int64_t j0 = 0; j0 < m; j0 += kCK) {
    __syncthreads();
    load_chunk(j0);
    __syncthreads();
#pragma unroll 8
    for (int cc = 0; cc < kCK; ++cc) {
      const float x0 = xs[cc][2 * ty], x1 = xs[cc][2 * ty + 1];
#pragma unroll
      for (int c = 0; c < KPC; ++c) {
        const float v = vs[cc][tx + 16 * c];
        acc[0][c] = fmaf(x0, v, acc[0][c]);
        acc[1][c] = fmaf(x1, v, acc[1][c]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t i = r0 + 2 * ty + a;
#pragma unroll
    for (int c = 0; c < KPC; ++c) {
      const float pv = (i < l_local) ? acc[a][c] : 0.f;
      ps[2 * ty + a][tx + 16 * c] = pv;
      if (i < l_local) P[i * KP + tx + 16 * c] = pv;
    }
  }
  __syncthreads();
  if (tid < KP) {
    double s = 0.0;
    for (int rr = 0; rr < kRB; ++rr) s += (double)ps[rr][tid];
    colsumP_part[(int64_t)blockIdx.x * KP + tid] = s;
  }

  // ---------------- phase 2: spike / tail energies; thread -> row (tid & 31), 8 columns
  const int rr = tid & 31;
  const int cg = tid >> 5;  // columns cg*8 .. cg*8+7 of the chunk
  double eS = 0.0, eT = 0.0, eST = 0.0, eX = 0.0;
  for (int64_t j0 = 0; j0 < m; j0 += kCK) {
    __syncthreads();
    load_chunk(j0);
    __syncthreads();
    float s8[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s8[q] = 0.f;
#pragma unroll 4
    for (int r = 0; r < KP; ++r) {
      const float pv = ps[rr][r];
#pragma unroll
      for (int q = 0; q < 8; ++q) s8[q] = fmaf(pv, vs[cg * 8 + q][r], s8[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float xc = xs[cg * 8 + q][rr];
      const double S = (double)s8[q];
      const double T = (double)xc - S;
      eS = fma(S, S, eS);
      eT = fma(T, T, eT);
      eST = fma(S, T, eST);
      eX = fma((double)xc, (double)xc, eX);
    }
  }
  // fixed-order block reduction
  for (int o = 16; o > 0; o >>= 1) {
    eS += __shfl_xor_sync(0xFFFFFFFFu, eS, o);
    eT += __shfl_xor_sync(0xFFFFFFFFu, eT, o);
    eST += __shfl_xor_sync(0xFFFFFFFFu, eST, o);
    eX += __shfl_xor_sync(0xFFFFFFFFu, eX, o);
  }
  if ((tid & 31) == 0) {
    red[tid >> 5][0] = eS; red[tid >> 5][1] = eT; red[tid >> 5][2] = eST; red[tid >> 5][3] = eX;
  }
  __syncthreads();
  if (tid < 4) {
    double s = 0.0;
    for (int w = 0; w < kProjThreads / 32; ++w) s += red[w][tid];
    en_part[(int64_t)blockIdx.x * 4 + tid] = s;
  }
}

// energy[0..4) = sum S^2, T^2, ST, xc^2 ; energy[4..4+KP) = column sums of P
// one CTA per output value: strided partial sums + fixed-order tree (deterministic)
__global__ void project_reduce_kernel(const double* __restrict__ en_part, const double* __restrict__ colsumP_part,
                                      int nparts, int KP, double* __restrict__ energy) {
  __shared__ double sh[256];
  const int o = blockIdx.x;
  const double* src = o < 4 ? en_part + o : colsumP_part + (o - 4);
  const int stride = o < 4 ? 4 : KP;
  double s = 0.0;
  for (int q = threadIdx.x; q < nparts; q += 256) s += src[(int64_t)q * stride];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) energy[o] = sh[0];
}

// p_i = x_i . mu_hat = P[i][k] + ||mu||: counts of p_i > 0 and p_i < 0 added to
// cnt[0], cnt[1] as integer-valued doubles (exact, order-free; exchanged with the energies)
__global__ void sign_count_kernel(const float* __restrict__ P, int64_t l, int kpad, int k,
                                  const double* __restrict__ diag, double* __restrict__ cnt) {
  __shared__ unsigned int sp, sn;
  if (threadIdx.x == 0) { sp = 0; sn = 0; }
  __syncthreads();
  const double nrm = diag[0];
  unsigned int pos = 0, neg = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < l; i += (int64_t)gridDim.x * blockDim.x) {
    const double p = (double)P[i * kpad + k] + nrm;
    pos += p > 0.0 ? 1u : 0u;
    neg += p < 0.0 ? 1u : 0u;
  }
  if (nrm > 0.0) {
    atomicAdd(&sp, pos);
    atomicAdd(&sn, neg);
  }
  __syncthreads();
  if (threadIdx.x == 0 && (sp || sn)) {
    atomicAdd(&cnt[0], (double)sp);
    atomicAdd(&cnt[1], (double)sn);
  }
}

}  // namespace

avd_status launch_sign_count(Ctx* c) {
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c->cfg.l_local, 256), 2LL * c->num_sms));
  sign_count_kernel<<<grid, 256, 0, c->stream>>>(c->P, c->cfg.l_local, c->k_pad, c->k, c->diag,
                                                 c->energy + 4 + c->k_pad);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_project(Ctx* c, const float* X) {
  AVD_CUDA(cudaMemsetAsync(c->energy + 4 + c->k_pad, 0, 2 * sizeof(double), c->stream));
  c->sign_valid = project_tc_supported(c, X);
  if (project_tc_supported(c, X)) {
    AVD_TRY(launch_project_tc(c, X));
    project_reduce_kernel<<<4 + c->k_pad, 256, 0, c->stream>>>(c->en_part, c->colsumP_part, c->n_proj_ctas, c->k_pad,
                                                                c->energy);
    AVD_LAUNCHED(c);
    return launch_sign_count(c);  // P[:, k] = xc . mu_hat (split_v_kernel)
  }
  const unsigned grid = (unsigned)c->n_proj_ctas;
  switch (c->k_pad / 16) {
#define CASE(K)                                                                                         \
  case K:                                                                                               \
    project_kernel<K><<<grid, kProjThreads, 0, c->stream>>>(X, c->cfg.l_local, c->cfg.m, c->mu, c->V32, \
                                                            c->P, c->en_part, c->colsumP_part);         \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6)
#undef CASE
    default: set_error("unsupported k_pad"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  project_reduce_kernel<<<4 + c->k_pad, 256, 0, c->stream>>>(c->en_part, c->colsumP_part, c->n_proj_ctas, c->k_pad,
                                                              c->energy);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

}  // namespace avd
