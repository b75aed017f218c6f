// k_eig.cu — K4: top-k eigenpairs of the centred Gram G (fp64, on device) by block subspace
// iteration with Rayleigh-Ritz: V_k, sigma_k = sqrt(lambda_k) are the right singular vectors /
// values of Xc that define the rank-k spike.
//
//   Q_0 = orth(random m x p), p = roundup16(k + 8)
//   repeat:  Y = G Q ; H = Q^T Y ; (W, theta) = eig(H)           (Rayleigh-Ritz)
//            U = Q W ; Z = Y W (= G U)  ; res_r = ||Z_r - theta_r U_r|| / theta_1, r < k
//            stop when max res_r <= tol ;  Q = orth(Z)              (SVQB, twice)
// p x p symmetric eigenproblems are solved by a one-CTA parallel (round-robin) Jacobi.
// Everything is fp64; every reduction has a fixed order (deterministic).
#include <cfloat>
#include "common.cuh"

namespace avd {

namespace {

// ---------------------------------------------------------------- G_int -> G (fp64)
__global__ void gram_finalize_kernel(const long long* __restrict__ Gi, int64_t m, int64_t m_pad,
                                     const int32_t* __restrict__ shift, double unit, double* __restrict__ G) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t a = blockIdx.y;
  if (b >= m) return;
  const bool upper = (a / 128) <= (b / 128);
  const long long v = upper ? Gi[a * m_pad + b] : Gi[b * m_pad + a];
  G[a * m + b] = ldexp((double)v * unit, -(shift[a] + shift[b]));
}

__global__ void trace_kernel(const double* __restrict__ G, int64_t m, double* __restrict__ out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) s += G[j * m + j];
  sh[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 256; ++i) t += sh[i];
    *out = t;
  }
}

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ double rnd_sym(uint32_t seed, uint32_t a, uint32_t b) {
  const uint32_t h = mix32(a * 0x9E3779B1u ^ mix32(b ^ mix32(seed)));
  return ((double)(h >> 8) + 0.5) * (2.0 / 16777216.0) - 1.0;
}

// Q[j][c] = U(-1,1) for columns with flag (or all when flags == nullptr)
__global__ void rand_fill_kernel(double* __restrict__ Q, int64_t m, int p, uint32_t seed,
                                 const int* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * p) return;
  const int c = (int)(t % p);
  if (flags && !flags[c]) return;
  Q[t] = rnd_sym(seed, (uint32_t)(t / p), (uint32_t)c);
}

// ---------------------------------------------------------------- Y = G Q  (m x m) (m x p)
constexpr int kGB = 32;  // rows of Y per CTA and K chunk
template <int PC>  // PC = p / 16 column groups
__global__ void __launch_bounds__(256) gemm_gq_kernel(const double* __restrict__ G, const double* __restrict__ Q,
                                                      int64_t m, double* __restrict__ Y) {
  constexpr int p = PC * 16;
  __shared__ double sG[kGB][kGB + 1];
  __shared__ double sQ[kGB][p];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = (int64_t)blockIdx.x * kGB;
  double acc[2][PC];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < PC; ++c) acc[a][c] = 0.0;
  for (int64_t k0 = 0; k0 < m; k0 += kGB) {
    for (int t = threadIdx.x; t < kGB * kGB; t += 256) {
      const int rr = t / kGB, kk = t % kGB;
      sG[rr][kk] = (r0 + rr < m && k0 + kk < m) ? G[(r0 + rr) * m + k0 + kk] : 0.0;
    }
    for (int t = threadIdx.x; t < kGB * p; t += 256) {
      const int kk = t / p, cc = t % p;
      sQ[kk][cc] = (k0 + kk < m) ? Q[(k0 + kk) * p + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kGB; ++kk) {
      const double g0 = sG[ty * 2][kk], g1 = sG[ty * 2 + 1][kk];
#pragma unroll
      for (int c = 0; c < PC; ++c) {
        const double qv = sQ[kk][tx + 16 * c];
        acc[0][c] = fma(g0, qv, acc[0][c]);
        acc[1][c] = fma(g1, qv, acc[1][c]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int64_t r = r0 + ty * 2 + a;
    if (r < m)
#pragma unroll
      for (int c = 0; c < PC; ++c) Y[r * p + tx + 16 * c] = acc[a][c];
  }
}

// ---------------------------------------------------------------- C = A^T B partials (m x p)
constexpr int kRedRows = 32;
__global__ void __launch_bounds__(256) atb_partial_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                          int64_t m, int p, double* __restrict__ part) {
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + kRedRows * p;
  const int64_t r0 = (int64_t)blockIdx.x * kRedRows;
  for (int t = threadIdx.x; t < kRedRows * p; t += 256) {
    const int rr = t / p;
    const bool ok = r0 + rr < m;
    sA[t] = ok ? A[r0 * p + t] : 0.0;
    sB[t] = ok ? B[r0 * p + t] : 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < p * p; t += 256) {
    const int i = t / p, j = t % p;
    double s = 0.0;
#pragma unroll 8
    for (int rr = 0; rr < kRedRows; ++rr) s = fma(sA[rr * p + i], sB[rr * p + j], s);
    part[(int64_t)blockIdx.x * p * p + t] = s;
  }
}
__global__ void red_sum_kernel(const double* __restrict__ part, int nparts, int n, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double s = 0.0;
  for (int q = 0; q < nparts; ++q) s += part[(int64_t)q * n + t];
  out[t] = s;
}

// ---------------------------------------------------------------- Out = In * M (m x p)(p x p)
__global__ void __launch_bounds__(256) matpp_kernel(const double* __restrict__ In0, double* __restrict__ Out0,
                                                    const double* __restrict__ In1, double* __restrict__ Out1,
                                                    const double* __restrict__ M, int64_t m, int p) {
  extern __shared__ double sm[];
  double* sM = sm;                 // p*p
  double* sI = sm + p * p;         // 16 rows x p
  for (int t = threadIdx.x; t < p * p; t += 256) sM[t] = M[t];
  const int64_t r0 = (int64_t)blockIdx.x * 16;
  for (int w = 0; w < 2; ++w) {
    const double* In = w ? In1 : In0;
    double* Out = w ? Out1 : Out0;
    if (!In) continue;
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * p; t += 256) sI[t] = (r0 + t / p < m) ? In[r0 * p + t] : 0.0;
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * p; t += 256) {
      const int rr = t / p, cc = t % p;
      if (r0 + rr >= m) continue;
      double s = 0.0;
      for (int q = 0; q < p; ++q) s = fma(sI[rr * p + q], sM[q * p + cc], s);
      Out[(r0 + rr) * p + cc] = s;
    }
  }
}

// ---------------------------------------------------------------- residuals of Ritz pairs
__global__ void resid_kernel(const double* __restrict__ Z, const double* __restrict__ U,
                             const double* __restrict__ theta, int64_t m, int p, double* __restrict__ res) {
  __shared__ double sh[256];
  const int r = blockIdx.x;
  const double th = theta[r];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double d = Z[j * p + r] - th * U[j * p + r];
    s = fma(d, d, s);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double t0 = fabs(theta[0]) > 0 ? fabs(theta[0]) : 1.0;
    res[r] = sqrt(sh[0]) / t0;
  }
}

// ---------------------------------------------------------------- p x p symmetric Jacobi
// mode 0: W = eigenvectors (columns, sorted by eigenvalue desc), evals = eigenvalues
// mode 1: W = eigvecs * diag(d^-1/2) (0 for d <= 1e-13 d_max), bad[c] = 1 for zeroed columns
__global__ void __launch_bounds__(512) jacobi_kernel(const double* __restrict__ Ain, int p, int mode,
                                                     double* __restrict__ Wout, double* __restrict__ evals,
                                                     int* __restrict__ bad) {
  extern __shared__ double sm[];
  const int ld = p + 1;
  double* A = sm;
  double* V = sm + p * ld;
  __shared__ double cs[kMaxP / 2][2];
  __shared__ int pq[kMaxP / 2][2];
  __shared__ int rotated;
  __shared__ double dsh[kMaxP];
  __shared__ int rank_sh[kMaxP];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int t = tid; t < p * p; t += nt) {
    const int i = t / p, j = t % p;
    A[i * ld + j] = 0.5 * (Ain[i * p + j] + Ain[j * p + i]);
    V[i * ld + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int half = p / 2;
  for (int sweep = 0; sweep < 40; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int step = 0; step < p - 1; ++step) {
      if (tid < half) {
        int a, b;
        if (tid == 0) { a = p - 1; b = step; }
        else { a = (step + tid) % (p - 1); b = (step - tid + (p - 1)) % (p - 1); }
        const int P_ = min(a, b), Q_ = max(a, b);
        pq[tid][0] = P_; pq[tid][1] = Q_;
        const double app = A[P_ * ld + P_], aqq = A[Q_ * ld + Q_], apq = A[P_ * ld + Q_];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > 1e-300 && fabs(apq) > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
          const double th = (aqq - app) / (2.0 * apq);
          double t;
          if (fabs(th) > 1e150) t = 0.5 / th;
          else t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
          rotated = 1;
        }
        cs[tid][0] = c; cs[tid][1] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int t = tid; t < half * p; t += nt) {
        const int i = t / p, col = t % p;
        const double c = cs[i][0], s = cs[i][1];
        if (s == 0.0) continue;
        const int P_ = pq[i][0], Q_ = pq[i][1];
        const double ap = A[P_ * ld + col], aq = A[Q_ * ld + col];
        A[P_ * ld + col] = c * ap - s * aq;
        A[Q_ * ld + col] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J, V <- V J
      for (int t = tid; t < half * p; t += nt) {
        const int i = t / p, row = t % p;
        const double c = cs[i][0], s = cs[i][1];
        if (s == 0.0) continue;
        const int P_ = pq[i][0], Q_ = pq[i][1];
        const double ap = A[row * ld + P_], aq = A[row * ld + Q_];
        A[row * ld + P_] = c * ap - s * aq;
        A[row * ld + Q_] = s * ap + c * aq;
        const double vp = V[row * ld + P_], vq = V[row * ld + Q_];
        V[row * ld + P_] = c * vp - s * vq;
        V[row * ld + Q_] = s * vp + c * vq;
      }
      __syncthreads();
      if (tid < half && cs[tid][1] != 0.0) {
        const int P_ = pq[tid][0], Q_ = pq[tid][1];
        A[P_ * ld + Q_] = 0.0;
        A[Q_ * ld + P_] = 0.0;
      }
      __syncthreads();
    }
    if (!rotated) break;
  }
  // sort eigenvalues descending (ties by index)
  if (tid < p) dsh[tid] = A[tid * ld + tid];
  __syncthreads();
  if (tid < p) {
    int rk = 0;
    const double di = dsh[tid];
    for (int j = 0; j < p; ++j) rk += (dsh[j] > di) || (dsh[j] == di && j < tid);
    rank_sh[tid] = rk;
  }
  __syncthreads();
  double dmax = 0.0;
  for (int j = 0; j < p; ++j) dmax = fmax(dmax, dsh[j]);
  for (int t = tid; t < p * p; t += nt) {
    const int row = t / p, i = t % p;  // source column i -> rank_sh[i]
    double f = 1.0;
    if (mode == 1) f = (dsh[i] > 1e-13 * dmax && dsh[i] > 0.0) ? 1.0 / sqrt(dsh[i]) : 0.0;
    Wout[row * p + rank_sh[i]] = V[row * ld + i] * f;
  }
  if (tid < p) {
    evals[rank_sh[tid]] = dsh[tid];
    if (mode == 1 && bad) bad[rank_sh[tid]] = (dsh[tid] > 1e-13 * dmax && dsh[tid] > 0.0) ? 0 : 1;
  }
}

// V_out[j][r] = sign_r * U[j][r] (r < k), sign making the largest-|.| entry positive
// (smallest j on ties; R8); sigma_r = sqrt(max(theta_r, 0)); V32 fp32 copy.
__global__ void finalize_vectors_kernel(const double* __restrict__ U, const double* __restrict__ theta, int64_t m,
                                        int p, int k, int k_pad, double* __restrict__ V, double* __restrict__ sigma,
                                        float* __restrict__ V32) {
  __shared__ double sv[256];
  __shared__ int64_t sj[256];
  const int r = blockIdx.x;
  double best = -1.0;
  int64_t bj = 0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double a = fabs(U[j * p + r]);
    if (a > best) { best = a; bj = j; }
  }
  sv[threadIdx.x] = best;
  sj[threadIdx.x] = bj;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int t = 1; t < 256; ++t)
      if (sv[t] > sv[0] || (sv[t] == sv[0] && sj[t] < sj[0])) { sv[0] = sv[t]; sj[0] = sj[t]; }
  }
  __syncthreads();
  const double sg = U[sj[0] * p + r] < 0.0 ? -1.0 : 1.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double v = sg * U[j * p + r];
    V[j * k + r] = v;
    V32[j * k_pad + r] = (float)v;
  }
  if (threadIdx.x == 0) sigma[r] = sqrt(fmax(theta[r], 0.0));
}

}  // namespace

avd_status launch_gram_finalize(Ctx* c) {
  const int64_t m = c->cfg.m;
  const double unit = (c->nd == 3) ? 16384.0 : 1.0;
  dim3 grid((unsigned)ceil_div(m, 256), (unsigned)m);
  gram_finalize_kernel<<<grid, 256, 0, c->stream>>>(c->gram_i, m, c->m_pad, c->shift, unit, c->G);
  AVD_LAUNCHED(c);
  trace_kernel<<<1, 256, 0, c->stream>>>(c->G, m, c->trace);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

namespace {

avd_status launch_gemm_gq(Ctx* c) {
  const int64_t m = c->cfg.m;
  const unsigned grid = (unsigned)ceil_div(m, kGB);
  switch (c->p / 16) {
#define CASE(PC) case PC: gemm_gq_kernel<PC><<<grid, 256, 0, c->stream>>>(c->G, c->Q, m, c->Y); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_atb(Ctx* c, const double* A, const double* B, double* out) {
  const int64_t m = c->cfg.m;
  const int p = c->p;
  const size_t sm = 2 * kRedRows * p * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(atb_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  atb_partial_kernel<<<c->n_red, 256, sm, c->stream>>>(A, B, m, p, c->red_part);
  AVD_LAUNCHED(c);
  red_sum_kernel<<<(unsigned)ceil_div(p * p, 256), 256, 0, c->stream>>>(c->red_part, c->n_red, p * p, out);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_jacobi(Ctx* c, const double* A, int mode, double* W, double* ev, int* bad) {
  const size_t sm = 2 * (size_t)c->p * (c->p + 1) * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  jacobi_kernel<<<1, 512, sm, c->stream>>>(A, c->p, mode, W, ev, bad);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status launch_matpp(Ctx* c, const double* In0, double* Out0, const double* In1, double* Out1, const double* M) {
  const int p = c->p;
  const size_t sm = ((size_t)p * p + 16 * p) * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(matpp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  matpp_kernel<<<(unsigned)ceil_div(c->cfg.m, 16), 256, sm, c->stream>>>(In0, Out0, In1, Out1, M, c->cfg.m, p);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// Q <- orth(Z) by SVQB (twice); rank-deficient directions are re-drawn at random.
avd_status svqb(Ctx* c, double* Z, double* Q, uint32_t seed) {
  int* bad = reinterpret_cast<int*>(c->resid + c->p);  // scratch after resid[p]
  double* ev = c->theta + c->p;                         // scratch evals
  for (int pass = 0; pass < 2; ++pass) {
    double* src = pass == 0 ? Z : Q;
    AVD_TRY(launch_atb(c, src, src, c->H));
    AVD_TRY(launch_jacobi(c, c->H, 1, c->W, ev, bad));
    AVD_TRY(launch_matpp(c, src, c->U, nullptr, nullptr, c->W));  // U as temp
    AVD_CUDA(cudaMemcpyAsync(Q, c->U, sizeof(double) * c->cfg.m * c->p, cudaMemcpyDeviceToDevice, c->stream));
    if (pass == 0) {
      rand_fill_kernel<<<(unsigned)ceil_div(c->cfg.m * c->p, 256), 256, 0, c->stream>>>(Q, c->cfg.m, c->p,
                                                                                         seed, bad);
      AVD_LAUNCHED(c);
    }
  }
  return AVD_OK;
}

}  // namespace

avd_status run_eig(Ctx* c) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  const uint32_t seed = (uint32_t)(c->cfg.seed ^ (c->cfg.seed >> 32)) * 2654435761u + 12345u;
  rand_fill_kernel<<<(unsigned)ceil_div(m * p, 256), 256, 0, c->stream>>>(c->Z, m, p, seed, nullptr);
  AVD_LAUNCHED(c);
  AVD_TRY(svqb(c, c->Z, c->Q, seed + 1));
  const int max_it = c->cfg.max_iters > 0 ? c->cfg.max_iters : 200;
  const double tol = c->cfg.eig_tol > 0 ? c->cfg.eig_tol : 1e-10;
  int it = 0;
  double maxres = 0.0;
  bool conv = false;
  for (it = 1; it <= max_it; ++it) {
    AVD_TRY(launch_gemm_gq(c));                              // Y = G Q
    AVD_TRY(launch_atb(c, c->Q, c->Y, c->H));                // H = Q^T Y
    AVD_TRY(launch_jacobi(c, c->H, 0, c->W, c->theta, nullptr));
    AVD_TRY(launch_matpp(c, c->Y, c->Z, c->Q, c->U, c->W));  // Z = Y W, U = Q W
    resid_kernel<<<k, 256, 0, c->stream>>>(c->Z, c->U, c->theta, m, p, c->resid);
    AVD_LAUNCHED(c);
    AVD_CUDA(cudaMemcpyAsync(c->eig_host, c->theta, sizeof(double) * p, cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaMemcpyAsync(c->eig_host + p, c->resid, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));
    maxres = 0.0;
    for (int r = 0; r < k; ++r) maxres = std::max(maxres, c->eig_host[p + r]);
    if (!(c->eig_host[0] > 0.0)) { maxres = 0.0; conv = true; break; }  // G == 0: nothing to iterate
    if (maxres <= tol) { conv = true; break; }
    if (it == max_it) break;
    AVD_TRY(svqb(c, c->Z, c->Q, seed + 7919u * (uint32_t)it));
  }
  c->iters = std::min(it, max_it);
  c->max_resid = maxres;
  c->sigma_next = (k < p) ? std::sqrt(std::max(c->eig_host[k], 0.0)) : 0.0;
  AVD_CUDA(cudaMemsetAsync(c->V32, 0, sizeof(float) * m * c->k_pad, c->stream));
  finalize_vectors_kernel<<<k, 256, 0, c->stream>>>(c->U, c->theta, m, p, k, c->k_pad, c->V, c->sigma, c->V32);
  AVD_LAUNCHED(c);
  return conv ? AVD_OK : AVD_ENOCONV;
}

}  // namespace avd
