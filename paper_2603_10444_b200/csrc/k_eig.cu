// k_eig.cu — K4: top-k eigenpairs of the centred Gram G (fp64, on device) by block subspace
// iteration with Rayleigh-Ritz: V_k, sigma_k = sqrt(lambda_k) are the right singular vectors /
// values of Xc that define the rank-k spike.
//
//   Q_0 = orth(random m x p), p = roundup16(k + 8)
//   repeat:  Y = G Q ; H = Q^T Y ; (W, theta) = eig(H)            (Rayleigh-Ritz)
//            U = Q W ; Z = Y W (= G U) ; res_r = ||Z_r - theta_r U_r|| / theta_1, r < k
//            stop when max res_r <= tol
//            Q = orth(G Z)   (two products per orthonormalisation: G^2 U, Cholesky-QR2)
// p x p problems run in one CTA each: parallel (round-robin) Jacobi for Rayleigh-Ritz,
// Cholesky + triangular inverse for CholQR; the m-length reductions feeding them are
// multi-CTA partial sums finished inside those one-CTA kernels in a fixed order.
// Rank deficiency (G = 0, rank(G) < p, m < p) flags the failing columns, which are re-drawn at
// random and re-orthonormalised (R11).  Everything is fp64 and deterministic.
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
  // K3 adds tile (A, B), A <= B, transposed: element (a, b) of an upper tile sits at Gi[b][a]
  const bool upper = (a / 128) <= (b / 128);
  const long long v = upper ? Gi[b * m_pad + a] : Gi[a * m_pad + b];
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

// ---------------------------------------------------------------- Y = G Q  (split-K partials)
// CTA: 64 rows of Y x all p columns, K range [kz*kchunk, (kz+1)*kchunk); 128 threads, each an
// 8-row x (p/16)-column register tile; register-prefetched double buffer (the next K stage's
// global loads are in flight while the current stage computes).  Ypart[kz][m][p].
constexpr int kGM = 64;   // rows per CTA
constexpr int kGK = 32;   // K per smem stage
template <int PC>
__global__ void __launch_bounds__(128, (PC <= 4 ? 3 : 1)) gemm_gq_kernel(const double* __restrict__ G, const double* __restrict__ Q,
                                                      int64_t m, int64_t kchunk, double* __restrict__ Ypart) {
  constexpr int p = PC * 16;
  constexpr int NG = (kGM * kGK) / 128;   // G values per thread per stage
  constexpr int NQ = (kGK * p) / 128;     // Q values per thread per stage
  constexpr int SG = kGK * (kGM + 2);     // doubles of one transposed G tile [k][row]
  constexpr int SQ = kGK * p;
  extern __shared__ __align__(16) double gsm[];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // rows 8ty..8ty+7, cols tx+16c
  const int64_t r0 = (int64_t)blockIdx.x * kGM;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk;
  const int64_t kend = min(m, kbeg + kchunk);
  double acc[8][PC];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int c = 0; c < PC; ++c) acc[a][c] = 0.0;
  double gv[NG], qv[NQ];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      const int t = threadIdx.x + e * 128;
      const int rr = t / kGK, kk = t % kGK;
      gv[e] = (r0 + rr < m && k0 + kk < kend) ? __ldg(G + (r0 + rr) * m + k0 + kk) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < NQ; ++e) {
      const int t = threadIdx.x + e * 128;
      const int kk = t / p;
      qv[e] = (k0 + kk < kend) ? __ldg(Q + (k0 + kk) * p + (t % p)) : 0.0;
    }
  };
  auto store = [&](int buf) {
    double* sG = gsm + buf * (SG + SQ);
    double* sQ = sG + SG;
#pragma unroll
    for (int e = 0; e < NG; ++e) {
      const int t = threadIdx.x + e * 128;
      sG[(t % kGK) * (kGM + 2) + t / kGK] = gv[e];
    }
#pragma unroll
    for (int e = 0; e < NQ; ++e) sQ[threadIdx.x + e * 128] = qv[e];
  };
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = kbeg; k0 < kend; k0 += kGK, buf ^= 1) {
    const bool more = k0 + kGK < kend;
    if (more) load(k0 + kGK);
    const double* sG = gsm + buf * (SG + SQ);
    const double* sQ = sG + SG;
#pragma unroll 2
    for (int kk = 0; kk < kGK; ++kk) {
      double g[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = *reinterpret_cast<const double2*>(sG + kk * (kGM + 2) + 8 * ty + 2 * h);
        g[2 * h] = v.x;
        g[2 * h + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < PC; ++c) {
        const double q = sQ[kk * p + tx + 16 * c];
#pragma unroll
        for (int a = 0; a < 8; ++a) acc[a][c] = fma(g[a], q, acc[a][c]);
      }
    }
    if (more) store(buf ^ 1);
    __syncthreads();
  }
  double* Yp = Ypart + (int64_t)blockIdx.y * m * p;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int64_t r = r0 + 8 * ty + a;
    if (r < m)
#pragma unroll
      for (int c = 0; c < PC; ++c) Yp[r * p + tx + 16 * c] = acc[a][c];
  }
}

__global__ void ksum_kernel(const double* __restrict__ part, int nparts, int64_t n, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double s = part[t];
  for (int q = 1; q < nparts; ++q) s += part[(int64_t)q * n + t];
  out[t] = s;
}

// ---------------------------------------------------------------- C = A^T B partials (m x p)
// CTA: kRedRowsC rows in 64-row smem chunks; thread owns PC^2 outputs (p^2 = 256 PC^2).
constexpr int kRedChunk = 64;
template <int PC>
__global__ void __launch_bounds__(256) atb_partial_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                                          int64_t m, double* __restrict__ part) {
  constexpr int p = PC * 16;
  constexpr int U = PC * PC;
  extern __shared__ double sm[];
  double* sA = sm;
  double* sB = sm + kRedChunk * p;
  double acc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) acc[u] = 0.0;
  const int64_t rbase = (int64_t)blockIdx.x * kRedRowsC;
  for (int ch = 0; ch < kRedRowsC / kRedChunk; ++ch) {
    const int64_t r0 = rbase + ch * kRedChunk;
    if (r0 >= m) break;
    __syncthreads();
    for (int t = threadIdx.x; t < kRedChunk * p; t += 256) {
      const int rr = t / p;
      const bool ok = r0 + rr < m;
      sA[t] = ok ? A[r0 * p + t] : 0.0;
      sB[t] = ok ? B[r0 * p + t] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = threadIdx.x + 256 * u;
      const int i = t / p, j = t % p;
      double s = acc[u];
#pragma unroll 8
      for (int rr = 0; rr < kRedChunk; ++rr) s = fma(sA[rr * p + i], sB[rr * p + j], s);
      acc[u] = s;
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) part[(int64_t)blockIdx.x * p * p + threadIdx.x + 256 * u] = acc[u];
}

// ---------------------------------------------------------------- Out = In * M (m x p)(p x p)
// in place allowed (each CTA stages its rows before writing them)
__global__ void __launch_bounds__(256) matpp_kernel(const double* In0, double* Out0, const double* In1,
                                                    double* Out1, const double* __restrict__ M, int64_t m, int p) {
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

// out[t] = sum_q part[q][t] in a fixed order (independent loads, unrolled)
__global__ void psum_kernel(const double* __restrict__ part, int nparts, int n, double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int q = 0;
  for (; q + 8 <= nparts; q += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] += part[(int64_t)(q + u) * n + t];
  }
  for (; q < nparts; ++q) a[0] += part[(int64_t)q * n + t];
  out[t] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// sum nparts partials of a p x p matrix into smem A (ld), symmetrised
__device__ void load_sym(const double* __restrict__ part, int nparts, int p, double* A, int ld) {
  for (int t = threadIdx.x; t < p * p; t += blockDim.x) {
    const int i = t / p, j = t % p;
    if (j < i) continue;
    double s = 0.0, s2 = 0.0;
    for (int q = 0; q < nparts; ++q) {
      s += part[(int64_t)q * p * p + i * p + j];
      s2 += part[(int64_t)q * p * p + j * p + i];
    }
    const double v = 0.5 * (s + s2);
    A[i * ld + j] = v;
    A[j * ld + i] = v;
  }
}

// ---------------------------------------------------------------- p x p symmetric Jacobi
// Parallel round-robin Jacobi, one CTA of 16 warps.  In each of the p-1 steps of a sweep the p/2
// disjoint pairs are owned by warps (pair i -> warp i % 16); lane 0 of the owner computes the
// rotation (Rutishauser, fp32 seeds + Newton to fp64 accuracy) and broadcasts it by shuffle, the
// warp rotates rows P,Q (lanes over columns), barrier, then columns P,Q of A and V (lanes over
// rows), barrier.  W = eigenvectors (columns sorted by eigenvalue desc), evals; stats[0] = sweeps.
constexpr int kJW = 16;  // warps
__device__ __forceinline__ double rcp_fast(double x) {  // 1/x, MUFU seed + 2 Newton steps (~1 ulp)
  double r = (double)(1.0f / (float)x);
  r = r * fma(-x, r, 2.0);
  return r * fma(-x, r, 2.0);
}
__device__ __forceinline__ double rsqrt_fast(double x) {  // 1/sqrt(x), x in the fp32 range
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x * r, r, 1.5);
  return r * fma(-0.5 * x * r, r, 1.5);
}
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double& c, double& s, bool& rot) {
  c = 1.0;
  s = 0.0;
  rot = false;
  // skip when a_pq^2 <= 1e-26 a_pp a_qq (|a_pq| <= 1e-13 sqrt(a_pp a_qq)) or a_pq is below fp32 range
  if (!(apq * apq > 1e-26 * fabs(app * aqq)) || fabs(apq) < 1e-30 || fabs(apq) > 1e30) return;
  // Rutishauser: th = (a_qq - a_pp) / (2 a_pq), t = sign(th) / (|th| + sqrt(th^2 + 1))
  const double th = 0.5 * (aqq - app) * rcp_fast(apq);
  double t;
  const double ath = fabs(th);
  if (ath > 1e18) {
    t = 0.5 / th;
  } else {
    const double y = fma(th, th, 1.0);
    const double ri = rcp_fast(ath + y * rsqrt_fast(y));
    t = th >= 0.0 ? ri : -ri;
  }
  c = rsqrt_fast(fma(t, t, 1.0));
  s = t * c;
  rot = true;
}

__device__ __forceinline__ void rr_pair(int p, int step, int i, int& P, int& Q) {
  int a, b;
  if (i == 0) { a = p - 1; b = step; }
  else { a = (step + i) % (p - 1); b = (step - i + (p - 1)) % (p - 1); }
  P = min(a, b);
  Q = max(a, b);
}

__global__ void __launch_bounds__(kJW * 32) jacobi_kernel(const double* __restrict__ Hin, int p,
                                                          double* __restrict__ Wout, double* __restrict__ evals,
                                                          int* __restrict__ stats) {
  extern __shared__ double sm[];
  const int ld = p + 1;
  double* A = sm;
  double* V = sm + p * ld;
  __shared__ int rotated;
  __shared__ double dsh[kMaxP];
  __shared__ int rank_sh[kMaxP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int escale;
  if (warp == 0) {  // power-of-two scale 2^-e of the matrix (exact), so MUFU seeds stay in range
    double d = 0.0;
    for (int i = lane; i < p; i += 32) d = fmax(d, fabs(Hin[i * p + i]));
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xFFFFFFFFu, d, o));
    if (lane == 0) escale = (d > 0.0 && d < 1e300) ? ilogb(d) : 0;
  }
  __syncthreads();
  const int e = escale;
  for (int i = warp; i < p; i += kJW)
    for (int j = lane; j < p; j += 32) {
      A[i * ld + j] = ldexp(0.5 * (Hin[i * p + j] + Hin[j * p + i]), -e);
      V[i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int half = p / 2;
  int sweep = 0;
  for (; sweep < 30; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    int rot_any = 0;
    for (int step = 0; step < p - 1; ++step) {
      // ---- rows (J^T A) for the pairs owned by this warp
      double cs_c[4], cs_s[4];
      int pp[4], qq[4];
      // lane u computes the rotation of this warp's u-th pair (all in parallel)
      double myc = 1.0, mys = 0.0;
      {
        const int i = warp + kJW * lane;
        if (lane < 4 && i < half) {
          int P, Q;
          rr_pair(p, step, i, P, Q);
          bool rot;
          jacobi_rotation(A[P * ld + P], A[Q * ld + Q], A[P * ld + Q], myc, mys, rot);
          rot_any |= rot;
        }
      }
      int np = 0;
      for (int i = warp; i < half; i += kJW, ++np) {
        int P, Q;
        rr_pair(p, step, i, P, Q);
        const double c = __shfl_sync(0xFFFFFFFFu, myc, np);
        const double s = __shfl_sync(0xFFFFFFFFu, mys, np);
        cs_c[np] = c; cs_s[np] = s; pp[np] = P; qq[np] = Q;
        if (s != 0.0) {
          for (int col = lane; col < p; col += 32) {
            const double ap = A[P * ld + col], aq = A[Q * ld + col];
            A[P * ld + col] = c * ap - s * aq;
            A[Q * ld + col] = s * ap + c * aq;
          }
        }
      }
      __syncthreads();
      // ---- columns (A J, V J)
      for (int u = 0; u < np; ++u) {
        const double c = cs_c[u], s = cs_s[u];
        if (s == 0.0) continue;
        const int P = pp[u], Q = qq[u];
        for (int row = lane; row < p; row += 32) {
          const double ap = A[row * ld + P], aq = A[row * ld + Q];
          A[row * ld + P] = c * ap - s * aq;
          A[row * ld + Q] = s * ap + c * aq;
          const double vp = V[row * ld + P], vq = V[row * ld + Q];
          V[row * ld + P] = c * vp - s * vq;
          V[row * ld + Q] = s * vp + c * vq;
        }
      }
      __syncthreads();
    }
    if (rot_any) rotated = 1;
    __syncthreads();
    if (!rotated) break;
  }
  if (threadIdx.x < p) dsh[threadIdx.x] = A[threadIdx.x * ld + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < p) {
    int rk = 0;
    const double di = dsh[threadIdx.x];
    for (int j = 0; j < p; ++j) rk += (dsh[j] > di) || (dsh[j] == di && j < (int)threadIdx.x);
    rank_sh[threadIdx.x] = rk;
  }
  __syncthreads();
  for (int row = warp; row < p; row += kJW)
    for (int i = lane; i < p; i += 32) Wout[row * p + rank_sh[i]] = V[row * ld + i];
  if (threadIdx.x < p) evals[rank_sh[threadIdx.x]] = ldexp(dsh[threadIdx.x], e);
  if (threadIdx.x == 0 && stats) stats[0] = sweep + 1;
}

// ---------------------------------------------------------------- Cholesky-QR step
// B = H (p x p, symmetrised) = R^T R; Rinv = R^{-1} (upper).  Columns whose pivot is <= 1e-13 of
// the largest diagonal are flagged bad[c] = 1 and get a zero Rinv column.  16 warps, rows owned
// by warps and lanes over columns; every thread recomputes the pivot (no serial section).
__global__ void __launch_bounds__(kJW * 32) chol_inv_kernel(const double* __restrict__ Hin, int p,
                                                            double* __restrict__ Rinv, int* __restrict__ bad) {
  extern __shared__ double sm[];
  const int ld = p + 1;
  double* B = sm;           // becomes R (upper)
  double* X = sm + p * ld;  // Rinv
  __shared__ int badsh[kMaxP];
  __shared__ double dmax_sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = warp; i < p; i += kJW)
    for (int j = lane; j < p; j += 32) {
      B[i * ld + j] = 0.5 * (Hin[i * p + j] + Hin[j * p + i]);
      X[i * ld + j] = 0.0;
    }
  __syncthreads();
  if (warp == 0) {
    double d = 0.0;
    for (int i = lane; i < p; i += 32) d = fmax(d, B[i * ld + i]);
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xFFFFFFFFu, d, o));
    if (lane == 0) dmax_sh = d;
  }
  __syncthreads();
  // exact even power-of-two normalisation: B' = B 2^-e2, R = R' 2^(e2/2), Rinv = Rinv' 2^-(e2/2)
  const int e2 = (dmax_sh > 0.0 && dmax_sh < 1e300) ? 2 * (ilogb(dmax_sh) / 2) : 0;
  for (int i = warp; i < p; i += kJW)
    for (int j = lane; j < p; j += 32) B[i * ld + j] = ldexp(B[i * ld + j], -e2);
  __syncthreads();
  const double tol = 1e-13 * ldexp(dmax_sh, -e2);
  for (int j = 0; j < p; ++j) {
    const double d = B[j * ld + j];
    const bool ok = d > tol && d > 0.0;
    const double inv = ok ? rsqrt_fast(d) : 0.0;   // 1 / R_jj
    const double rjj = d * inv;
    // trailing update with the row of R computed on the fly: B[i][k] -= R[j][i] R[j][k]
    for (int i = j + 1 + warp; i < p; i += kJW) {
      const double rji = B[j * ld + i] * inv;
      for (int k = i + lane; k < p; k += 32) B[i * ld + k] -= rji * (B[j * ld + k] * inv);
    }
    __syncthreads();
    if (warp == 0) {
      for (int k = j + 1 + lane; k < p; k += 32) B[j * ld + k] *= inv;
      if (lane == 0) { B[j * ld + j] = rjj; badsh[j] = ok ? 0 : 1; }
    }
    __syncthreads();
  }
  // Rinv = R^{-1} from the bottom row up; X[i][.] accumulates sum_{k>i} R[i][k] Rinv[k][.]
  for (int j = p - 1; j >= 0; --j) {
    const bool okj = !badsh[j];
    const double inv = okj ? rcp_fast(B[j * ld + j]) : 0.0;
    if (warp == 0)
      for (int cc = lane; cc < p; cc += 32) X[j * ld + cc] = okj ? (((cc == j) ? 1.0 : 0.0) - X[j * ld + cc]) * inv : 0.0;
    __syncthreads();
    for (int i = warp; i < j; i += kJW) {
      const double rij = B[i * ld + j];
      for (int cc = j + lane; cc < p; cc += 32) X[i * ld + cc] = fma(rij, X[j * ld + cc], X[i * ld + cc]);
    }
    __syncthreads();
  }
  for (int i = warp; i < p; i += kJW)
    for (int cc = lane; cc < p; cc += 32) Rinv[i * p + cc] = ldexp(X[i * ld + cc], -e2 / 2);
  for (int cc = threadIdx.x; cc < p; cc += blockDim.x) bad[cc] = badsh[cc];
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

// Y = G In (split-K partials summed in a fixed order)
avd_status gemm_g(Ctx* c, const double* In, double* Out) {
  const int64_t m = c->cfg.m;
  const int ks = c->gemm_ks;
  const int64_t kchunk = round_up(ceil_div(m, ks), kGK);
  dim3 grid((unsigned)ceil_div(m, kGM), (unsigned)ks);
  switch (c->p / 16) {
#define CASE(PC)                                                                                          \
  case PC: {                                                                                              \
    const int sm = 2 * (kGK * (kGM + 2) + kGK * PC * 16) * (int)sizeof(double);                           \
    AVD_CUDA(cudaFuncSetAttribute(gemm_gq_kernel<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));  \
    gemm_gq_kernel<PC><<<grid, 128, sm, c->stream>>>(c->G, In, m, kchunk, c->Ypart);                      \
    break;                                                                                                \
  }
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  const int64_t n = m * c->p;
  ksum_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c->stream>>>(c->Ypart, ks, n, Out);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// H = A^T B (m-length reduction): per-CTA partials, then a multi-CTA fixed-order sum into c->H
avd_status atb(Ctx* c, const double* A, const double* B) {
  const int64_t m = c->cfg.m;
  const int p = c->p;
  const size_t sm = 2 * kRedChunk * p * sizeof(double);
  switch (p / 16) {
#define CASE(PC)                                                                                      \
  case PC:                                                                                            \
    AVD_CUDA(cudaFuncSetAttribute(atb_partial_kernel<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    atb_partial_kernel<PC><<<c->n_red, 256, sm, c->stream>>>(A, B, m, c->red_part);                   \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  psum_kernel<<<(unsigned)ceil_div(p * p, 128), 128, 0, c->stream>>>(c->red_part, c->n_red, p * p, c->H);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status matpp(Ctx* c, const double* In0, double* Out0, const double* In1, double* Out1, const double* M) {
  const int p = c->p;
  const size_t sm = ((size_t)p * p + 16 * p) * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(matpp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  matpp_kernel<<<(unsigned)ceil_div(c->cfg.m, 16), 256, sm, c->stream>>>(In0, Out0, In1, Out1, M, c->cfg.m, p);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// Q <- orth(Y) by Cholesky-QR2; rank-deficient columns are re-drawn at random between passes.
avd_status orth(Ctx* c, const double* Y, double* Q, uint32_t seed) {
  int* bad = reinterpret_cast<int*>(c->resid + c->p);
  const int p = c->p;
  const size_t sm = 2 * (size_t)p * (p + 1) * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  for (int pass = 0; pass < 2; ++pass) {
    const double* src = pass == 0 ? Y : Q;
    AVD_TRY(atb(c, src, src));
    chol_inv_kernel<<<1, kJW * 32, sm, c->stream>>>(c->H, p, c->W, bad);
    AVD_LAUNCHED(c);
    AVD_TRY(matpp(c, src, Q, nullptr, nullptr, c->W));
    if (pass == 0) {
      rand_fill_kernel<<<(unsigned)ceil_div(c->cfg.m * p, 256), 256, 0, c->stream>>>(Q, c->cfg.m, p, seed, bad);
      AVD_LAUNCHED(c);
    }
  }
  return AVD_OK;
}

}  // namespace

// Subspace iteration: every iteration applies G^2 (two GEMMs) and re-orthonormalises; a
// Rayleigh-Ritz check runs on a schedule predicted from the observed residual decay (at most
// every 4 iterations, always on the last one), so the p x p Jacobi runs ~3-4 times per solve.
avd_status run_eig(Ctx* c) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  const uint32_t seed = (uint32_t)(c->cfg.seed ^ (c->cfg.seed >> 32)) * 2654435761u + 12345u;
  int* jstats = reinterpret_cast<int*>(c->theta + p);  // [16] sweeps per RR solve
  AVD_CUDA(cudaMemsetAsync(jstats, 0, 16 * sizeof(int), c->stream));
  const size_t jsm = 2 * (size_t)p * (p + 1) * sizeof(double);
  AVD_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jsm));
  rand_fill_kernel<<<(unsigned)ceil_div(m * p, 256), 256, 0, c->stream>>>(c->Z, m, p, seed, nullptr);
  AVD_LAUNCHED(c);
  AVD_TRY(orth(c, c->Z, c->Q, seed + 1));
  const int max_it = c->cfg.max_iters > 0 ? c->cfg.max_iters : 100;
  const double tol = c->cfg.eig_tol > 0 ? c->cfg.eig_tol : 1e-6;  // V angle <~ tol * lambda_1 / gap_k
  int it = 0, next_rr = 2, prev_it = 0, rr_count = 0;
  double maxres = 0.0, prev_res = -1.0;
  bool conv = false;
  for (it = 1; it <= max_it; ++it) {
    AVD_TRY(gemm_g(c, c->Q, c->Y));                         // Y = G Q
    if (it == next_rr || it == max_it) {
      ++rr_count;
      AVD_TRY(atb(c, c->Q, c->Y));                          // H = Q^T Y
      jacobi_kernel<<<1, kJW * 32, jsm, c->stream>>>(c->H, p, c->W, c->theta, jstats + std::min(rr_count - 1, 15));
      AVD_LAUNCHED(c);
      AVD_TRY(matpp(c, c->Y, c->Z, c->Q, c->U, c->W));      // Z = Y W, U = Q W (Ritz vectors)
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
      // predicted residual decay per G^2 step: observed, else (theta_p / theta_k)^2
      double rate = -1.0;
      if (prev_res > 0.0 && maxres < prev_res) rate = std::pow(maxres / prev_res, 1.0 / (double)(it - prev_it));
      else if (c->eig_host[k - 1] > 0.0) rate = std::pow(std::max(c->eig_host[p - 1], 0.0) / c->eig_host[k - 1], 2.0);
      int step = 1;
      if (rate > 0.0 && rate < 0.95) {
        const double need = std::log(tol / maxres) / std::log(rate);
        step = (int)std::max(1.0, std::min(8.0, std::floor(need)));
      }
      prev_res = maxres;
      prev_it = it;
      next_rr = it + step;
      AVD_TRY(gemm_g(c, c->Z, c->Y));                       // Y = G Z = G^2 U
    } else {
      AVD_TRY(gemm_g(c, c->Y, c->Z));                       // Z = G Y = G^2 Q
      std::swap(c->Y, c->Z);
    }
    AVD_TRY(orth(c, c->Y, c->Q, seed + 7919u * (uint32_t)it));
  }
  c->iters = std::min(it, max_it);
  c->rr_count = rr_count;
  c->max_resid = maxres;
  c->sigma_next = (k < p) ? std::sqrt(std::max(c->eig_host[k], 0.0)) : 0.0;
  int sw[16];
  AVD_CUDA(cudaMemcpyAsync(sw, jstats, sizeof(sw), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  c->jacobi_sweeps = 0;
  for (int q = 0; q < std::min(rr_count, 16); ++q) c->jacobi_sweeps += sw[q];  // total over all RR solves
  AVD_CUDA(cudaMemsetAsync(c->V32, 0, sizeof(float) * m * c->k_pad, c->stream));
  finalize_vectors_kernel<<<k, 256, 0, c->stream>>>(c->U, c->theta, m, p, k, c->k_pad, c->V, c->sigma, c->V32);
  AVD_LAUNCHED(c);
  return conv ? AVD_OK : AVD_ENOCONV;
}

}  // namespace avd
