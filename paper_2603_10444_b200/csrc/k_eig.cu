// k_eig.cu — K4: top-k eigenpairs of the centred Gram G (on device) by block subspace iteration
// with Rayleigh-Ritz: V_k, sigma_k = sqrt(lambda_k) are the right singular vectors / values of
// Xc that define the rank-k spike.
//
//   Q_0 = orth(random m x p), p = roundup16(k + 8)
//   power step:  Q <- orth(G (G Q))                    G in fp32 (L2-resident copy), fp32 FMA
//   RR check:    Y = G Q (fp64) ; H = Q^T Y ; (W, theta) = eig(H)           (Rayleigh-Ritz)
//                U = Q W ; Z = Y W (= G U) ; res_r = ||Z_r - theta_r U_r|| / theta_1, r < k
//                stop when max res_r <= tol, else Q <- orth(G Z)
// The power steps only steer the subspace; every reported quantity (theta, U, the residual
// that decides convergence) comes from the fp64 product with the exact G, so the fp32 operator
// perturbs nothing that is returned (its ~1e-8 relative error sits far below tol).
//
// Kernels: Y = G Q is a stream-K SIMT GEMM (fp32 or fp64; every CTA gets the same number of
// 32-row K units, partial row-block segments are summed by a fixup kernel in a fixed order);
// the m-length p x p reductions (Q^T Y, Y^T Y) are per-CTA partials whose LAST CTA (atomic
// ticket) sums them in a fixed order and then runs the p x p step in place: Cholesky + triangular
// inverse for CholQR, or the parallel Jacobi eigensolver for Rayleigh-Ritz.
// Rank deficiency (G = 0, rank(G) < p, m < p) flags the failing columns, which are re-drawn at
// random and re-orthonormalised (R11).  Deterministic: no floating-point atomics.
#include <cfloat>
#include "common.cuh"

namespace avd {

#ifdef AVD_EIG_PROBE
__device__ long long g_probe_clk[16];  // tools/eig_micro.cu: phase timestamps of one-CTA kernels
#define PROBE(i) do { if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) g_probe_clk[i] = clock64(); } while (0)
#else
#define PROBE(i) do { } while (0)
#endif

namespace {

// ---------------------------------------------------------------- G_int -> G (fp64), G32 (fp32)
// Both with leading dimension m_pad; rows/columns >= m are zero.
// 32 x 32 tiles, 32 x 8 threads.  K3 adds tile (A, B), A <= B (128-blocks), transposed: element
// (a, b) of an upper tile sits at Gi[b][a]; those tiles are read row-wise (coalesced) and
// transposed through shared memory, so every global access is coalesced.
__global__ void __launch_bounds__(256) gram_finalize_kernel(const long long* __restrict__ Gi, int64_t m, int64_t m_pad,
                                     const int32_t* __restrict__ shift, const long long* __restrict__ qsum,
                                     const double* __restrict__ ysq, const double* __restrict__ mu,
                                     const float* __restrict__ mu0, double l, double inv_l, double unit,
                                     double* __restrict__ G, float* __restrict__ G32) {
  __shared__ long long tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t a0 = (int64_t)blockIdx.y * 32, b0 = (int64_t)blockIdx.x * 32;
  const bool upper = (a0 / 128) <= (b0 / 128);  // uniform over the 32 x 32 tile
  if (upper) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int bb = ty + 8 * r;
      tile[bb][tx] = (b0 + bb < m && a0 + tx < m) ? Gi[(b0 + bb) * m_pad + a0 + tx] : 0ll;
    }
    __syncthreads();
  }
  const int64_t b = b0 + tx;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int aa = ty + 8 * r;
    const int64_t a = a0 + aa;
    double g = 0.0;
    if (a < m && b < m) {
      const long long v = upper ? tile[tx][aa] : Gi[a * m_pad + b];
      // exact centring of the quantised matrix: sum_i (q_ia - qbar_a)(q_ib - qbar_b)
      //   = sum_i q_ia q_ib - S_a S_b / l   (S = column sums of q, exact integers)
      // v unit = sum_i q_ia q_ib.  The diagonal is the centred energy itself, from the fp64
      // sums of the fused pass: sum_i (x_ia - mu_a)^2 = sum_i (x_ia - mu0_a)^2 - l (mu_a - mu0_a)^2
      // (no dither noise, no cancellation: mu0 is the sampled centre)
      if (a == b) {
        const double dm = mu[a] - (double)mu0[a];
        g = ysq[a] - l * dm * dm;
      } else {
        const double corr = ((double)qsum[a] * (double)qsum[b]) * inv_l;
        g = ldexp((double)v * unit - corr, -(shift[a] + shift[b]));
      }
    }
    G[a * m_pad + b] = g;
    G32[a * m_pad + b] = (float)g;
  }
}

// tr(G), max_a G_aa (= max |G_ab| for the positive semidefinite G), and
// ||X||_F^2 = sum_a [sum_i (x_ia - mu0_a)^2 + 2 mu0_a sum_i x_ia - l mu0_a^2] -> stats[m] (every
// term is a nonnegative-dominated fp64 sum; PAPER.md:15 total energy)
__global__ void __launch_bounds__(1024) trace_kernel(const double* __restrict__ G, int64_t m, int64_t ld,
                                                    const double* __restrict__ ysq, const float* __restrict__ mu0,
                                                    double l, double* __restrict__ stats, double* __restrict__ out,
                                                    double* __restrict__ gmax) {
  // fixed order: strided per-thread sums, xor-shuffle tree per warp, warp partials in order
  __shared__ double sh[32], shm[32], shd[32];
  double s = 0.0, mx = 0.0, dg = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 1024) {
    const double g = G[j * ld + j];
    s += g;
    mx = fmax(mx, fabs(g));
    const double c0 = (double)mu0[j];
    dg += ysq[j] + c0 * (2.0 * stats[j] - l * c0);
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    dg += __shfl_xor_sync(0xFFFFFFFFu, dg, o);
  }
  if ((threadIdx.x & 31) == 0) { sh[threadIdx.x >> 5] = s; shm[threadIdx.x >> 5] = mx; shd[threadIdx.x >> 5] = dg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, u = 0.0, d = 0.0;
    for (int i = 0; i < 32; ++i) { t += sh[i]; u = fmax(u, shm[i]); d += shd[i]; }
    out[0] = t;
    stats[m] = d;
    *gmax = u;
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

// Q[j][c] = U(-1,1) for columns with flag (or all when flags == nullptr); Q32 mirrors it
__global__ void rand_fill_kernel(double* __restrict__ Q, float* __restrict__ Q32, int64_t m, int p, uint32_t seed,
                                 const int* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * p) return;
  const int c = (int)(t % p);
  if (flags && !flags[c]) return;
  const double v = rnd_sym(seed, (uint32_t)(t / p), (uint32_t)c);
  Q[t] = v;
  if (Q32) Q32[t] = (float)v;
}

// ---------------------------------------------------------------- Y = G Q, split-K
// Unit = (row block rb of BM rows, K range ks of the KS equal slices of the 32-row K tiles):
// CTA rb * KS + ks computes the BM x p partial product of its K range (fp32 or fp64 FMA in
// registers) and stores it to part[rb][ks]; the LAST CTA of a row block (acq_rel ticket) sums
// the KS partials in ks order in fp64 and writes Y (fp64) and its optional fp32 mirror — one
// kernel, no atomics on data, bit-deterministic.  G is symmetric, so the (rows r0.., K k0..)
// tile is read as G[k][r0..] (contiguous rows, no transpose).
// 128 threads: ty = tid / 8 owns rows ty*NR .. +NR, tx = tid % 8 owns column pairs 16 c2 + 2 tx.
constexpr int kSkBK = 32;
constexpr int kSkThreads = 128;
constexpr int kSkStages = 3;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ticket += 1 with acq_rel semantics at GPU scope (no full sequentially-consistent fence)
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* t) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
  return old;
}

template <typename T, int NR, int NC>
__global__ void __launch_bounds__(kSkThreads) gemm_kernel(const T* __restrict__ G, int64_t ldg,
                                                          const T* __restrict__ Qin, int64_t m, int KT, int KS,
                                                          T* __restrict__ part, unsigned* __restrict__ tickets,
                                                          double* __restrict__ Y, float* __restrict__ Y32) {
  constexpr int BM = 16 * NR;
  constexpr int p = 8 * NC;
  constexpr int SG = kSkBK * BM;          // elements of one G stage
  constexpr int SQ = kSkBK * p;           // elements of one Q stage
  constexpr int EPC = 16 / sizeof(T);     // elements per 16-B chunk
  extern __shared__ __align__(16) unsigned char sk_raw[];
  __shared__ unsigned last_sh;
  T* sm = reinterpret_cast<T*>(sk_raw);
  const int tid = threadIdx.x;
  const int ty = tid >> 3, tx = tid & 7;
  const int rb = blockIdx.x / KS, ks = blockIdx.x % KS;
  const int kt0 = (int)(((int64_t)KT * ks) / KS), kt1 = (int)(((int64_t)KT * (ks + 1)) / KS);
  const int n = kt1 - kt0;

  auto load_stage = [&](int slot, int kt) {
    T* sG = sm + slot * (SG + SQ);
    T* sQ = sG + SG;
    const int64_t k0 = (int64_t)kt * kSkBK;
    const int64_t r0 = (int64_t)rb * BM;
    constexpr int GCH = SG / EPC;  // 16-B chunks of the G tile
    for (int ch = tid; ch < GCH; ch += kSkThreads) {
      const int kk = ch / (BM / EPC), cc = ch % (BM / EPC);
      const bool ok = k0 + kk < m;
      const T* src = ok ? G + (k0 + kk) * ldg + r0 + cc * EPC : G;
      cp_async16((uint32_t)__cvta_generic_to_shared(sG + kk * BM + cc * EPC), src, ok);
    }
    constexpr int QCH = SQ / EPC;
    for (int ch = tid; ch < QCH; ch += kSkThreads) {
      const int kk = ch / (p / EPC);
      const bool ok = k0 + kk < m;
      const T* src = ok ? Qin + k0 * p + ch * EPC : Qin;
      cp_async16((uint32_t)__cvta_generic_to_shared(sQ + ch * EPC), src, ok);
    }
  };

  T acc[NR][NC];
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[r][q] = T(0);
#pragma unroll
  for (int s = 0; s < kSkStages - 1; ++s) {
    if (s < n) load_stage(s, kt0 + s);
    cp_commit();
  }
  for (int i = 0; i < n; ++i) {
    cp_wait<kSkStages - 2>();
    __syncthreads();
    if (i + kSkStages - 1 < n) load_stage((i + kSkStages - 1) % kSkStages, kt0 + i + kSkStages - 1);
    cp_commit();
    const T* sG = sm + (i % kSkStages) * (SG + SQ);
    const T* sQ = sG + SG;
#pragma unroll 4
    for (int kk = 0; kk < kSkBK; ++kk) {
      T g[NR], q[NC];
#pragma unroll
      for (int r = 0; r < NR; r += EPC) {
        if constexpr (sizeof(T) == 4) {
          const float4 v = *reinterpret_cast<const float4*>(sG + kk * BM + ty * NR + r);
          g[r] = v.x; g[r + 1] = v.y; g[r + 2] = v.z; g[r + 3] = v.w;
        } else {
          const double2 v = *reinterpret_cast<const double2*>(sG + kk * BM + ty * NR + r);
          g[r] = v.x; g[r + 1] = v.y;
        }
      }
#pragma unroll
      for (int c2 = 0; c2 < NC / 2; ++c2) {
        if constexpr (sizeof(T) == 4) {
          const float2 v = *reinterpret_cast<const float2*>(sQ + kk * p + 16 * c2 + 2 * tx);
          q[2 * c2] = v.x; q[2 * c2 + 1] = v.y;
        } else {
          const double2 v = *reinterpret_cast<const double2*>(sQ + kk * p + 16 * c2 + 2 * tx);
          q[2 * c2] = v.x; q[2 * c2 + 1] = v.y;
        }
      }
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int q2 = 0; q2 < NC; ++q2) acc[r][q2] = fma(g[r], q[q2], acc[r][q2]);
    }
  }
  cp_wait<0>();
  // partial product of this K slice -> part[rb][ks] (BM x p, row-major)
  T* pp = part + ((int64_t)rb * KS + ks) * (BM * p);
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int c2 = 0; c2 < NC / 2; ++c2) {
      T* d = pp + (ty * NR + r) * p + 16 * c2 + 2 * tx;
      if constexpr (sizeof(T) == 4) *reinterpret_cast<float2*>(d) = make_float2(acc[r][2 * c2], acc[r][2 * c2 + 1]);
      else *reinterpret_cast<double2*>(d) = make_double2(acc[r][2 * c2], acc[r][2 * c2 + 1]);
    }
  __syncthreads();
  if (tid == 0) last_sh = (ticket_acq_rel(&tickets[rb]) == (unsigned)(KS - 1)) ? 1u : 0u;
  __syncthreads();
  if (!last_sh) return;
  // the row block's last CTA: fixed-order sum of the KS partials
  const T* base = part + (int64_t)rb * KS * (BM * p);
  for (int e = tid * 2; e < BM * p; e += kSkThreads * 2) {
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < KS; ++q) {
      const T* src = base + (int64_t)q * (BM * p) + e;
      if constexpr (sizeof(T) == 4) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(src));
        s0 += (double)v.x; s1 += (double)v.y;
      } else {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src));
        s0 += v.x; s1 += v.y;
      }
    }
    const int64_t row = (int64_t)rb * BM + e / p;
    if (row < m) {
      const int64_t o = row * p + e % p;
      *reinterpret_cast<double2*>(Y + o) = make_double2(s0, s1);
      if (Y32) *reinterpret_cast<float2*>(Y32 + o) = make_float2((float)s0, (float)s1);
    }
  }
  if (tid == 0) tickets[rb] = 0u;  // re-armed for the next launch (stream-ordered)
}

// ---------------------------------------------------------------- p x p helpers (one CTA)
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
// Jacobi rotation (c, s) for the pair (p, q) of a symmetric matrix scaled to ~1.  The angle is
// computed in fp32 (Rutishauser: th = (a_qq - a_pp) / (2 a_pq), t = sign(th) / (|th| + sqrt(th^2+1)))
// — the rotation only has to shrink a_pq, which a 2^-24-accurate angle does by ~1e-7 per visit —
// while (c, s) are made orthogonal to fp64 accuracy: c^2 + s^2 = 1 + d from the fp32 pair, scaled by
// (1 + d)^(-1/2) = 1 - d/2 + 3d^2/8 (|d| <~ 1e-7), so every applied transform is an exact-in-fp64
// similarity and the eigenvalues keep fp64 accuracy.  Skipped when |a_pq| <= 1e-9 sqrt(a_pp a_qq).
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double& c, double& s, bool& rot) {
  c = 1.0;
  s = 0.0;
  rot = false;
  // |a_pq| <= 1e-9 sqrt(a_pp a_qq): eigenvalue error ~1e-18 relative, eigenvector error ~1e-9 / gap
  if (!(apq * apq > 1e-18 * fabs(app * aqq)) || fabs(apq) < 1e-30 || fabs(apq) > 1e30) return;
  const float th = __fdividef(0.5f * (float)(aqq - app), (float)apq);
  const float ath = fabsf(th);
  if (!(ath < 1e18f)) return;  // |a_pq| below 1e-18 |a_qq - a_pp|: nothing left to rotate
  float t = __frcp_rn(ath + sqrtf(fmaf(th, th, 1.0f)));
  t = th >= 0.f ? t : -t;
  const float c32 = rsqrtf(fmaf(t, t, 1.0f));
  const double c0 = (double)c32, s0 = (double)(t * c32);
  const double d = fma(c0, c0, s0 * s0) - 1.0;
  const double r = fma(d, fma(0.375, d, -0.5), 1.0);
  c = c0 * r;
  s = s0 * r;
  rot = true;
}
__device__ __forceinline__ void rr_pair(int p, int step, int i, int& P, int& Q) {
  int a, b;
  if (i == 0) { a = p - 1; b = step; }
  else { a = (step + i) % (p - 1); b = (step - i + (p - 1)) % (p - 1); }
  P = min(a, b);
  Q = max(a, b);
}

// Parallel (round-robin) Jacobi on the symmetric A (P x P, ld LDA, scaled so max|a_ii| ~ 1) with
// V^T (ld P).  Per step: warp u computes the rotation J_u of its pair (P_u, Q_u) (lane 0), then,
// after one barrier, rewrites ITS two rows of A as rows of J_u^T A J (lane w takes the column
// pair (P_w, Q_w) of the step, so each 2x2 block sees both rotations) and its two rows of
// V^T (V <- V J).  Every row belongs to exactly one pair: no two warps touch the same element.
// Two barriers per step.  Returns the number of sweeps.
template <int P, int LDA>
__device__ int jacobi_block(double* A, double* Vt, double* rc, double* rs, int* rp, int* rq, int* flag, int max_sweeps) {
  constexpr int half = P / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    for (int step = 0; step < P - 1; ++step) {
      __syncthreads();
#ifdef AVD_EIG_PROBE
      long long t_a = clock64();
#endif
      if (warp == 0) {
        bool any = false;
        for (int u = lane; u < half; u += 32) {  // all rotations of the step, one lane each
          int p0, q0;
          rr_pair(P, step, u, p0, q0);
          double c, s;
          bool rot;
          jacobi_rotation(A[p0 * LDA + p0], A[q0 * LDA + q0], A[p0 * LDA + q0], c, s, rot);
          rc[u] = c;
          rs[u] = s;
          rp[u] = p0;
          rq[u] = q0;
          any |= rot;
        }
        if (__any_sync(0xFFFFFFFFu, any) && lane == 0) *flag = 1;
      }
#ifdef AVD_EIG_PROBE
      long long t_b = clock64();
#endif
      __syncthreads();
#ifdef AVD_EIG_PROBE
      long long t_c = clock64();
      if (threadIdx.x == 0) { g_probe_clk[8] += t_b - t_a; g_probe_clk[9] += t_c - t_b; }
#endif
      for (int u = warp; u < half; u += nwarps) {
        const double cu = rc[u], su = rs[u];
        const int p1 = rp[u], q1 = rq[u];
        for (int w = lane; w < half; w += 32) {
          const double cw = rc[w], sw = rs[w];
          if (su == 0.0 && sw == 0.0) continue;
          const int p2 = rp[w], q2 = rq[w];
          const double a = A[p1 * LDA + p2], b = A[p1 * LDA + q2], c_ = A[q1 * LDA + p2], d = A[q1 * LDA + q2];
          // rows: J_u^T, then columns: J_w
          const double a1 = cu * a - su * c_, b1 = cu * b - su * d;
          const double c1 = su * a + cu * c_, d1 = su * b + cu * d;
          const double a2 = cw * a1 - sw * b1, b2 = sw * a1 + cw * b1;
          const double c2 = cw * c1 - sw * d1, d2 = sw * c1 + cw * d1;
          A[p1 * LDA + p2] = a2;
          A[p1 * LDA + q2] = b2;
          A[q1 * LDA + p2] = c2;
          A[q1 * LDA + q2] = d2;
        }
        if (su != 0.0) {
          // V <- V J_u: rows p1, q1 of V^T, two columns per lane
          for (int j = 2 * lane; j < P; j += 64) {
            double2* vp = reinterpret_cast<double2*>(Vt + p1 * P + j);
            double2* vq = reinterpret_cast<double2*>(Vt + q1 * P + j);
            const double2 x = *vp, y = *vq;
            *vp = make_double2(cu * x.x - su * y.x, cu * x.y - su * y.y);
            *vq = make_double2(su * x.x + cu * y.x, su * x.y + cu * y.y);
          }
        }
      }
    }
    __syncthreads();
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  return sweep + 1;
}

// Cholesky B = R^T R (upper; B scaled so max diag ~ 1).  Each thread keeps its entries of the
// upper triangle in registers for the whole factorisation; at step j the owners of row j
// publish it (double-buffered row), one barrier, and every owner of an entry (i, k), i > j,
// applies b_ik -= b_ji b_jk / b_jj.  Outputs R into B (upper, zero below), dinv[j] = 1 / R_jj and
// bad[j] = 1 for pivots <= 1e-13 of the largest diagonal (zero row).
template <int P, int LDA, int NT>
__device__ void chol_block(double* B, double* dinv, int* bad) {
  constexpr int NU = P * (P + 1) / 2;
  constexpr int E = (NU + NT - 1) / NT;
  __shared__ double rowbuf[2][P];
  __shared__ double dmax_sh;
  int ei[E], ek[E];
  double v[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int e = threadIdx.x + NT * q;
    ei[q] = P;  // none
    ek[q] = P;
    v[q] = 0.0;
    if (e < NU) {
      // packed upper triangle, row-major: row i holds P - i entries
      int i = 0, rem = e;
      while (rem >= P - i) { rem -= P - i; ++i; }
      ei[q] = i;
      ek[q] = i + rem;
      v[q] = B[i * LDA + i + rem];
    }
  }
  if (threadIdx.x < 32) {
    double d = 0.0;
    for (int i = threadIdx.x; i < P; i += 32) d = fmax(d, B[i * LDA + i]);
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xFFFFFFFFu, d, o));
    if (threadIdx.x == 0) dmax_sh = d;
  }
  __syncthreads();
  const double tol = 1e-13 * dmax_sh;
  for (int j = 0; j < P; ++j) {
    double* row = rowbuf[j & 1];
#pragma unroll
    for (int q = 0; q < E; ++q)
      if (ei[q] == j) row[ek[q]] = v[q];
    __syncthreads();
    const double d = row[j];
    const bool ok = d > tol && d > 0.0;
    const double inv = ok ? rsqrt_fast(d) : 0.0;
    const double invd = inv * inv;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if (ei[q] > j && ei[q] < P) v[q] = fma(-row[ei[q]] * invd, row[ek[q]], v[q]);
      else if (ei[q] == j) v[q] = (ek[q] == j) ? (ok ? d * inv : 0.0) : v[q] * inv;  // R row j (final)
    }
    if (threadIdx.x == 0) { dinv[j] = inv; bad[j] = ok ? 0 : 1; }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < P * P; t += NT) B[(t / P) * LDA + t % P] = 0.0;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (ei[q] < P) B[ei[q] * LDA + ek[q]] = v[q];
  __syncthreads();
}

// ---------------------------------------------------------------- fused m-length reduction
constexpr int kRedRows = kRedRowsC;  // rows per partial
template <int PC>
struct RedCfg {
  static constexpr int threads = PC <= 4 ? 1024 : 512;  // register budget of the PC^2 accumulators
  static constexpr int chunk = PC <= 3 ? kRedRows : 64;  // rows staged in smem at a time (one load wave)
};
// part[blk] = A[rows of blk]^T B[rows of blk] (p x p), register-tiled over the first 256 threads
// (thread (ti, tj) owns outputs (ti + 16a, tj + 16b)); the last CTA to finish sums the partials
// in block order (symmetrised) and then:
//   MODE 0: H = the sum (out0)
//   MODE 1: Cholesky -> R (out0, upper, p x p), 1/R_jj (out1), bad flags (ibad); stats[0] = 1 when
//           a second CholQR pass is needed (a bad column, or cond(R)^2 > 1e6 from its diagonal)
//   MODE 2: Jacobi -> W (out0, eigenvectors sorted by eigenvalue desc), theta (out1), sweeps
// gate != nullptr && *gate == 0: nothing to do (second CholQR pass not needed).
// The partial sum reads each partial once (two adjacent elements per load) and symmetrises in smem.
template <int MODE, int PC>
__global__ void __launch_bounds__(RedCfg<PC>::threads) atb_fused_kernel(
    const double* __restrict__ A, const double* __restrict__ B, int64_t m, double* __restrict__ part,
    unsigned* __restrict__ ticket, double* __restrict__ out0, double* __restrict__ out1, int* __restrict__ ibad,
    int* __restrict__ stats, const int* __restrict__ gate, int max_sweeps) {
  constexpr int p = PC * 16;
  constexpr int NT = RedCfg<PC>::threads;
  constexpr int kRedChunk = RedCfg<PC>::chunk;
  if (gate && *gate == 0) return;
  extern __shared__ __align__(16) double fsm[];
  __shared__ unsigned last_sh;
  PROBE(0);
  {
    double* sA = fsm;
    double* sB = fsm + kRedChunk * p;
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    const bool comp = threadIdx.x < 256;
    double acc[PC][PC];
#pragma unroll
    for (int a = 0; a < PC; ++a)
#pragma unroll
      for (int b = 0; b < PC; ++b) acc[a][b] = 0.0;
    const int64_t rbase = (int64_t)blockIdx.x * kRedRows;
    for (int ch = 0; ch < kRedRows / kRedChunk; ++ch) {
      const int64_t r0 = rbase + ch * kRedChunk;
      if (r0 >= m) break;
      __syncthreads();
      for (int t = threadIdx.x; t < kRedChunk * p / 2; t += NT) {
        const int rr = (2 * t) / p;
        const bool ok = r0 + rr < m;
        const double2 va = ok ? reinterpret_cast<const double2*>(A + r0 * p)[t] : make_double2(0.0, 0.0);
        const double2 vb = ok ? reinterpret_cast<const double2*>(B + r0 * p)[t] : make_double2(0.0, 0.0);
        reinterpret_cast<double2*>(sA)[t] = va;
        reinterpret_cast<double2*>(sB)[t] = vb;
      }
      __syncthreads();
      if (comp) {
#pragma unroll 4
        for (int rr = 0; rr < kRedChunk; ++rr) {
          double av[PC], bv[PC];
#pragma unroll
          for (int a = 0; a < PC; ++a) av[a] = sA[rr * p + ti + 16 * a];
#pragma unroll
          for (int b = 0; b < PC; ++b) bv[b] = sB[rr * p + tj + 16 * b];
#pragma unroll
          for (int a = 0; a < PC; ++a)
#pragma unroll
            for (int b = 0; b < PC; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
      }
    }
    if (comp) {
      double* dst = part + (int64_t)blockIdx.x * p * p;
#pragma unroll
      for (int a = 0; a < PC; ++a)
#pragma unroll
        for (int b = 0; b < PC; ++b) dst[(ti + 16 * a) * p + tj + 16 * b] = acc[a][b];
    }
  }
  // CTA's partial stores -> barrier -> one acq_rel ticket (release of the CTA's stores, acquire
  // of every other CTA's for the last one) -> barrier
  PROBE(1);
  __syncthreads();
  if (threadIdx.x == 0) last_sh = (ticket_acq_rel(ticket) == gridDim.x - 1) ? 1u : 0u;
  __syncthreads();
  if (!last_sh) return;
  PROBE(2);
  const int nparts = gridDim.x;
  constexpr int ld = p + 1;
  double* S = fsm;            // p x ld
  double* X = fsm + p * ld;   // p x p (V^T for MODE 2)
  __shared__ double aux[p];
  __shared__ double rcs[2][p / 2];
  __shared__ int rpq[2][p / 2];
  __shared__ int flag_sh, badsh[p], rank_sh[p], escale;
  // fixed-order sum of the partials: thread t owns the element pair (2t, 2t+1), all loads of a
  // batch of 8 partials in flight at once
  for (int t = threadIdx.x; t < p * p / 2; t += NT) {
    double2 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = make_double2(0.0, 0.0);
    int q = 0;
    for (; q + 8 <= nparts; q += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(reinterpret_cast<const double2*>(part + (int64_t)(q + u) * p * p) + t);
#pragma unroll
      for (int u = 0; u < 8; ++u) { a[u].x += v[u].x; a[u].y += v[u].y; }
    }
    for (; q < nparts; ++q) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(part + (int64_t)q * p * p) + t);
      a[0].x += v.x;
      a[0].y += v.y;
    }
    const double vx = ((a[0].x + a[1].x) + (a[2].x + a[3].x)) + ((a[4].x + a[5].x) + (a[6].x + a[7].x));
    const double vy = ((a[0].y + a[1].y) + (a[2].y + a[3].y)) + ((a[4].y + a[5].y) + (a[6].y + a[7].y));
    const int e0 = 2 * t;
    X[e0] = vx;  // staging (X is free until the solve)
    X[e0 + 1] = vy;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < p * p; t += NT) {
    const int i = t / p, j = t % p;
    S[i * ld + j] = 0.5 * (X[i * p + j] + X[j * p + i]);
  }
  if (threadIdx.x == 0) *ticket = 0u;  // re-arm for the next launch (stream-ordered)
  __syncthreads();
  PROBE(3);
  if (MODE == 0) {
    for (int t = threadIdx.x; t < p * p; t += NT) out0[t] = S[(t / p) * ld + t % p];
    return;
  }
  // exact power-of-two normalisation (keeps MUFU seeds in range): S' = S 2^-e
  if (threadIdx.x < 32) {
    double d = 0.0;
    for (int i = threadIdx.x; i < p; i += 32) d = fmax(d, fabs(S[i * ld + i]));
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xFFFFFFFFu, d, o));
    if (threadIdx.x == 0) {
      int e = (d > 0.0 && d < 1e300) ? ilogb(d) : 0;
      if (MODE == 1) e = 2 * (e / 2);  // even, so R scales by 2^(e/2)
      escale = e;
    }
  }
  __syncthreads();
  const int e = escale;
  const double sc = ldexp(1.0, -e);
  for (int t = threadIdx.x; t < p * p; t += NT) S[(t / p) * ld + t % p] *= sc;
  __syncthreads();
  if (MODE == 1) {
    PROBE(4);
    chol_block<p, ld, NT>(S, aux, badsh);
    PROBE(5);
    const double rs = ldexp(1.0, e / 2), ri = ldexp(1.0, -e / 2);
    for (int t = threadIdx.x; t < p * p; t += NT) out0[t] = S[(t / p) * ld + t % p] * rs;
    for (int t = threadIdx.x; t < p; t += NT) {
      out1[t] = aux[t] * ri;
      ibad[t] = badsh[t];
    }
    if (stats && threadIdx.x < 32) {
      double lo = 1e300, hi = 0.0;
      int nb = 0;
      for (int j = threadIdx.x; j < p; j += 32) {
        if (badsh[j]) { ++nb; continue; }
        lo = fmin(lo, aux[j]);
        hi = fmax(hi, aux[j]);
      }
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
        nb += __shfl_xor_sync(0xFFFFFFFFu, nb, o);
      }
      if (threadIdx.x == 0) stats[0] = (nb > 0 || !(hi <= 1e4 * lo)) ? 1 : 0;
    }
    return;
  }
  // MODE 2: Rayleigh-Ritz eigensolve (X holds V^T, ld p)
  for (int t = threadIdx.x; t < p * p; t += NT) X[t] = (t / p == t % p) ? 1.0 : 0.0;
  PROBE(4);
  const int sweeps = jacobi_block<p, ld>(S, X, rcs[0], rcs[1], rpq[0], rpq[1], &flag_sh, max_sweeps);
  PROBE(5);
  if (threadIdx.x < p) aux[threadIdx.x] = S[threadIdx.x * ld + threadIdx.x];
  __syncthreads();
  if (threadIdx.x < p) {
    int rk = 0;
    const double di = aux[threadIdx.x];
    for (int j = 0; j < p; ++j) rk += (aux[j] > di) || (aux[j] == di && j < (int)threadIdx.x);
    rank_sh[threadIdx.x] = rk;
  }
  __syncthreads();
  // W[row][rank(col)] = V[row][col] = V^T[col][row]
  for (int t = threadIdx.x; t < p * p; t += NT) {
    const int col = t / p, row = t % p;
    out0[row * p + rank_sh[col]] = X[col * p + row];
  }
  if (threadIdx.x < p) out1[rank_sh[threadIdx.x]] = aux[threadIdx.x] * ldexp(1.0, e);
  if (threadIdx.x == 0 && stats) stats[0] = sweeps;
}

// Q = Y R^{-1} (R upper from CholQR) by row-wise forward substitution, one thread per row,
// right-looking so every q_k finalises after one multiply: acc_c -= q_k R_kc (c > k).
// Columns flagged bad come out zero (re-drawn at random afterwards).  Q32 mirrors Q.
template <int P>
__global__ void __launch_bounds__(32) trsm_kernel(const double* Y, const double* __restrict__ R,
                                                  const double* __restrict__ dinv, const int* __restrict__ bad,
                                                  const int* __restrict__ gate, int64_t m, double* Q,
                                                  float* __restrict__ Q32) {
  if (gate && *gate == 0) return;
  extern __shared__ double sR[];  // [P * P]
  __shared__ double sd[P];
  for (int t = threadIdx.x; t < P * P / 2; t += blockDim.x)
    reinterpret_cast<double2*>(sR)[t] = reinterpret_cast<const double2*>(R)[t];
  for (int t = threadIdx.x; t < P; t += blockDim.x) sd[t] = bad[t] ? 0.0 : dinv[t];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  double acc[P];
#pragma unroll
  for (int c = 0; c < P; c += 2) {
    const double2 v = reinterpret_cast<const double2*>(Y + r * P)[c / 2];
    acc[c] = v.x;
    acc[c + 1] = v.y;
  }
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const double qk = acc[k] * sd[k];
    acc[k] = qk;
#pragma unroll
    for (int c = k + 1; c < P; ++c) acc[c] = fma(-qk, sR[k * P + c], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < P; c += 2) {
    reinterpret_cast<double2*>(Q + r * P)[c / 2] = make_double2(acc[c], acc[c + 1]);
    if (Q32) reinterpret_cast<float2*>(Q32 + r * P)[c / 2] = make_float2((float)acc[c], (float)acc[c + 1]);
  }
}

// ---------------------------------------------------------------- Out = In * M (m x p)(p x p)
// in place allowed (each CTA stages its rows before writing them); optional fp32 mirrors
__global__ void __launch_bounds__(256) matpp_kernel(const double* In0, double* Out0, float* Out0f, const double* In1,
                                                    double* Out1, float* Out1f, const double* __restrict__ M, int64_t m, int p) {
  extern __shared__ double sm[];
  double* sM = sm;                 // p*p
  double* sI = sm + p * p;         // 16 rows x p
  for (int t = threadIdx.x; t < p * p; t += 256) sM[t] = M[t];
  const int64_t r0 = (int64_t)blockIdx.x * 16;
  for (int w = 0; w < 2; ++w) {
    const double* In = w ? In1 : In0;
    double* Out = w ? Out1 : Out0;
    float* Outf = w ? Out1f : Out0f;
    if (!In) continue;
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * p; t += 256) sI[t] = (r0 + t / p < m) ? In[r0 * p + t] : 0.0;
    __syncthreads();
    for (int t = threadIdx.x; t < 16 * p; t += 256) {
      const int rr = t / p, cc = t % p;
      if (r0 + rr >= m) continue;
      double s0 = 0.0, s1 = 0.0;
      int q = 0;
      for (; q + 1 < p; q += 2) {
        s0 = fma(sI[rr * p + q], sM[q * p + cc], s0);
        s1 = fma(sI[rr * p + q + 1], sM[(q + 1) * p + cc], s1);
      }
      if (q < p) s0 = fma(sI[rr * p + q], sM[q * p + cc], s0);
      const double s = s0 + s1;
      Out[(r0 + rr) * p + cc] = s;
      if (Outf) Outf[(r0 + rr) * p + cc] = (float)s;
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

// V_out[j][r] = sign_r * U[j][r] (r < k), sign making the largest-|.| entry positive
// (smallest j on ties; R8); sigma_r = sqrt(max(theta_r, 0)); V32 fp32 copy.
// Also t_r = sum_a d_a^2 v_ra^2 (lambda_r (1 - 2 v_ra^2) + v_ra^2 G_aa) over the columns with
// rounding errors (precision bound, run_eig).
__global__ void finalize_vectors_kernel(const double* __restrict__ U, const double* __restrict__ theta, int64_t m,
                                        int p, int k, int k_pad, const int32_t* __restrict__ shift,
                                        const double* __restrict__ qerr, const double* __restrict__ G, int64_t ldg,
                                        double* __restrict__ V, double* __restrict__ sigma, float* __restrict__ V32,
                                        double* __restrict__ prec) {
  __shared__ double sv[256], st[256];
  __shared__ int64_t sj[256];
  const int r = blockIdx.x;
  double best = -1.0, tr = 0.0;
  int64_t bj = 0;
  const double lam = fmax(theta[r], 0.0);
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double u = U[j * p + r];
    const double a = fabs(u);
    if (a > best) { best = a; bj = j; }
    if (qerr[j] != 0.0) {
      const double u2 = u * u;
      tr += ldexp(u2 * fmax(lam * (1.0 - 2.0 * u2) + u2 * G[j * ldg + j], 0.0), -2 * shift[j]);
    }
  }
  sv[threadIdx.x] = best;
  sj[threadIdx.x] = bj;
  st[threadIdx.x] = tr;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) st[threadIdx.x] += st[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    prec[r] = st[0];
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

// Bound of the spike-energy error (run_eig): var(d E_spike) <= sum_a d_a^2 (w_a (1 - 2 P_aa) +
// P_aa^2 G_aa), w_a = sum_r lambda_r v_ra^2, P_aa = sum_r v_ra^2 -> prec[k]; one CTA, fixed order
__global__ void __launch_bounds__(1024) prec_energy_kernel(const double* __restrict__ V, const double* __restrict__ theta,
                                                           int64_t m, int k, const int32_t* __restrict__ shift,
                                                           const double* __restrict__ qerr,
                                                           const double* __restrict__ G, int64_t ldg,
                                                           double* __restrict__ prec) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 1024) {
    if (qerr[j] == 0.0) continue;
    double P = 0.0, w = 0.0;
    for (int r = 0; r < k; ++r) {
      const double v2 = V[j * k + r] * V[j * k + r];
      P += v2;
      w = fma(fmax(theta[r], 0.0), v2, w);
    }
    acc += ldexp(fmax(w * (1.0 - 2.0 * P) + P * P * G[j * ldg + j], 0.0), -2 * shift[j]);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 32; ++i) t += sh[i];
    prec[k] = t;
  }
}

// ---------------------------------------------------------------- mean-bias diagnostics
// ("Mean bias phenomenon"): the mean direction mu_hat and the
// top right singular vector v_1 of the UNCENTRED X, whose Gram is X^T X = G + l mu mu^T.
// ||mu|| (one CTA, fixed order) -> diag[0]; q_0 = mu / ||mu|| -> diag[4..4+m_pad)
__global__ void mu_norm_kernel(const double* __restrict__ mu, int64_t m, int64_t m_pad, double* __restrict__ diag) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) s = fma(mu[j], mu[j], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  const double nrm = sqrt(sh[0]);
  if (threadIdx.x == 0) diag[0] = nrm;
  double* q = diag + 4;
  for (int64_t j = threadIdx.x; j < m_pad; j += 256) q[j] = (j < m && nrm > 0.0) ? mu[j] / nrm : 0.0;
}

// m-length fixed-order dot products of one CTA (256 threads): returns (a . b, b . b)
__device__ __forceinline__ double2 cta_dots(const double* __restrict__ a, const double* __restrict__ b, int64_t m,
                                            double* sh) {
  double s = 0.0, t = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    s = fma(a[j], b[j], s);
    t = fma(b[j], b[j], t);
  }
  sh[threadIdx.x] = s;
  sh[256 + threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sh[threadIdx.x] += sh[threadIdx.x + w];
      sh[256 + threadIdx.x] += sh[256 + threadIdx.x + w];
    }
    __syncthreads();
  }
  const double2 r = make_double2(sh[0], sh[256]);
  __syncthreads();
  return r;
}

// One power step on the uncentred Gram:  dst = (G + l mu mu^T) src / ||src||.  Every CTA
// recomputes mu.src and ||src|| (fixed order) so no inter-CTA reduction is needed; one warp per
// row of the L2-resident G32, fp64 accumulation.
__global__ void __launch_bounds__(256) power_u_kernel(const float* __restrict__ G32, int64_t ld,
                                                      const double* __restrict__ mu, int64_t m, double l,
                                                      const double* __restrict__ src, double* __restrict__ dst) {
  __shared__ double sh[512];
  const double2 d = cta_dots(mu, src, m, sh);
  const double inv = d.y > 0.0 ? 1.0 / sqrt(d.y) : 0.0;
  const double lmq = l * d.x * inv;  // l (mu . q)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t a = (int64_t)blockIdx.x * 8 + warp; a < m; a += (int64_t)gridDim.x * 8) {
    const float* row = G32 + a * ld;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int64_t b = lane;
    for (; b + 96 < m; b += 128) {
      acc0 = fma((double)row[b], src[b], acc0);
      acc1 = fma((double)row[b + 32], src[b + 32], acc1);
      acc2 = fma((double)row[b + 64], src[b + 64], acc2);
      acc3 = fma((double)row[b + 96], src[b + 96], acc3);
    }
    for (; b < m; b += 32) acc0 = fma((double)row[b], src[b], acc0);
    double acc = (acc0 + acc1) + (acc2 + acc3);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if (lane == 0) dst[a] = acc * inv + lmq * mu[a];
  }
}

// q = src / ||src||, y = Gu q (= dst):  diag[1] = q.y (Rayleigh quotient), diag[2] =
// ||y - (q.y) q|| / (q.y) (residual), diag[3] = mu . q
__global__ void power_u_stats_kernel(const double* __restrict__ mu, int64_t m, const double* __restrict__ src,
                                     const double* __restrict__ dst, double* __restrict__ diag) {
  __shared__ double sh[512];
  const double2 a = cta_dots(src, dst, m, sh);   // (src . dst, dst . dst)
  const double2 b = cta_dots(mu, src, m, sh);    // (mu . src, src . src)
  const double ns = sqrt(b.y);
  const double lam = ns > 0.0 ? a.x / ns : 0.0;  // q.y with q = src/|src|, y = dst
  // ||y - lam q||^2 elementwise (no cancellation), fixed order
  double r = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += 256) {
    const double e = dst[j] - (ns > 0.0 ? lam * src[j] / ns : 0.0);
    r = fma(e, e, r);
  }
  sh[threadIdx.x] = r;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    diag[1] = lam;
    diag[2] = lam > 0.0 ? sqrt(sh[0]) / lam : 0.0;
    diag[3] = ns > 0.0 ? b.x / ns : 0.0;
  }
}

}  // namespace

avd_status launch_gram_finalize(Ctx* c) {
  const int64_t m = c->cfg.m;
  const double unit = (c->nd == 3) ? 16384.0 : 1.0;
  dim3 grid((unsigned)(c->m_pad / 32), (unsigned)(c->m_pad / 32));
  gram_finalize_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(c->gram_i, m, c->m_pad, c->shift, c->qsum, c->ysq, c->mu,
                                                            c->mu0, (double)c->cfg.l_global,
                                                            1.0 / (double)c->cfg.l_global, unit, c->G, c->G32);
  AVD_LAUNCHED(c);
  trace_kernel<<<1, 1024, 0, c->stream>>>(c->G, m, c->m_pad, c->ysq, c->mu0, (double)c->cfg.l_global, c->stats,
                                          c->trace, c->gmax);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// split-K geometry shared by the plan (workspace) and the launches
void gemm_geometry(int64_t m, int64_t m_pad, int p, int num_sms, bool fp32, int* BM, int* KS, int* RB, int* KT) {
  *BM = (fp32 && p <= 64) ? 128 : 64;  // = 16 * NR of the gemm32 / gemm64 instantiations
  *RB = (int)(m_pad / *BM);
  *KT = (int)ceil_div(m, kSkBK);
  const int64_t want = (int64_t)num_sms * (fp32 ? 3 : 2);  // resident CTAs (smem-bound)
  *KS = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, *RB), *KT));
}
size_t gemm_part_bytes(int64_t m, int64_t m_pad, int p, int num_sms) {
  size_t best = 0;
  for (int f = 0; f < 2; ++f) {
    int BM, KS, RB, KT;
    gemm_geometry(m, m_pad, p, num_sms, f == 0, &BM, &KS, &RB, &KT);
    best = std::max(best, (size_t)RB * KS * BM * p * (f == 0 ? sizeof(float) : sizeof(double)));
  }
  return (size_t)round_up((int64_t)best, 256) + sizeof(unsigned) * (size_t)(m_pad / 64 + 1);  // partials + tickets
}

namespace {

// Y = G In (fp64 G, fp64 math) or Y = G32 In32 (fp32); Y fp64 (+ optional fp32 mirror)
template <typename T, int NR, int NC>
avd_status gemm_launch(Ctx* c, const T* Gm, const T* In, double* Y, float* Y32) {
  int BM, KS, RB, KT;
  const int p = 8 * NC;
  gemm_geometry(c->cfg.m, c->m_pad, p, c->num_sms, sizeof(T) == 4, &BM, &KS, &RB, &KT);
  if (BM != 16 * NR) { set_error("gemm geometry mismatch"); return AVD_EINVAL; }
  const int sm = kSkStages * (kSkBK * BM + kSkBK * p) * (int)sizeof(T);
  AVD_CUDA(smem_attr(gemm_kernel<T, NR, NC>, sm));
  const size_t pb = gemm_part_bytes(c->cfg.m, c->m_pad, c->p, c->num_sms);
  T* part = reinterpret_cast<T*>(c->gemm_part);
  unsigned* tickets = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(c->gemm_part) + pb -
                                                  sizeof(unsigned) * (size_t)(c->m_pad / 64 + 1));
  gemm_kernel<T, NR, NC><<<RB * KS, kSkThreads, sm, c->stream>>>(Gm, c->m_pad, In, c->cfg.m, KT, KS, part, tickets, Y,
                                                                 Y32);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status gemm64(Ctx* c, const double* In, double* Y, float* Y32) {
  switch (c->p / 16) {
#define CASE(PC) case PC: return gemm_launch<double, 4, 2 * PC>(c, c->G, In, Y, Y32);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
  set_error("unsupported p");
  return AVD_EINVAL;
}
avd_status gemm32(Ctx* c, const float* In, double* Y, float* Y32) {
  switch (c->p / 16) {
#define CASE(PC) case PC: return gemm_launch<float, (PC <= 4 ? 8 : 4), 2 * PC>(c, c->G32, In, Y, Y32);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
  set_error("unsupported p");
  return AVD_EINVAL;
}

template <int MODE>
avd_status atb_fused(Ctx* c, const double* A, const double* B, double* out0, double* out1, int* ibad, int* stats,
                     const int* gate = nullptr, int max_sweeps = 40) {
  const int p = c->p;
  const int n_red = (int)ceil_div(c->cfg.m, kRedRows);
  const int chunk = p <= 48 ? kRedRows : 64;
  const size_t sm = std::max<size_t>(2 * (size_t)chunk * p, (size_t)p * (p + 1) + (size_t)p * p) * sizeof(double);
  switch (p / 16) {
#define CASE(PC)                                                                                                \
  case PC:                                                                                                      \
    AVD_CUDA(smem_attr(atb_fused_kernel<MODE, PC>, (int)sm)); \
    atb_fused_kernel<MODE, PC><<<n_red, RedCfg<PC>::threads, sm, c->stream>>>(A, B, c->cfg.m, c->red_part, c->ticket, out0, out1,  \
                                                              ibad, stats, gate, max_sweeps);                   \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status matpp(Ctx* c, const double* In0, double* Out0, float* Out0f, const double* In1, double* Out1,
                 float* Out1f, const double* M) {
  const int p = c->p;
  const size_t sm = ((size_t)p * p + 16 * p) * sizeof(double);
  AVD_CUDA(smem_attr(matpp_kernel, (int)sm));
  matpp_kernel<<<(unsigned)ceil_div(c->cfg.m, 16), 256, sm, c->stream>>>(In0, Out0, Out0f, In1, Out1, Out1f, M,
                                                                         c->cfg.m, p);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

avd_status trsm(Ctx* c, const double* Y, const double* R, const double* dinv, const int* bad, const int* gate) {
  const unsigned grid = (unsigned)ceil_div(c->cfg.m, 32);
  switch (c->p / 16) {
#define CASE(PC)                                                                                              \
  case PC:                                                                                                    \
    AVD_CUDA(smem_attr(trsm_kernel<16 * PC>, 256 * PC * PC * 8)); \
    trsm_kernel<16 * PC><<<grid, 32, 256 * PC * PC * 8, c->stream>>>(Y, R, dinv, bad, gate, c->cfg.m, c->Q, c->Q32); \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
    default: set_error("unsupported p"); return AVD_EINVAL;
  }
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// Q <- orth(Y) by Cholesky-QR (Q32 mirrors Q).  The second pass (CholQR2) runs only when the
// first one flagged it (a rank-deficient column, re-drawn at random in between, or
// cond(R)^2 > 1e6, where one pass leaves orthogonality errors above ~1e-10); otherwise its two
// kernels exit at once.
avd_status orth(Ctx* c, const double* Y, uint32_t seed) {
  int* bad = reinterpret_cast<int*>(c->resid + c->p);
  int* need2 = bad + c->p;
  const int p = c->p;
  for (int pass = 0; pass < 2; ++pass) {
    const double* src = pass == 0 ? Y : c->Q;
    const int* gate = pass == 0 ? nullptr : need2;
    AVD_TRY(atb_fused<1>(c, src, src, c->W, c->H, bad, pass == 0 ? need2 : nullptr, gate));  // R -> W, 1/R_jj -> H
    AVD_TRY(trsm(c, src, c->W, c->H, bad, gate));                   // in place allowed (row-wise)
    if (pass == 0) {
      rand_fill_kernel<<<(unsigned)ceil_div(c->cfg.m * p, 256), 256, 0, c->stream>>>(c->Q, c->Q32, c->cfg.m, p, seed, bad);
      AVD_LAUNCHED(c);
    }
  }
  return AVD_OK;
}

}  // namespace

// A-posteriori bound of the Gram operand's quantisation error (DESIGN.md §8 "Gram precision").
// The operand is q_ia = y_ia + e_ia, y = (x - mu0) 2^shift, with dithered rounding errors e that
// are zero-mean, independent and var e <= 1/4 (exactly 0 for a column whose every entry is on the
// grid: qerr_a = 0).  The diagonal of G is the exact centred energy (fp64 sums of the fused pass),
// the off-diagonal is E_ab = d_a d_b sum_i (e_ia xc_ib + xc_ia e_ib) + O(e^2) (d_a = 2^-shift_a),
// so to first order, with X~ v_r = sigma_r u_r and X~^T u_r = sigma_r v_r,
//   d lambda_r = v_r^T E v_r = 2 sum_ia d_a v_ra e_ia (sigma_r u_ri - v_ra xc_ia),
//   var <= t_r = sum_a d_a^2 v_ra^2 (lambda_r (1 - 2 v_ra^2) + v_ra^2 G_aa)      (finalize kernel)
//   d E_spike = sum_r d lambda_r = 2 sum_ia d_a e_ia (S_ia - P_aa xc_ia),  P = V_k V_k^T,
//   var <= sum_a d_a^2 (w_a (1 - 2 P_aa) + P_aa^2 G_aa),  w_a = sum_r lambda_r v_ra^2 (prec kernel)
// (S the spike matrix).  A column carried by one massive entry (v_r ~ e_a) drops out, as it
// should: its diagonal is exact.  E_tail = tr(G) - E_spike inherits d E_spike (tr(G) is exact up
// to the fp32 rounding of y, counted as 1e-9 tr(G)).  At 5 sigma:
//   prec_sigma = max_r 2.5 sqrt(t_r) / lambda_r  (relative error of sigma_r = d lambda / 2 lambda)
//   prec_share = max(5 std(d E_spike) / E_spike, (5 std(d E_spike) + 1e-9 tr(G)) / E_tail)
// The automatic digit rule raises the operand to 3 digits when prec_sigma > 5e-5 or
// prec_share > 5e-6 (half the north-star tolerances 1e-4 / 1e-5).
avd_status precision_bound(Ctx* c) {
  const int k = c->k;
  double* h = c->eig_host + 2 * kMaxP;  // pinned scratch: t_r [k <= 95], var(d E_spike), tr(G)
  AVD_CUDA(cudaMemcpyAsync(h, c->prec, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaMemcpyAsync(h + k + 1, c->trace, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  double ps = 0.0, e_spike = 0.0;
  for (int r = 0; r < k; ++r) {
    const double lam = std::max(c->eig_host[r], 0.0);  // Ritz values of the last check (theta)
    const double t = std::max(h[r], 0.0);
    if (lam > 0.0) ps = std::max(ps, 2.5 * std::sqrt(t) / lam);
    e_spike += lam;
  }
  const double sd_spike = std::sqrt(std::max(h[k], 0.0));
  const double trace = h[k + 1];
  const double e_tail = std::max(trace - e_spike, 0.0);
  double pe = 0.0;
  if (e_spike > 0.0) pe = std::max(pe, 5.0 * sd_spike / e_spike);
  if (sd_spike > 0.0 && e_tail > 0.0) pe = std::max(pe, (5.0 * sd_spike + 1e-9 * trace) / e_tail);
  else if (sd_spike > 0.0) pe = HUGE_VAL;
  c->prec_sigma = ps;
  c->prec_share = pe;
  return AVD_OK;
}

// Subspace iteration: power steps Q <- orth(G^2 Q) in fp32; a Rayleigh-Ritz check (fp64) runs
// on a schedule predicted from the observed residual decay (at most every 8 steps, always on the
// last one), so the p x p Jacobi runs ~2-3 times per solve.
avd_status run_eig(Ctx* c) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  const uint32_t seed = (uint32_t)(c->cfg.seed ^ (c->cfg.seed >> 32)) * 2654435761u + 12345u;
  int* jstats = reinterpret_cast<int*>(c->theta + p);  // [16] sweeps per RR solve
  AVD_CUDA(cudaMemsetAsync(jstats, 0, 16 * sizeof(int), c->stream));
  AVD_CUDA(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned), c->stream));
  {  // split-K tickets (re-armed by every launch; cleared here once per solve)
    const size_t pb = gemm_part_bytes(m, c->m_pad, p, c->num_sms), tb = sizeof(unsigned) * (size_t)(c->m_pad / 64 + 1);
    AVD_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(c->gemm_part) + pb - tb, 0, tb, c->stream));
  }
  rand_fill_kernel<<<(unsigned)ceil_div(m * p, 256), 256, 0, c->stream>>>(c->Z, nullptr, m, p, seed, nullptr);
  AVD_LAUNCHED(c);
  AVD_TRY(orth(c, c->Z, seed + 1));
  const int max_it = c->cfg.max_iters > 0 ? c->cfg.max_iters : 200;
  const double tol = c->cfg.eig_tol > 0 ? c->cfg.eig_tol : 1e-6;  // V angle <~ tol * lambda_1 / gap_k
  int it = 0, next_rr = 2, prev_it = 0, rr_count = 0;
  double maxres = 0.0, prev_res = -1.0, pred_res = -1.0;
  bool conv = false;
  for (it = 1; it <= max_it; ++it) {
    if (it == next_rr || it == max_it) {
      ++rr_count;
      AVD_TRY(gemm64(c, c->Q, c->Y, nullptr));           // Y = G Q (exact G, fp64)
      // an intermediate check only needs an orthonormal basis of the subspace and honest
      // residuals: its Jacobi is capped at 3 sweeps (the residuals of the rotated basis are still
      // true residuals, so a capped solve can only delay convergence, never fake it); a check
      // that could end the solve (predicted residual within 10x of tol, or the last iteration)
      // runs to full convergence.
      const bool final_ish = it == max_it || (pred_res >= 0.0 && pred_res <= 10.0 * tol);
      AVD_TRY(atb_fused<2>(c, c->Q, c->Y, c->W, c->theta, nullptr, jstats + std::min(rr_count - 1, 15), nullptr,
                           final_ish ? 40 : 3));
      AVD_TRY(matpp(c, c->Y, c->Z, c->Z32, c->Q, c->U, nullptr, c->W));  // Z = Y W, U = Q W (Ritz vectors)
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
        step = (int)std::max(1.0, std::min(8.0, std::ceil(need)));
      }
      prev_res = maxres;
      prev_it = it;
      next_rr = it + step;
      pred_res = (rate > 0.0 && rate < 0.95) ? maxres * std::pow(rate, (double)step) : -1.0;
      AVD_TRY(gemm32(c, c->Z32, c->Y, nullptr));        // Y = G Z = G^2 U
    } else {
      AVD_TRY(gemm32(c, c->Q32, c->Z, c->Z32));         // Z = G Q
      AVD_TRY(gemm32(c, c->Z32, c->Y, nullptr));        // Y = G Z = G^2 Q
    }
    AVD_TRY(orth(c, c->Y, seed + 7919u * (uint32_t)it));
  }
  c->iters = std::min(it, max_it);
  c->rr_count = rr_count;
  c->max_resid = maxres;
  c->sigma_next = (k < p) ? std::sqrt(std::max(c->eig_host[k], 0.0)) : 0.0;
  // the per-solve sweep counts stay at theta + p; the report stage reads them with its packed copy
  AVD_CUDA(cudaMemsetAsync(c->V32, 0, sizeof(float) * m * c->k_pad, c->stream));
  finalize_vectors_kernel<<<k, 256, 0, c->stream>>>(c->U, c->theta, m, p, k, c->k_pad, c->shift, c->qerr, c->G,
                                                    c->m_pad, c->V, c->sigma, c->V32, c->prec);
  AVD_LAUNCHED(c);
  prec_energy_kernel<<<1, 1024, 0, c->stream>>>(c->V, c->theta, m, k, c->shift, c->qerr, c->G, c->m_pad, c->prec);
  AVD_LAUNCHED(c);
  AVD_TRY(precision_bound(c));
  return conv ? AVD_OK : AVD_ENOCONV;
}

// Mean-bias diagnostics on the replicated G and mu (no exchange): power iteration on the uncentred
// Gram from q_0 = mu_hat (already aligned when the mean dominates), in blocks of
// 4 steps until the residual is <= 1e-8 (at most 64 steps).  Fills c->sigma1_u = sqrt(lambda_1),
// c->alpha1 = |mu . v_1| (= (sigma_1 / l) u_1^T 1), c->cos_mu_v1 = alpha1 / ||mu||.
avd_status run_uncentred(Ctx* c) {
  const int64_t m = c->cfg.m;
  mu_norm_kernel<<<1, 256, 0, c->stream>>>(c->mu, m, c->m_pad, c->diag);
  AVD_LAUNCHED(c);
  double* q = c->diag + 4;
  double* y = q + c->m_pad;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), 4LL * c->num_sms);
  double* h = c->eig_host + 3 * kMaxP;  // pinned scratch, 4 doubles
  for (int t = 0; t < 4; ++t) h[t] = 0.0;
  int it = 0;
  for (int blk = 0; blk < 16; ++blk) {
    for (int t = 0; t < 4; ++t, ++it) {
      power_u_kernel<<<grid, 256, 0, c->stream>>>(c->G32, c->m_pad, c->mu, m, (double)c->cfg.l_global, q, y);
      AVD_LAUNCHED(c);
      std::swap(q, y);  // q now holds the unnormalised product
    }
    power_u_kernel<<<grid, 256, 0, c->stream>>>(c->G32, c->m_pad, c->mu, m, (double)c->cfg.l_global, q, y);
    AVD_LAUNCHED(c);
    power_u_stats_kernel<<<1, 256, 0, c->stream>>>(c->mu, m, q, y, c->diag);
    AVD_LAUNCHED(c);
    AVD_CUDA(cudaMemcpyAsync(h, c->diag, sizeof(double) * 4, cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));
    if (!(h[0] > 0.0) || h[2] <= 1e-8) break;
  }
  c->iters_u = it;
  c->sigma1_u = std::sqrt(std::max(h[1], 0.0));
  c->alpha1 = std::fabs(h[3]);
  c->cos_mu_v1 = h[0] > 0.0 ? std::min(1.0, std::fabs(h[3]) / h[0]) : 0.0;
  c->resid_u = h[2];
  return AVD_OK;
}

}  // namespace avd
