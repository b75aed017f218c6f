#include <vector>
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
#include <cstdlib>
#include <cstddef>
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
// (seed + 7919 * *itp when itp != nullptr: the iteration counter of the device-resident loop)
__global__ void rand_fill_kernel(double* __restrict__ Q, float* __restrict__ Q32, int64_t m, int p, uint32_t seed,
                                 const int* __restrict__ flags, const int* __restrict__ itp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * p) return;
  const int c = (int)(t % p);
  if (flags && !flags[c]) return;
  if (itp) seed += 7919u * (uint32_t)(*itp);
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
                                                          double* __restrict__ Y, float* __restrict__ Y32,
                                                          const int* __restrict__ skip, int rb0) {
  if (skip && *skip) return;  // device-side gate (eigensolver graph: Z comes from the RR check)
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
  const int rb = rb0 + (int)(blockIdx.x / KS), ks = (int)(blockIdx.x % KS);
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
  T* pp = part + ((int64_t)(rb - rb0) * KS + ks) * (BM * p);
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
  const T* base = part + (int64_t)(rb - rb0) * KS * (BM * p);
  for (int e = tid * 2; e < BM * p; e += kSkThreads * 2) {
    // the KS partials in order; loads batched 8 at a time so they are in flight together (the
    // sum is still the sequential q order)
    double s0 = 0.0, s1 = 0.0;
    int q = 0;
    for (; q + 8 <= KS; q += 8) {
      double a0[8], a1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const T* src = base + (int64_t)(q + u) * (BM * p) + e;
        if constexpr (sizeof(T) == 4) {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(src));
          a0[u] = (double)v.x; a1[u] = (double)v.y;
        } else {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(src));
          a0[u] = v.x; a1[u] = v.y;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) { s0 += a0[u]; s1 += a1[u]; }
    }
    for (; q < KS; ++q) {
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
__device__ __forceinline__ void jacobi_rotation(double app, double aqq, double apq, double& c, double& s, bool& rot,
                                                double thr2 = 1e-18) {
  c = 1.0;
  s = 0.0;
  rot = false;
  // |a_pq| <= 1e-9 sqrt(a_pp a_qq): eigenvalue error ~1e-18 relative, eigenvector error ~1e-9 / gap
  if (!(apq * apq > thr2 * fabs(app * aqq)) || fabs(apq) < 1e-30 || fabs(apq) > 1e30) return;
  const float th = __fdividef(0.5f * (float)(aqq - app), (float)apq);
  const float ath = fabsf(th);
  if (!(ath < 1e18f)) return;  // |a_pq| below 1e-18 |a_qq - a_pp|: nothing left to rotate
  float t = __fdividef(1.0f, ath + sqrtf(fmaf(th, th, 1.0f)));
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

// One-sided (Hestenes) Jacobi on the symmetric positive semidefinite A (P x P, ld LDA): rotate
// column pairs of A (A <- A J) and of V (rows of V^T) until every pair of columns is orthogonal;
// then A = H V has orthogonal columns, ||A_j|| = lambda_j and V holds the eigenvectors (for PSD H the
// singular and eigen decompositions coincide).  The rotation of a pair comes from its Gram entries
// (alpha = |a_p|^2, beta = |a_q|^2, gamma = a_p . a_q) by the same Rutishauser formula as the
// two-sided method; stop when gamma^2 <= 1e-20 alpha beta for every pair.  Step s rotates the P/2
// disjoint pairs of the round-robin ordering; half-warp u owns pair u (its two columns of A and two
// rows of V^T), so a step needs no synchronisation inside, only one barrier before the next step.
// Half-warps rather than warps: the step is bound by the shuffle pipe (three fp64 butterflies per
// pair), and a 16-lane butterfly serves two pairs per warp instruction with one level fewer.
// kfix < P: the basis is ordered (columns >= kfix span the unconverged tail of the spectrum) and
// rotations between two tail columns are skipped — they only mix tail vectors among themselves, so
// the leading kfix pairs are exact eigenpairs of A once the coupling pairs are orthogonal, and the
// tail block (whose Ritz vectors are not converged anyway) costs no sweeps.  Returns the sweeps.
template <int P, int LDA>
__device__ int jacobi_onesided(double* A, double* Vt, int* fl, int max_sweeps, int kfix) {
  constexpr int half = P / 2;
  constexpr int E = (P + 15) / 16;  // column elements per lane
  const int hw = threadIdx.x >> 4, hl = threadIdx.x & 15;
  const int nhw = blockDim.x >> 4;
  const unsigned hmask = (threadIdx.x & 16) ? 0xFFFF0000u : 0x0000FFFFu;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) fl[sweep & 1] = 0;  // read after this sweep's last barrier
    __syncthreads();
    for (int step = 0; step < P - 1; ++step) {
      for (int u = hw; u < half; u += nhw) {
        int pc, qc;
        rr_pair(P, step, u, pc, qc);
        if (pc >= kfix) continue;  // tail-tail pair (pc < qc)
        double ap[E], aq[E];
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int i = hl + 16 * t;
          ap[t] = i < P ? A[i * LDA + pc] : 0.0;
          aq[t] = i < P ? A[i * LDA + qc] : 0.0;
          al = fma(ap[t], ap[t], al);
          be = fma(aq[t], aq[t], be);
          ga = fma(ap[t], aq[t], ga);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          al += __shfl_xor_sync(hmask, al, o);
          be += __shfl_xor_sync(hmask, be, o);
          ga += __shfl_xor_sync(hmask, ga, o);
        }
        double c, sn;
        bool rot;
        jacobi_rotation(al, be, ga, c, sn, rot, 1e-20);  // identical in every lane of the half
        if (!rot) continue;
        if (hl == 0) fl[sweep & 1] = 1;
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int i = hl + 16 * t;
          if (i < P) {
            A[i * LDA + pc] = c * ap[t] - sn * aq[t];
            A[i * LDA + qc] = sn * ap[t] + c * aq[t];
            const double vp = Vt[pc * P + i], vq = Vt[qc * P + i];
            Vt[pc * P + i] = c * vp - sn * vq;
            Vt[qc * P + i] = sn * vp + c * vq;
          }
        }
      }
      __syncthreads();
    }
    if (!fl[sweep & 1]) break;
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
    int* __restrict__ stats, const int* __restrict__ gate, int max_sweeps, const int* __restrict__ msw) {
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
  __shared__ int jfl[2];         // per-sweep "any rotation" flag
  __shared__ int badsh[p], rank_sh[p], escale;
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
  // msw[0]: sweep cap, msw[1]: leading block of an ordered basis (p: none)
  const int sweeps = jacobi_onesided<p, ld>(S, X, jfl, msw ? msw[0] : max_sweeps, msw ? msw[1] : p);
  // lambda_j = ||A e_j||, A = H V (fixed-order per-warp sums)
  for (int j = threadIdx.x >> 5; j < p; j += NT / 32) {
    double t = 0.0;
    for (int i = threadIdx.x & 31; i < p; i += 32) t = fma(S[i * ld + j], S[i * ld + j], t);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if ((threadIdx.x & 31) == 0) aux[j] = sqrt(t);
  }
  PROBE(5);
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
// Also the precision-bound sums (run_eig): t_r = sum_a d_a^2 v_ra^2 (lambda_r (1 - 2 v_ra^2) +
// v_ra^2 G_aa) and sum_a d_a^2 (w_a (1 - 2 P_aa) + P_aa^2 G_aa), w_a = sum_r lambda_r v_ra^2,
// P_aa = sum_r v_ra^2, over the columns with rounding errors (qerr != 0).
// Three kernels: per-block partials (one thread per row j of U, coalesced row reads), one CTA
// combining the partials in block order, and the sign-applied copy.
constexpr int kFinThreads = 128;
constexpr int kFinKMax = 96;
__global__ void __launch_bounds__(kFinThreads) fin_part_kernel(const double* __restrict__ U,
                                                              const double* __restrict__ theta, int64_t m, int p,
                                                              int k, const int32_t* __restrict__ shift,
                                                              const double* __restrict__ qerr,
                                                              const double* __restrict__ G, int64_t ldg,
                                                              double* __restrict__ part) {
  constexpr int NW = kFinThreads / 32;
  __shared__ double sv[NW][kFinKMax], st[NW][kFinKMax + 1];
  __shared__ int64_t sj[NW][kFinKMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * kFinThreads + threadIdx.x;
  const bool ok = j < m;
  const bool err = ok && qerr[j] != 0.0;
  const double gjj = err ? G[j * ldg + j] : 0.0;
  const double d2 = err ? ldexp(1.0, -2 * shift[j]) : 0.0;
  double Pjj = 0.0, wj = 0.0;
  for (int r = 0; r < k; ++r) {
    const double u = ok ? U[j * p + r] : 0.0;
    const double lam = fmax(theta[r], 0.0);
    const double u2 = u * u;
    Pjj += u2;
    wj = fma(lam, u2, wj);
    double best = ok ? fabs(u) : -1.0;
    int64_t bj = j;
    double t = err ? d2 * u2 * fmax(lam * (1.0 - 2.0 * u2) + u2 * gjj, 0.0) : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      const int64_t oj = __shfl_xor_sync(0xFFFFFFFFu, bj, o);
      if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
      t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    }
    if (lane == 0) { sv[warp][r] = best; sj[warp][r] = bj; st[warp][r] = t; }
  }
  double e = err ? d2 * fmax(wj * (1.0 - 2.0 * Pjj) + Pjj * Pjj * gjj, 0.0) : 0.0;
  for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xFFFFFFFFu, e, o);
  if (lane == 0) st[warp][kFinKMax] = e;
  __syncthreads();
  double* out = part + (int64_t)blockIdx.x * (3 * k + 1);
  for (int r = threadIdx.x; r <= k; r += kFinThreads) {
    if (r == k) {
      double tt = 0.0;
      for (int w = 0; w < NW; ++w) tt += st[w][kFinKMax];
      out[3 * k] = tt;
      continue;
    }
    double b = sv[0][r], tt = st[0][r];
    int64_t jj = sj[0][r];
    for (int w = 1; w < NW; ++w) {
      if (sv[w][r] > b || (sv[w][r] == b && sj[w][r] < jj)) { b = sv[w][r]; jj = sj[w][r]; }
      tt += st[w][r];
    }
    out[r] = b;
    out[k + r] = (double)jj;
    out[2 * k + r] = tt;
  }
}
// one warp per r (block r < k) plus one for the energy bound (block k): lanes take the block
// partials q = lane, lane + 32, ... (fixed order), then a fixed xor tree
__global__ void __launch_bounds__(32) fin_final_kernel(const double* __restrict__ part, int nb, int k,
                                                      const double* __restrict__ theta, const double* __restrict__ U,
                                                      int p, double* __restrict__ sigma, double* __restrict__ sgn,
                                                      double* __restrict__ prec) {
  const int r = blockIdx.x, lane = threadIdx.x;
  const int stride = 3 * k + 1;
  if (r == k) {
    double t = 0.0;
    for (int q = lane; q < nb; q += 32) t += part[(int64_t)q * stride + 3 * k];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if (lane == 0) prec[k] = t;
    return;
  }
  double b = -1.0, t = 0.0;
  int64_t jj = INT64_MAX;
  for (int q = lane; q < nb; q += 32) {
    const double* pq = part + (int64_t)q * stride;
    const double v = pq[r];
    const int64_t vj = (int64_t)pq[k + r];
    if (v > b || (v == b && vj < jj)) { b = v; jj = vj; }
    t += pq[2 * k + r];
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xFFFFFFFFu, b, o);
    const int64_t oj = __shfl_xor_sync(0xFFFFFFFFu, jj, o);
    if (ob > b || (ob == b && oj < jj)) { b = ob; jj = oj; }
    t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
  }
  if (lane == 0) {
    sgn[r] = U[jj * p + r] < 0.0 ? -1.0 : 1.0;
    sigma[r] = sqrt(fmax(theta[r], 0.0));
    prec[r] = t;
  }
}
__global__ void fin_write_kernel(const double* __restrict__ U, const double* __restrict__ sgn, int64_t m, int p, int k,
                                 int k_pad, double* __restrict__ V, float* __restrict__ V32) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * k_pad) return;
  const int64_t j = t / k_pad;
  const int r = (int)(t % k_pad);
  if (r < k) {
    const double v = sgn[r] * U[j * p + r];
    V[j * k + r] = v;
    V32[t] = (float)v;
  } else {
    V32[t] = 0.f;
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

__global__ void f64_to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) b[t] = (float)a[t];
}

// ---------------------------------------------------------------- uncentred top-k (f2)
// w_r = mu . Q_r (fixed order; one warp per column r)
__global__ void mu_dot_cols_kernel(const double* __restrict__ mu, const double* __restrict__ Q, int64_t m, int p,
                                   double* __restrict__ w) {
  const int r = blockIdx.x, lane = threadIdx.x;
  double s = 0.0;
  for (int64_t j = lane; j < m; j += 32) s = fma(mu[j], Q[j * p + r], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if (lane == 0) w[r] = s;
}
// Y += l mu w^T (the rank-one term of the uncentred Gram X^T X = G + l mu mu^T)
__global__ void rank1_kernel(double* __restrict__ Y, const double* __restrict__ mu, const double* __restrict__ w,
                             int64_t m, int p, double l) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * p) return;
  Y[t] = fma(l * mu[t / p], w[t % p], Y[t]);
}
// start block of the uncentred solve: column 0 = mu_hat (diag + 4), columns 1.. = the centred
// Ritz vectors U[:, 0 .. p-2]
__global__ void unc_start_kernel(const double* __restrict__ U, const double* __restrict__ muhat, int64_t m, int p,
                                 double* __restrict__ Z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m * p) return;
  const int64_t j = t / p;
  const int r = (int)(t % p);
  Z[t] = r == 0 ? muhat[j] : U[j * p + (r - 1)];
}
// sigma_i = sqrt(theta_i), alpha_i = |mu . u_i| of the Ritz vectors U (i < k); one warp per i
__global__ void unc_out_kernel(const double* __restrict__ U, const double* __restrict__ theta,
                               const double* __restrict__ mu, int64_t m, int p, int k, double* __restrict__ out) {
  const int i = blockIdx.x, lane = threadIdx.x;
  double s = 0.0;
  for (int64_t j = lane; j < m; j += 32) s = fma(mu[j], U[j * p + i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
  if (lane == 0) {
    out[i] = sqrt(fmax(theta[i], 0.0));
    out[k + i] = fabs(s);
  }
}

// ---------------------------------------------------------------- device-resident loop control
// The subspace iteration runs as ONE CUDA graph: WHILE(loop) { begin; IF(rr) {RR check; ctl_rr};
// IF(pow) {power step; orth; ctl_end} } — every decision the host used to take between launches
// (when to run a Rayleigh-Ritz check, how many Jacobi sweeps it may take, convergence) is taken
// here, on the device, from the same quantities and with the same rules.
struct EigCtl {
  int it;           // current iteration (1-based)
  int next_rr;      // iteration of the next Rayleigh-Ritz check
  int prev_it;      // iteration of the previous check
  int rr_count;     // checks so far
  int conv;         // 1: converged
  int max_it;
  int msw;          // Jacobi sweep cap of the current check (3 intermediate, 40 final)
  int kfix;         // (must follow msw) leading block of the check's ordered basis, p if unordered
  int last_sweeps;  // sweeps of the last check's Jacobi (atb_fused MODE 2 writes it)
  int rr_now;       // this iteration ran a check (the power step starts from its Z = G U)
  int blocks_u;     // uncentred power iteration: blocks of 4 steps
  int iters_u;
  int stop;         // the last check ended the loop
  int stop_u;       // the uncentred loop is done
  int rr_fast;      // this check is intermediate: its G Q product may be the fp32/int8 one
  int rr_exact;     // 1 - rr_fast (the gate of the other product)
  int k, p;
  double tol, prev_res, pred_res, maxres;
};
static_assert(sizeof(EigCtl) <= kEigCtlBytes, "EigCtl too large");
static_assert(offsetof(EigCtl, blocks_u) == 4 * kCtlBlocksU && offsetof(EigCtl, iters_u) == 4 * kCtlBlocksU + 4,
              "report reads blocks_u / iters_u by index");

__global__ void ctl_init_kernel(EigCtl* ctl, int max_it, double tol, int k, int p) {
  if (threadIdx.x != 0) return;
  ctl->k = k;
  ctl->p = p;
  ctl->kfix = p;
  ctl->it = 1;
  ctl->next_rr = 2;
  ctl->prev_it = 0;
  ctl->rr_count = 0;
  ctl->conv = 0;
  ctl->max_it = max_it;
  ctl->msw = 3;
  ctl->last_sweeps = 0;
  ctl->rr_now = 0;
  ctl->rr_fast = 0;
  ctl->rr_exact = 1;
  ctl->stop = 0;
  ctl->tol = tol;
  ctl->prev_res = -1.0;
  ctl->pred_res = -1.0;
  ctl->maxres = 0.0;
}
// top of the loop body: does this iteration run a check?  (sets both IF handles every iteration)
__global__ void ctl_begin_kernel(EigCtl* ctl, cudaGraphConditionalHandle h_rr, cudaGraphConditionalHandle h_pow) {
  if (threadIdx.x != 0) return;
  const int it = ctl->it;
  const bool rr = it == ctl->next_rr || it == ctl->max_it;
  // an intermediate check only needs an orthonormal basis of the subspace and honest residuals:
  // its Jacobi is capped at 3 sweeps (the residuals of the rotated basis are still true
  // residuals, so a capped solve can only delay convergence, never fake it); a check that could
  // end the solve (predicted residual within 10x of tol, or the last iteration) runs to full
  // convergence.
  const bool final_ish = it == ctl->max_it || (ctl->pred_res >= 0.0 && ctl->pred_res <= 10.0 * ctl->tol);
  ctl->msw = final_ish ? 40 : 3;
  // after a check, the power steps keep Q's columns in Ritz order (CholQR of G^2 Z, Z = Y W sorted),
  // so the tail-tail rotations can be skipped (jacobi_block)
  ctl->kfix = ctl->rr_count > 0 ? ctl->k : ctl->p;
  ctl->rr_now = rr ? 1 : 0;
  // an intermediate check only steers the basis and predicts the schedule: its product need not be
  // the fp64 one (a check that could end the solve always is)
  ctl->rr_fast = (rr && !final_ish) ? 1 : 0;
  ctl->rr_exact = 1 - ctl->rr_fast;
  if (h_rr) cudaGraphSetConditional(h_rr, rr ? 1u : 0u);  // 0 handles: host-driven profiling mode
  if (h_pow) cudaGraphSetConditional(h_pow, 1u);
}
// after a check: convergence, else the next check predicted from the observed residual decay
// per G^2 step (or (theta_p / theta_k)^2 before two checks exist), at most 8 steps ahead
__global__ void ctl_rr_kernel(EigCtl* ctl, const double* __restrict__ theta, const double* __restrict__ resid, int p,
                              int k, int* __restrict__ jstats, cudaGraphConditionalHandle h_loop,
                              cudaGraphConditionalHandle h_pow) {
  if (threadIdx.x != 0) return;
  const int it = ctl->it;
  const int rc = ctl->rr_count++;
  jstats[rc < 15 ? rc : 15] = ctl->last_sweeps;
  double maxres = 0.0;
  for (int r = 0; r < k; ++r) maxres = fmax(maxres, resid[r]);
  bool stop = false;
  if (!(theta[0] > 0.0)) { maxres = 0.0; ctl->conv = 1; stop = true; }  // G == 0: nothing to iterate
  else if (maxres <= ctl->tol && ctl->rr_fast) { maxres = 2.0 * ctl->tol; }  // confirm with an exact check
  else if (maxres <= ctl->tol) { ctl->conv = 1; stop = true; }
  else if (it == ctl->max_it) { stop = true; }
  ctl->maxres = maxres;
  if (!stop) {
    double rate = -1.0;
    if (ctl->prev_res > 0.0 && maxres < ctl->prev_res) rate = pow(maxres / ctl->prev_res, 1.0 / (double)(it - ctl->prev_it));
    else if (theta[k - 1] > 0.0) rate = pow(fmax(theta[p - 1], 0.0) / theta[k - 1], 2.0);
    int step = 1;
    if (rate > 0.0 && rate < 0.95) {
      const double need = log(ctl->tol / maxres) / log(rate);
      step = (int)fmax(1.0, fmin(8.0, ceil(need)));
    }
    ctl->prev_res = maxres;
    ctl->prev_it = it;
    ctl->next_rr = it + step;
    ctl->pred_res = (rate > 0.0 && rate < 0.95) ? maxres * pow(rate, (double)step) : -1.0;
  }
  ctl->stop = stop ? 1 : 0;
  if (stop && h_loop) cudaGraphSetConditional(h_loop, 0u);
  if (h_pow) cudaGraphSetConditional(h_pow, stop ? 0u : 1u);
}
__global__ void ctl_end_kernel(EigCtl* ctl) {
  if (threadIdx.x == 0) ctl->it += 1;
}
// uncentred power iteration: stop after the residual reaches 1e-8 (or mu = 0), at most 16 blocks
__global__ void ctl_u_init_kernel(EigCtl* ctl) {
  if (threadIdx.x == 0) { ctl->blocks_u = 0; ctl->iters_u = 0; ctl->stop_u = 0; }
}
__global__ void ctl_u_kernel(EigCtl* ctl, const double* __restrict__ diag, cudaGraphConditionalHandle h_u) {
  if (threadIdx.x != 0) return;
  ctl->blocks_u += 1;
  ctl->iters_u += 4;
  if (!(diag[0] > 0.0) || diag[2] <= 1e-8 || ctl->blocks_u >= 16) {
    ctl->stop_u = 1;
    if (h_u) cudaGraphSetConditional(h_u, 0u);
  }
}

}  // namespace

// split-K geometry shared by the plan (workspace) and the launches: as many K slices as fill
// ONE wave of resident CTAs (3 fp32 / 2 fp64 CTAs per SM, smem-bound) — a partial second wave
// would double the kernel's time
// CTAs of the split-K GEMM resident at once: 3 (fp32) / 2 (fp64) per SM for the register-tiled
// row blocks, and for the 32-row blocks of small m (c1, c2: a 16 MB G32 in L2, every product
// latency-bound) as many as shared memory holds, up to 8 per SM
int64_t gemm_resident(int num_sms, bool fp32, int BM, int p) {
  if (!fp32 && BM == 128) {  // fp64 128-row register tiles (p <= 48): shared memory allows one per SM
    const int64_t sm = (int64_t)kSkStages * (kSkBK * BM + kSkBK * p) * 8 + 2064;
    return (int64_t)num_sms * std::max<int64_t>(1, (228 * 1024) / sm);
  }
  if (!(fp32 && BM <= 32)) return (int64_t)num_sms * (fp32 ? 3 : 2);
  const int64_t sm = (int64_t)kSkStages * (kSkBK * BM + kSkBK * p) * 4 + 2064;  // + static + reserved
  return (int64_t)num_sms * std::max<int64_t>(3, std::min<int64_t>(8, (228 * 1024) / sm));
}
void gemm_geometry(int64_t m, int64_t m_pad, int p, int num_sms, bool fp32, int* BM, int* KS, int* RB, int* KT) {
  *KT = (int)ceil_div(m, kSkBK);
  const int64_t want = (int64_t)num_sms * (fp32 ? 3 : 2);  // resident CTAs (smem-bound)
  // the largest row block (register tile) that still leaves every CTA >= 8 K tiles of work:
  // small m (c1, c2) takes 32-row blocks so the grid fills without slivers of K per CTA
  // fp64 (the Rayleigh-Ritz product): 8 x 6 register tiles for p <= 48 halve the shared-memory
  // operand bytes per DFMA (a 4 x 6 tile needs ~1.7x the SM's shared-memory bandwidth)
  const int big = ((fp32 && p <= 64) || (!fp32 && p <= 48 && m >= 4096)) ? 128 : 64;
  *BM = big;
  for (int bm = big; bm >= 32; bm /= 2) {
    *BM = bm;
    const int64_t rb = m_pad / bm;
    if (std::min<int64_t>(want / rb, *KT) * 8 <= *KT || want / rb < 1) break;
  }
  *RB = (int)(m_pad / *BM);
  // 32-row blocks: more CTAs in flight and >= 4 K tiles each (the K loop is latency-bound there)
  const bool small = fp32 && *BM <= 32;
  const int64_t res = gemm_resident(num_sms, fp32, *BM, p);
  *KS = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(res / *RB, *KT), std::max<int64_t>(1, *KT / (small ? 4 : 8))));
}
size_t gemm_part_bytes(int64_t m, int64_t m_pad, int p, int num_sms) {
  size_t best = 0;
  for (int f = 0; f < 2; ++f) {  // RB x KS <= the resident-CTA count for any row range (gemm_launch)
    int BM, KS, RB, KT;
    gemm_geometry(m, m_pad, p, num_sms, f == 0, &BM, &KS, &RB, &KT);
    const int64_t want = gemm_resident(num_sms, f == 0, BM, p);
    best = std::max(best, (size_t)std::max<int64_t>(want, (int64_t)RB * KS) * BM * p *
                              (f == 0 ? sizeof(float) : sizeof(double)));
  }
  return (size_t)round_up((int64_t)best, 256) + sizeof(unsigned) * (size_t)(m_pad / 32 + 1);  // partials + tickets
}

namespace {

// Y = G In (fp64 G, fp64 math) or Y = G32 In32 (fp32); Y fp64 (+ optional fp32 mirror)
// rows [r0, r1) of Y only (multiples of 128; all rows when r1 <= r0): the distributed eigensolve
template <typename T, int NR, int NC>
avd_status gemm_launch(Ctx* c, const T* Gm, const T* In, double* Y, float* Y32, const int* skip, int64_t r0 = 0,
                       int64_t r1 = 0) {
  int BM, KS, RB, KT;
  const int p = 8 * NC;
  gemm_geometry(c->cfg.m, c->m_pad, p, c->num_sms, sizeof(T) == 4, &BM, &KS, &RB, &KT);
  if (BM != 16 * NR) { set_error("gemm geometry mismatch"); return AVD_EINVAL; }
  int rb0 = 0;
  if (r1 > r0) {  // a row range: fewer row blocks, more K slices (same partial-buffer bound)
    rb0 = (int)(r0 / BM);
    RB = (int)ceil_div(r1 - r0, BM);
    const int64_t want = gemm_resident(c->num_sms, sizeof(T) == 4, BM, p);
    KS = (int)std::max<int64_t>(1, std::min<int64_t>(want / RB, KT));
  }
  const int sm = kSkStages * (kSkBK * BM + kSkBK * p) * (int)sizeof(T);
  AVD_CUDA(smem_attr(gemm_kernel<T, NR, NC>, sm));
  const size_t pb = gemm_part_bytes(c->cfg.m, c->m_pad, c->p, c->num_sms);
  T* part = reinterpret_cast<T*>(c->gemm_part);
  unsigned* tickets = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(c->gemm_part) + pb -
                                                  sizeof(unsigned) * (size_t)(c->m_pad / 32 + 1));
  gemm_kernel<T, NR, NC><<<RB * KS, kSkThreads, sm, c->stream>>>(Gm, c->m_pad, In, c->cfg.m, KT, KS, part, tickets, Y,
                                                                 Y32, skip, rb0);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

int gemm_bm(const Ctx* c, bool fp32) {
  int BM, KS, RB, KT;
  gemm_geometry(c->cfg.m, c->m_pad, c->p, c->num_sms, fp32, &BM, &KS, &RB, &KT);
  return BM;
}
avd_status gemm64(Ctx* c, const double* In, double* Y, float* Y32, int64_t r0 = 0, int64_t r1 = 0,
                  const int* skip = nullptr) {
  const int bm = gemm_bm(c, false);
  switch (c->p / 16) {
#define CASE(PC)                                                                                        \
  case PC:                                                                                              \
    if constexpr (PC <= 3) if (bm == 128) return gemm_launch<double, 8, 2 * PC>(c, c->G, In, Y, Y32, skip, r0, r1); \
    return bm == 64 ? gemm_launch<double, 4, 2 * PC>(c, c->G, In, Y, Y32, skip, r0, r1)                   \
                    : gemm_launch<double, 2, 2 * PC>(c, c->G, In, Y, Y32, skip, r0, r1);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
  set_error("unsupported p");
  return AVD_EINVAL;
}
avd_status gemm32(Ctx* c, const float* In, double* Y, float* Y32, const int* skip = nullptr, int64_t r0 = 0,
                  int64_t r1 = 0) {
  const int bm = gemm_bm(c, true);
  switch (c->p / 16) {
#define CASE(PC)                                                                                        \
  case PC:                                                                                              \
    if (bm == 128 && PC <= 4) return gemm_launch<float, 8, 2 * PC>(c, c->G32, In, Y, Y32, skip, r0, r1);   \
    if (bm == 64) return gemm_launch<float, 4, 2 * PC>(c, c->G32, In, Y, Y32, skip, r0, r1);                \
    return gemm_launch<float, 2, 2 * PC>(c, c->G32, In, Y, Y32, skip, r0, r1);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
#undef CASE
  }
  set_error("unsupported p");
  return AVD_EINVAL;
}

template <int MODE>
avd_status atb_fused(Ctx* c, const double* A, const double* B, double* out0, double* out1, int* ibad, int* stats,
                     const int* gate = nullptr, int max_sweeps = 40, const int* msw = nullptr) {
  const int p = c->p;
  const int n_red = (int)ceil_div(c->cfg.m, kRedRows);
  const int chunk = p <= 48 ? kRedRows : 64;
  const size_t sm = std::max<size_t>(2 * (size_t)chunk * p, (size_t)p * (p + 1) + (size_t)p * p) * sizeof(double);
  switch (p / 16) {
#define CASE(PC)                                                                                                \
  case PC:                                                                                                      \
    AVD_CUDA(smem_attr(atb_fused_kernel<MODE, PC>, (int)sm)); \
    atb_fused_kernel<MODE, PC><<<n_red, RedCfg<PC>::threads, sm, c->stream>>>(A, B, c->cfg.m, c->red_part, c->ticket, out0, out1,  \
                                                              ibad, stats, gate, max_sweeps, msw);              \
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
// kernels exit at once.  itp: device iteration counter mixed into the re-draw seed.
avd_status orth(Ctx* c, const double* Y, uint32_t seed, const int* itp) {
  int* bad = reinterpret_cast<int*>(c->resid + c->p);
  int* need2 = bad + c->p;
  const int p = c->p;
  for (int pass = 0; pass < 2; ++pass) {
    const double* src = pass == 0 ? Y : c->Q;
    const int* gate = pass == 0 ? nullptr : need2;
    AVD_TRY(atb_fused<1>(c, src, src, c->W, c->H, bad, pass == 0 ? need2 : nullptr, gate));  // R -> W, 1/R_jj -> H
    AVD_TRY(trsm(c, src, c->W, c->H, bad, gate));                   // in place allowed (row-wise)
    if (pass == 0) {
      rand_fill_kernel<<<(unsigned)ceil_div(c->cfg.m * p, 256), 256, 0, c->stream>>>(c->Q, c->Q32, c->cfg.m, p, seed,
                                                                                     bad, itp);
      AVD_LAUNCHED(c);
    }
  }
  return AVD_OK;
}

uint32_t eig_seed(const Ctx* c) { return (uint32_t)(c->cfg.seed ^ (c->cfg.seed >> 32)) * 2654435761u + 12345u; }

// Capture the launches `fn` makes on c->stream into `g` (an empty conditional body graph); the
// host-side launch counter is restored (graph kernels are counted per executed iteration) and the
// number of kernels captured is returned in *nodes.
template <typename F>
avd_status capture_into(Ctx* c, cudaGraph_t g, int* nodes, F&& fn) {
  cudaStream_t user = c->stream;
  c->stream = c->cap_stream;
  const int64_t l0 = c->launches;
  avd_status st = AVD_OK;
  cudaError_t e = cudaStreamBeginCaptureToGraph(c->cap_stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    st = fn();
    cudaGraph_t out = g;
    const cudaError_t e2 = cudaStreamEndCapture(c->cap_stream, &out);
    if (st == AVD_OK && e2 != cudaSuccess) e = e2;
  }
  c->stream = user;
  *nodes = (int)(c->launches - l0);
  c->launches = l0;
  if (st != AVD_OK) return st;
  if (e != cudaSuccess) {
    set_error(std::string("graph capture failed: ") + cudaGetErrorString(e));
    return AVD_ECUDA;
  }
  return AVD_OK;
}

avd_status add_cond(cudaGraph_t g, const cudaGraphNode_t* deps, size_t ndeps, cudaGraphConditionalHandle h,
                    cudaGraphConditionalNodeType type, cudaGraphNode_t* node, cudaGraph_t* body) {
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = type;
  np.conditional.size = 1;
  AVD_CUDA(cudaGraphAddNode(node, g, deps, ndeps, &np));
  *body = np.conditional.phGraph_out[0];
  return AVD_OK;
}

// Loop bodies (graph bodies, or launched one by one by the host-driven profiling mode)
avd_status enqueue_rr(Ctx* c, cudaGraphConditionalHandle h_loop, cudaGraphConditionalHandle h_pow) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  int* jstats = reinterpret_cast<int*>(c->theta + p);
  if (c->gram_free) {
    AVD_TRY(gf_product(c, c->Q, c->Y, nullptr, nullptr));  // Y = Xhat^T (Xhat Q)
  } else {
    AVD_TRY(gemm64(c, c->Q, c->Y, nullptr, 0, 0, &ctl->rr_fast));  // Y = G Q (exact G, fp64)
    // intermediate checks: the power steps' product (gated on the device)
    if (eig_i8_enabled(c)) AVD_TRY(gemm_i8(c, c->Q, c->Y, nullptr, &ctl->rr_exact, 0, 0));
    else AVD_TRY(gemm32(c, c->Q32, c->Y, nullptr, &ctl->rr_exact));
  }
  AVD_TRY(atb_fused<2>(c, c->Q, c->Y, c->W, c->theta, nullptr, &ctl->last_sweeps, nullptr, 40, &ctl->msw));
  AVD_TRY(matpp(c, c->Y, c->Z, c->Z32, c->Q, c->U, nullptr, c->W));  // Z = Y W, U = Q W (Ritz vectors)
  resid_kernel<<<k, 256, 0, c->stream>>>(c->Z, c->U, c->theta, m, p, c->resid);
  AVD_LAUNCHED(c);
  ctl_rr_kernel<<<1, 32, 0, c->stream>>>(ctl, c->theta, c->resid, p, k, jstats, h_loop, h_pow);
  AVD_LAUNCHED(c);
  return AVD_OK;
}
avd_status enqueue_pow(Ctx* c) {
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  if (c->gram_free) {  // Gram-free: G Q = Xhat^T (Xhat Q), two streaming passes (k_gramfree.cu)
    AVD_TRY(gf_product(c, c->Q, c->Z, c->Z32, &ctl->rr_now));
    AVD_TRY(gf_product(c, c->Z, c->Y, nullptr, nullptr));
  } else if (eig_i8_enabled(c)) {  // int8 tensor-core products (k_eig_i8.cu)
    AVD_TRY(gemm_i8(c, c->Q, c->Z, c->Z32, &ctl->rr_now, 0, 0));  // Z = G Q (a check already made Z = G U)
    AVD_TRY(gemm_i8(c, c->Z, c->Y, nullptr, nullptr, 0, 0));       // Y = G Z = G^2 Q
  } else {
    AVD_TRY(gemm32(c, c->Q32, c->Z, c->Z32, &ctl->rr_now));  // Z = G Q (a check already made Z = G U)
    AVD_TRY(gemm32(c, c->Z32, c->Y, nullptr));                // Y = G Z = G^2 Q
  }
  AVD_TRY(orth(c, c->Y, eig_seed(c), &ctl->it));
  ctl_end_kernel<<<1, 32, 0, c->stream>>>(ctl);
  AVD_LAUNCHED(c);
  return AVD_OK;
}
avd_status enqueue_unc(Ctx* c, cudaGraphConditionalHandle h_u) {
  const int64_t m = c->cfg.m;
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  double* q = c->diag + 4;
  double* y = q + c->m_pad;
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), 4LL * c->num_sms);
  const double lg = (double)c->cfg.l_global;
  for (int t = 0; t < 4; ++t) {
    power_u_kernel<<<grid, 256, 0, c->stream>>>(c->G32, c->m_pad, c->mu, m, lg, (t & 1) ? y : q, (t & 1) ? q : y);
    AVD_LAUNCHED(c);
  }
  power_u_kernel<<<grid, 256, 0, c->stream>>>(c->G32, c->m_pad, c->mu, m, lg, q, y);
  AVD_LAUNCHED(c);
  power_u_stats_kernel<<<1, 256, 0, c->stream>>>(c->mu, m, q, y, c->diag);
  AVD_LAUNCHED(c);
  ctl_u_kernel<<<1, 32, 0, c->stream>>>(ctl, c->diag, h_u);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

// The eigensolver loop as one graph (built once per context; every pointer it uses is fixed):
//   WHILE(loop) { ctl_begin; IF(rr) { Y = G Q (fp64); Jacobi RR; Z = Y W, U = Q W; residuals;
//                 ctl_rr }; IF(pow) { Z = G32 Q32 (skipped after a check); Y = G32 Z32;
//                 Q = orth(Y); ctl_end } }
avd_status build_eig_graph(Ctx* c) {
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  cudaGraph_t g;
  AVD_CUDA(cudaGraphCreate(&g, 0));
  avd_status st = [&]() -> avd_status {
    cudaGraphConditionalHandle h_loop;
    AVD_CUDA(cudaGraphConditionalHandleCreate(&h_loop, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t wnode;
    cudaGraph_t body;
    AVD_TRY(add_cond(g, nullptr, 0, h_loop, cudaGraphCondTypeWhile, &wnode, &body));
    cudaGraphConditionalHandle h_rr, h_pow;
    AVD_CUDA(cudaGraphConditionalHandleCreate(&h_rr, body, 0, 0));
    AVD_CUDA(cudaGraphConditionalHandleCreate(&h_pow, body, 0, 0));
    int nb = 0;
    AVD_TRY(capture_into(c, body, &nb, [&]() -> avd_status {
      ctl_begin_kernel<<<1, 32, 0, c->stream>>>(ctl, h_rr, h_pow);
      AVD_LAUNCHED(c);
      return AVD_OK;
    }));
    cudaGraphNode_t begin_node;
    size_t n1 = 1;
    AVD_CUDA(cudaGraphGetNodes(body, &begin_node, &n1));
    cudaGraphNode_t rr_node, pow_node;
    cudaGraph_t rr_body, pow_body;
    AVD_TRY(add_cond(body, &begin_node, 1, h_rr, cudaGraphCondTypeIf, &rr_node, &rr_body));
    AVD_TRY(add_cond(body, &rr_node, 1, h_pow, cudaGraphCondTypeIf, &pow_node, &pow_body));
    AVD_TRY(capture_into(c, rr_body, &c->n_rr_nodes, [&]() { return enqueue_rr(c, h_loop, h_pow); }));
    AVD_TRY(capture_into(c, pow_body, &c->n_pow_nodes, [&]() { return enqueue_pow(c); }));
    c->n_begin_nodes = nb;
    AVD_CUDA(cudaGraphInstantiate(&c->eig_exec, g, 0));
    return AVD_OK;
  }();
  cudaGraphDestroy(g);
  return st;
}

// Uncentred power iteration (mean-bias diagnostics) as one graph on the side stream:
//   WHILE(u) { 4 power steps (q -> y -> q -> y -> q); y = Gu q; stats(q, y); ctl_u }
avd_status build_unc_graph(Ctx* c) {
  cudaGraph_t g;
  AVD_CUDA(cudaGraphCreate(&g, 0));
  avd_status st = [&]() -> avd_status {
    cudaGraphConditionalHandle h_u;
    AVD_CUDA(cudaGraphConditionalHandleCreate(&h_u, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t wnode;
    cudaGraph_t body;
    AVD_TRY(add_cond(g, nullptr, 0, h_u, cudaGraphCondTypeWhile, &wnode, &body));
    AVD_TRY(capture_into(c, body, &c->n_u_nodes, [&]() { return enqueue_unc(c, h_u); }));
    AVD_CUDA(cudaGraphInstantiate(&c->unc_exec, g, 0));
    return AVD_OK;
  }();
  cudaGraphDestroy(g);
  return st;
}

// AVD_EIG_NOGRAPH=1: the same loop bodies launched one by one by the host with a synchronisation
// per decision (profiling: ncu sees every kernel; numerically identical)
bool eig_nograph_env() {
  static const bool v = [] { const char* e = std::getenv("AVD_EIG_NOGRAPH"); return e && e[0] == '1'; }();
  return v;
}

// The Gram-free products are templated on the digit count, which the automatic
// escalation can change after the graph was captured, and each costs two passes over the operand,
// so their loop is host-driven (one synchronisation per decision is noise next to a product).
bool eig_nograph(const Ctx* c) {
  return eig_nograph_env() || (c->cfg.flags & AVD_FLAG_EIG_HOST_LOOP) != 0 || c->gram_free;
}

avd_status ensure_graphs(Ctx* c) {
  if (!c->side_stream) AVD_CUDA(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
  if (c->eig_exec || eig_nograph(c)) return AVD_OK;
  if (!c->cap_stream) AVD_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  if (!c->ev_fork) AVD_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  if (!c->ev_join) AVD_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  AVD_TRY(build_unc_graph(c));
  return build_eig_graph(c);
}

}  // namespace

avd_status launch_trace(Ctx* c) {
  trace_kernel<<<1, 1024, 0, c->stream>>>(c->G, c->cfg.m, c->m_pad, c->ysq, c->mu0, (double)c->cfg.l_global, c->stats,
                                          c->trace, c->gmax);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

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

// A-posteriori bound of the Gram operand's quantisation error (DESIGN.md §8 "Gram precision").
// The operand is q_ia = y_ia + e_ia, y = (x - mu0) 2^shift, with dithered rounding errors e that
// are zero-mean, independent and var e <= 1/4 (exactly 0 for a column whose every entry is on the
// grid: qerr_a = 0).  The diagonal of G is the exact centred energy (fp64 sums of the fused pass),
// the off-diagonal is E_ab = d_a d_b sum_i (e_ia xc_ib + xc_ia e_ib) + O(e^2) (d_a = 2^-shift_a),
// so to first order, with X~ v_r = sigma_r u_r and X~^T u_r = sigma_r v_r,
//   d lambda_r = v_r^T E v_r = 2 sum_ia d_a v_ra e_ia (sigma_r u_ri - v_ra xc_ia),
//   var <= t_r = sum_a d_a^2 v_ra^2 (lambda_r (1 - 2 v_ra^2) + v_ra^2 G_aa)      (fin kernels)
//   d E_spike = sum_r d lambda_r = 2 sum_ia d_a e_ia (S_ia - P_aa xc_ia),  P = V_k V_k^T,
//   var <= sum_a d_a^2 (w_a (1 - 2 P_aa) + P_aa^2 G_aa),  w_a = sum_r lambda_r v_ra^2 (fin kernels)
// (S the spike matrix).  A column carried by one massive entry (v_r ~ e_a) drops out, as it
// should: its diagonal is exact.  E_tail = tr(G) - E_spike inherits d E_spike (tr(G) is exact up
// to the fp32 rounding of y, counted as 1e-9 tr(G)).  At 5 sigma:
//   prec_sigma = max_r 2.5 sqrt(t_r) / lambda_r  (relative error of sigma_r = d lambda / 2 lambda)
//   prec_share = max(5 std(d E_spike) / E_spike, (5 std(d E_spike) + 1e-9 tr(G)) / E_tail)
// The automatic digit rule raises the operand to 3 digits when prec_sigma > 5e-5 or
// prec_share > 5e-6 (half the north-star tolerances 1e-4 / 1e-5).
// h: the pinned copy of [theta (p) | t_r (k) | var(d E_spike) | tr(G)].
static void precision_bound(Ctx* c, const double* theta, const double* h) {
  const int k = c->k;
  double ps = 0.0, e_spike = 0.0;
  for (int r = 0; r < k; ++r) {
    const double lam = std::max(theta[r], 0.0);
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
}

namespace {
// start block: Q_0 = orth(random), loop state reset (shared by every mode of the solve)
avd_status eig_prologue(Ctx* c) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  const uint32_t seed = eig_seed(c);
  const int max_it = std::max(2, c->cfg.max_iters > 0 ? c->cfg.max_iters : 200);
  const double tol = c->cfg.eig_tol > 0 ? c->cfg.eig_tol : 1e-6;  // V angle <~ tol * lambda_1 / gap_k
  int* jstats = reinterpret_cast<int*>(c->theta + p);  // [16] sweeps per RR solve
  AVD_CUDA(cudaMemsetAsync(jstats, 0, 16 * sizeof(int), c->stream));
  AVD_CUDA(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned), c->stream));
  {  // split-K tickets (re-armed by every launch; cleared here once per solve)
    const size_t pb = gemm_part_bytes(m, c->m_pad, p, c->num_sms), tb = sizeof(unsigned) * (size_t)(c->m_pad / 32 + 1);
    AVD_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(c->gemm_part) + pb - tb, 0, tb, c->stream));
  }
  ctl_init_kernel<<<1, 32, 0, c->stream>>>(ctl, max_it, tol, k, p);
  AVD_LAUNCHED(c);
  if (eig_i8_enabled(c)) AVD_TRY(eig_i8_prepare(c));  // G in digits for the power steps
  rand_fill_kernel<<<(unsigned)ceil_div(m * p, 256), 256, 0, c->stream>>>(c->Z, nullptr, m, p, seed, nullptr, nullptr);
  AVD_LAUNCHED(c);
  return orth(c, c->Z, seed + 1, nullptr);
}

// final vectors, sigma, the precision-bound sums; one synchronisation; fills the host fields
avd_status eig_epilogue(Ctx* c, bool count_graph) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  const int nb = (int)ceil_div(m, kFinThreads);
  fin_part_kernel<<<nb, kFinThreads, 0, c->stream>>>(c->U, c->theta, m, p, k, c->shift, c->qerr, c->G, c->m_pad,
                                                      c->red_part);
  AVD_LAUNCHED(c);
  fin_final_kernel<<<k + 1, 32, 0, c->stream>>>(c->red_part, nb, k, c->theta, c->U, p, c->sigma, c->H, c->prec);
  AVD_LAUNCHED(c);
  fin_write_kernel<<<(unsigned)ceil_div(m * c->k_pad, 256), 256, 0, c->stream>>>(c->U, c->H, m, p, k, c->k_pad, c->V,
                                                                                 c->V32);
  AVD_LAUNCHED(c);
  // one pinned copy: theta [p] | t_r [k], var(d E_spike) | tr(G) | ctl
  double* h = c->eig_host + 4 * kMaxP;
  EigCtl* hc = reinterpret_cast<EigCtl*>(c->eig_host + 6 * kMaxP);
  static_assert(6 * kMaxP + kEigCtlBytes / 8 <= kHostScratch, "pinned scratch too small");
  AVD_CUDA(cudaMemcpyAsync(h, c->theta, sizeof(double) * p, cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaMemcpyAsync(h + p, c->prec, sizeof(double) * (k + 1), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaMemcpyAsync(h + p + k + 1, c->trace, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(EigCtl), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  const int it = hc->it, rr = hc->rr_count;
  if (count_graph)
    c->launches += (int64_t)c->n_begin_nodes * it + (int64_t)c->n_rr_nodes * rr + (int64_t)c->n_pow_nodes * (it - 1);
  c->iters = std::min(it, hc->max_it);
  c->rr_count = rr;
  c->max_resid = hc->maxres;
  c->sigma_next = (k < p) ? std::sqrt(std::max(h[k], 0.0)) : 0.0;
  for (int r = 0; r < p; ++r) c->eig_host[r] = h[r];  // Ritz values of the last check
  precision_bound(c, h, h + p);
  return hc->conv ? AVD_OK : AVD_ENOCONV;
}

// host-driven loop (profiling mode, and the distributed solve): the same kernels and the same
// device control decisions as the graph, one synchronisation per decision
template <typename RR, typename POW>
avd_status eig_host_loop(Ctx* c, RR&& rr_body, POW&& pow_body) {
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  EigCtl* hc = reinterpret_cast<EigCtl*>(c->eig_host + 6 * kMaxP);
  for (;;) {
    ctl_begin_kernel<<<1, 32, 0, c->stream>>>(ctl, 0, 0);
    AVD_LAUNCHED(c);
    AVD_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(EigCtl), cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));
    const bool rr = hc->rr_now != 0;
    if (rr) {
      AVD_TRY(rr_body());
      AVD_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(EigCtl), cudaMemcpyDeviceToHost, c->stream));
      AVD_CUDA(cudaStreamSynchronize(c->stream));
      if (hc->stop) break;
    }
    AVD_TRY(pow_body(rr));
  }
  return AVD_OK;
}
}  // namespace

// Subspace iteration (device-resident): power steps Q <- orth(G^2 Q) in fp32; a Rayleigh-Ritz
// check (fp64) runs on a schedule predicted from the observed residual decay (at most every 8
// steps, always on the last one), so the p x p Jacobi runs ~2 times per solve.  The whole loop is
// one graph launch (build_eig_graph); the host synchronises once, after the final vectors and the
// precision bound, and meanwhile the uncentred power iteration runs on the side stream.
avd_status run_eig(Ctx* c) {
  AVD_TRY(ensure_graphs(c));
  AVD_TRY(eig_prologue(c));
  const bool nograph = eig_nograph(c);
  if (nograph) {
    AVD_TRY(eig_host_loop(c, [&]() { return enqueue_rr(c, 0, 0); }, [&](bool) { return enqueue_pow(c); }));
  } else {
    AVD_CUDA(cudaGraphLaunch(c->eig_exec, c->stream));
  }
  return eig_epilogue(c, !nograph);
}

// Y = G In for the context's current Gram operand (avd_gram_product): the formed fp64 G, or with
// AVD_FLAG_GRAM_FREE the two streaming passes Xhat^T (Xhat In)
avd_status gram_product(Ctx* c, const double* In, double* Y) {
  if (c->gram_free) {
    AVD_TRY(gf_prepare(c));
    AVD_TRY(gf_product(c, In, Y, nullptr, nullptr));
    return AVD_OK;
  }
  return gemm64(c, In, Y, nullptr);
}

// Distributed eigensolve: every rank holds the exchanged G, and each G Q product
// is split by rows — rank r computes the rows [r0, r1) of its share of the 128-row blocks; the
// other rows of the product are zero, so a SUM exchange of the whole m x p block is the
// all-gather (EIGZ: the fp32 Z = G Q of a power step, EIGY: the fp64 Y = G Z or the Rayleigh-Ritz
// product).  The p x p work, the orthonormalisation and the control decisions are replicated
// (identical inputs -> identical results on every rank).  Exchanges per power step: 2 (1.2 MB
// at c4), per check: 1.
avd_status run_eig_dist(Ctx* c, int rank, avd_exchange_fn fn, void* user) {
  const int world = c->cfg.world;
  if (world <= 1 || !fn) return run_eig(c);
  if (rank < 0 || rank >= world) { set_error("bad rank"); return AVD_EINVAL; }
  AVD_TRY(ensure_graphs(c));
  const int64_t m = c->cfg.m;
  const int p = c->p;
  const int64_t U = c->m_pad / 128;
  const int64_t r0 = 128 * (U * rank / world), r1 = 128 * (U * (rank + 1) / world);
  EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
  auto exch = [&](int which, void* ptr, int dt) -> avd_status {
    if (fn(which, ptr, dt, AVD_OP_SUM, (size_t)(m * p), user) != 0) {
      set_error("exchange callback failed (buffer " + std::to_string(which) + ")");
      return AVD_EEXCHANGE;
    }
    return AVD_OK;
  };
  AVD_TRY(eig_prologue(c));
  // (r1 <= r0 when there are more ranks than row blocks: the rank contributes zeros)
  auto rows_y = [&](auto&& gemm) -> avd_status {
    AVD_CUDA(cudaMemsetAsync(c->Y, 0, sizeof(double) * m * p, c->stream));
    if (r1 > r0) AVD_TRY(gemm());
    return exch(AVD_BUF_EIGY, c->Y, AVD_DT_F64);
  };
  auto rr_body = [&]() -> avd_status {
    AVD_TRY(rows_y([&]() { return gemm64(c, c->Q, c->Y, nullptr, r0, r1); }));  // Y = G Q (fp64)
    int* jstats = reinterpret_cast<int*>(c->theta + p);
    AVD_TRY(atb_fused<2>(c, c->Q, c->Y, c->W, c->theta, nullptr, &ctl->last_sweeps, nullptr, 40, &ctl->msw));
    AVD_TRY(matpp(c, c->Y, c->Z, c->Z32, c->Q, c->U, nullptr, c->W));
    resid_kernel<<<c->k, 256, 0, c->stream>>>(c->Z, c->U, c->theta, m, p, c->resid);
    AVD_LAUNCHED(c);
    ctl_rr_kernel<<<1, 32, 0, c->stream>>>(ctl, c->theta, c->resid, p, c->k, jstats, 0, 0);
    AVD_LAUNCHED(c);
    return AVD_OK;
  };
  const bool i8 = eig_i8_enabled(c);
  auto pow_body = [&](bool after_rr) -> avd_status {
    if (!after_rr) {  // Z = G Q (a check already made Z = G U on every rank)
      AVD_CUDA(cudaMemsetAsync(c->Z, 0, sizeof(double) * m * p, c->stream));
      if (r1 > r0) {
        if (i8) AVD_TRY(gemm_i8(c, c->Q, c->Z, nullptr, nullptr, r0, r1));
        else AVD_TRY(gemm32(c, c->Q32, c->Z, nullptr, nullptr, r0, r1));
      }
      AVD_TRY(exch(AVD_BUF_EIGZ, c->Z, AVD_DT_F64));
      if (!i8) {  // the SIMT product reads the fp32 mirror of the exchanged Z
        f64_to_f32_kernel<<<(unsigned)ceil_div(m * p, 256), 256, 0, c->stream>>>(c->Z, c->Z32, m * p);
        AVD_LAUNCHED(c);
      }
    }
    AVD_TRY(rows_y([&]() {  // Y = G Z
      return i8 ? gemm_i8(c, c->Z, c->Y, nullptr, nullptr, r0, r1) : gemm32(c, c->Z32, c->Y, nullptr, nullptr, r0, r1);
    }));
    AVD_TRY(orth(c, c->Y, eig_seed(c), &ctl->it));
    ctl_end_kernel<<<1, 32, 0, c->stream>>>(ctl);
    AVD_LAUNCHED(c);
    return AVD_OK;
  };
  AVD_TRY(eig_host_loop(c, rr_body, pow_body));
  return eig_epilogue(c, false);
}

// Mean-bias diagnostics on the replicated G and mu (no exchange): power iteration on the uncentred
// Gram from q_0 = mu_hat (already aligned when the mean dominates), in blocks of
// 4 steps until the residual is <= 1e-8 (at most 64 steps), as one graph on the side stream,
// concurrent with the subspace iteration (both only read G32 and mu).  diag[0] = ||mu||,
// diag[1] = lambda_1 (Rayleigh quotient), diag[2] = residual, diag[3] = mu . q; the report stage
// turns them into sigma1_u = sqrt(lambda_1), alpha1 = |mu . v_1| (= (sigma_1 / l) u_1^T 1,
// PAPER.md:559-561), cos_mu_v1 = alpha1 / ||mu||.
avd_status launch_uncentred(Ctx* c) {
  AVD_TRY(ensure_graphs(c));
  if (eig_nograph(c)) {
    EigCtl* ctl = reinterpret_cast<EigCtl*>(c->eig_ctl);
    EigCtl* hc = reinterpret_cast<EigCtl*>(c->eig_host + 6 * kMaxP);
    ctl_u_init_kernel<<<1, 32, 0, c->stream>>>(ctl);
    AVD_LAUNCHED(c);
    mu_norm_kernel<<<1, 256, 0, c->stream>>>(c->mu, c->cfg.m, c->m_pad, c->diag);
    AVD_LAUNCHED(c);
    for (;;) {
      AVD_TRY(enqueue_unc(c, 0));
      AVD_CUDA(cudaMemcpyAsync(hc, ctl, sizeof(EigCtl), cudaMemcpyDeviceToHost, c->stream));
      AVD_CUDA(cudaStreamSynchronize(c->stream));
      if (hc->stop_u) break;
    }
    c->launches -= (int64_t)c->n_u_nodes * hc->blocks_u;  // the report adds them for the graph mode
    return AVD_OK;
  }
  // AVD_UNC_SERIAL=1 (diagnostics): the uncentred loop on the context's own stream
  static const bool serial = [] { const char* e = std::getenv("AVD_UNC_SERIAL"); return e && e[0] == '1'; }();
  cudaStream_t side = serial ? c->stream : c->side_stream;
  AVD_CUDA(cudaEventRecord(c->ev_fork, c->stream));
  AVD_CUDA(cudaStreamWaitEvent(side, c->ev_fork, 0));
  cudaStream_t user = c->stream;
  c->stream = side;
  ctl_u_init_kernel<<<1, 32, 0, c->stream>>>(reinterpret_cast<EigCtl*>(c->eig_ctl));
  mu_norm_kernel<<<1, 256, 0, c->stream>>>(c->mu, c->cfg.m, c->m_pad, c->diag);
  c->stream = user;
  AVD_LAUNCHED(c);
  AVD_LAUNCHED(c);
  AVD_CUDA(cudaGraphLaunch(c->unc_exec, side));
  AVD_CUDA(cudaEventRecord(c->ev_join, side));
  return AVD_OK;
}
avd_status join_uncentred(Ctx* c) {
  if (eig_nograph(c)) return AVD_OK;
  AVD_CUDA(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return AVD_OK;
}

// Uncentred top-k: the top k right singular pairs of the
// UNCENTRED X, i.e. eigenpairs of X^T X = G + l mu mu^T, and alpha_i = mu . v_i (the expansion
// mu = sum_i alpha_i v_i, |.|: sign-free), by subspace iteration on G + l mu mu^T (fp64 products
// with the exact G plus the rank-one term) from the start block [mu_hat, U_{p-1}] — already close
// to the answer — with a Rayleigh-Ritz check after every step, until the top-k residuals are
// <= tol (at most 30 steps).  Writes out[0..k) = sigma_i, out[k..2k) = alpha_i.  Optional
// (AVD_FLAG_MEAN_TOPK): about one eigensolve of extra work.  Reuses the solve's scratch (V_k and
// sigma_k are already final).
avd_status run_uncentred_topk(Ctx* c, double* out) {
  const int64_t m = c->cfg.m;
  const int p = c->p, k = c->k;
  const double l = (double)c->cfg.l_global;
  const double tol = c->cfg.eig_tol > 0 ? c->cfg.eig_tol : 1e-6;
  double* w = c->resid + 3 * p;  // [p] scratch (resid holds 2p + flags)
  int* sweeps = reinterpret_cast<int*>(c->theta + p) + 15;
  const unsigned g = (unsigned)ceil_div(m * p, 256);
  unc_start_kernel<<<g, 256, 0, c->stream>>>(c->U, c->diag + 4, m, p, c->Z);
  AVD_LAUNCHED(c);
  AVD_TRY(orth(c, c->Z, eig_seed(c) + 977u, nullptr));
  double* h = c->eig_host + 4 * kMaxP;
  c->iters_uk = 0;
  for (int it = 1; it <= 30; ++it) {
    AVD_TRY(gemm64(c, c->Q, c->Y, nullptr));  // Y = G Q + l mu (mu^T Q)
    mu_dot_cols_kernel<<<p, 32, 0, c->stream>>>(c->mu, c->Q, m, p, w);
    AVD_LAUNCHED(c);
    rank1_kernel<<<g, 256, 0, c->stream>>>(c->Y, c->mu, w, m, p, l);
    AVD_LAUNCHED(c);
    AVD_TRY(atb_fused<2>(c, c->Q, c->Y, c->W, c->theta, nullptr, sweeps, nullptr, 40, nullptr));
    AVD_TRY(matpp(c, c->Y, c->Z, nullptr, c->Q, c->U, nullptr, c->W));  // Z = Gu U, U = Q W
    resid_kernel<<<k, 256, 0, c->stream>>>(c->Z, c->U, c->theta, m, p, c->resid);
    AVD_LAUNCHED(c);
    AVD_CUDA(cudaMemcpyAsync(h, c->resid, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaStreamSynchronize(c->stream));
    double mr = 0.0;
    for (int r = 0; r < k; ++r) mr = std::max(mr, h[r]);
    c->iters_uk = it;
    c->resid_uk = mr;
    if (mr <= tol) break;
    AVD_TRY(orth(c, c->Z, eig_seed(c) + 977u * (uint32_t)it, nullptr));  // Q = orth(Gu U)
  }
  unc_out_kernel<<<k, 32, 0, c->stream>>>(c->U, c->theta, c->mu, m, p, k, out);
  AVD_LAUNCHED(c);
  return AVD_OK;
}

void destroy_graphs(Ctx* c) {
  if (c->eig_exec) cudaGraphExecDestroy(c->eig_exec);
  if (c->unc_exec) cudaGraphExecDestroy(c->unc_exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  c->eig_exec = c->unc_exec = nullptr;
}

}  // namespace avd
