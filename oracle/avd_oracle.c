/*
 * avd_oracle.c — plain, slow, fp64 CPU oracle for the activation outlier-attribution
 * pass of arXiv 2603.10444 ("Mean Bias as the Dominant Source of Activation Outliers",
 * PAPER.md:1-27).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may link, import or execute this
 * file: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may.  It shares no code, header, table or helper with the CUDA library
 * (paper_2603_10444_b200/csrc); the two meet only through the seeded input generator
 * (synth/), which holds none of the method's arithmetic.
 *
 * Every function computes the plain definition in the paper's order and notation:
 *   mu       = (1/l) X^T 1
 *   Xc       = X - 1 mu^T
 *   spike    = truncated rank-k SVD of Xc, k = floor(0.01 m) PAPER.md:11-14
 *              (right singular vectors = eigenvectors of G = Xc^T Xc, sigma^2 = eigenvalues)
 *   tail     = Xc - spike
 *   ||X||^2  = ||M||^2 + ||spike||^2 + ||tail||^2
 *   E_top    = top 0.1% of entries by |X_ij|
 *   rho      = M^2/X^2, spike^2/X^2, tail^2/X^2
 *   cross    = 1 - sum(rho)  ("minor cross-terms")
 * Readings where the paper is silent are DESIGN.md "Readings" R1..R12 (cited inline).
 *
 * Build: gcc -O3 -mavx2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC (oracle/oracle.py).
 * OpenMP is used only across independent outputs or fixed row blocks whose partial sums are
 * added in block order, so no result depends on the thread count.  Scale (SURVEY §8(c) steps
 * 3, 5, 8): the Gram is accumulated from row chunks of Xc (no l x m fp64 copy), the Jacobi
 * eigensolver uses the parallel round-robin ordering, and E_top of large inputs is selected
 * with a bounded heap under the same comparator (equality with the full sort is pinned).
 * Parity: pinned by tests/test_oracle_pins.py (worked example, closed forms of the planted
 * generator, numpy SVD on small inputs, brute-force sort, invariants).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1
#define ORACLE_ENONFINITE 2
#define ORACLE_ENOMEM 6

/* ------------------------------------------------------------------ */
/* 1. feature-wise mean  mu = (1/l) X^T 1               */
/*    Two-pass: s_j summed in row order, then the correction           */
/*    c_j = sum_i (x_ij - mu_j) is added back (R13).         */
/* ------------------------------------------------------------------ */
void oracle_column_mean(const float* X, int64_t l, int64_t m, double* mu) {
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < m; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < l; ++i) s = s + (double)X[i * m + j];
    double mj = s / (double)l;
    double c = 0.0;
    for (int64_t i = 0; i < l; ++i) c = c + ((double)X[i * m + j] - mj);
    mu[j] = mj + c / (double)l;
  }
}

/* 2. centring  Xc = X - 1 mu^T, explicit fp64 copy. */
void oracle_center(const float* X, int64_t l, int64_t m, const double* mu, double* Xc) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < m; ++j) Xc[i * m + j] = (double)X[i * m + j] - mu[j];
}

/* 3. Gram  G = Xc^T Xc  (the right singular vectors of Xc are the eigenvectors of G and
 *    sigma_r^2 its eigenvalues — the SVD of PAPER.md:12-14).  G[a][b] = sum_i Xc[i][a] Xc[i][b],
 *    summed in row order i = 0, 1, ..., l-1 for every entry (b >= a, mirrored: G is symmetric).
 *    The sum is accumulated row by row (G[a][.] += Xc[i][a] Xc[i][.]): the same per-entry order as
 *    a dot product over i, without a transposed copy of Xc.  OpenMP splits the ROWS a of G
 *    (independent outputs); the order of every sum is unchanged by it.                          */
#define ORACLE_GRAM_RB 64  /* rows of Xc held per chunk */
#define ORACLE_GRAM_AB 16  /* rows a of G per task      */
static void gram_chunk(const double* xc, int64_t n, int64_t m, double* G) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t a0 = 0; a0 < m; a0 += ORACLE_GRAM_AB) {
    const int64_t a1 = a0 + ORACLE_GRAM_AB < m ? a0 + ORACLE_GRAM_AB : m;
    for (int64_t r = 0; r < n; ++r) {
      const double* xr = xc + r * m;
      for (int64_t a = a0; a < a1; ++a) {
        const double xa = xr[a];
        double* g = G + a * m;
        for (int64_t b = a; b < m; ++b) g[b] = g[b] + xa * xr[b];
      }
    }
  }
}
static void gram_mirror(int64_t m, double* G) {
#pragma omp parallel for schedule(static)
  for (int64_t a = 0; a < m; ++a)
    for (int64_t b = 0; b < a; ++b) G[a * m + b] = G[b * m + a];
}

void oracle_gram(const double* Xc, int64_t l, int64_t m, double* G) {
  memset(G, 0, sizeof(double) * (size_t)(m * m));
  for (int64_t i0 = 0; i0 < l; i0 += ORACLE_GRAM_RB) {
    const int64_t n = l - i0 < ORACLE_GRAM_RB ? l - i0 : ORACLE_GRAM_RB;
    gram_chunk(Xc + i0 * m, n, m, G);
  }
  gram_mirror(m, G);
}

/* Same Gram straight from the fp32 X: the rows of Xc = X - 1 mu^T are formed in
 * fp64 one chunk at a time (row-blocked Xc, so the l x m fp64 copy never exists — SURVEY §8(c)
 * step 3).  Bit-identical to oracle_gram(oracle_center(X, mu)).                                */
int oracle_gram_x(const float* X, int64_t l, int64_t m, const double* mu, double* G) {
  double* xc = (double*)malloc(sizeof(double) * (size_t)(ORACLE_GRAM_RB * m));
  if (!xc) return ORACLE_ENOMEM;
  memset(G, 0, sizeof(double) * (size_t)(m * m));
  for (int64_t i0 = 0; i0 < l; i0 += ORACLE_GRAM_RB) {
    const int64_t n = l - i0 < ORACLE_GRAM_RB ? l - i0 : ORACLE_GRAM_RB;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r)
      for (int64_t j = 0; j < m; ++j) xc[r * m + j] = (double)X[(i0 + r) * m + j] - mu[j];
    gram_chunk(xc, n, m, G);
  }
  gram_mirror(m, G);
  free(xc);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* 4. Symmetric eigendecomposition of G by Jacobi rotations            */
/*    (Golub & Van Loan, "Matrix Computations", Alg. 8.5.2 sym.schur2  */
/*    for each rotation; parallel ordering of Sec. 8.5.5: every sweep  */
/*    visits all pairs (p, q) in m'-1 steps of m'/2 DISJOINT pairs      */
/*    (round-robin "chess tournament" ordering, m' = m rounded up to   */
/*    even).  Rotations of one step touch disjoint index pairs, so     */
/*    J = prod J_u is applied as A <- J^T A J (rows, then columns) —   */
/*    mathematically the same as applying them one after another.     */
/*    A sweep with no rotation ends the iteration.                     */
/*    On return lam[0..m) is descending (ties by original index),      */
/*    lam_r clamped at 0 is NOT applied here (caller decides), and     */
/*    V[j*m + r] is component j of eigenvector r, with the sign rule   */
/*    "largest |entry| positive, smallest j on ties" (R8).   */
/*    Returns the number of sweeps used.                               */
/* ------------------------------------------------------------------ */
typedef struct { double lam; int64_t idx; } eig_pair;
static int cmp_eig_desc(const void* pa, const void* pb) {
  const eig_pair* a = (const eig_pair*)pa;
  const eig_pair* b = (const eig_pair*)pb;
  if (a->lam > b->lam) return -1;
  if (a->lam < b->lam) return 1;
  return (a->idx < b->idx) ? -1 : (a->idx > b->idx);
}

/* pair u of step s among n (even) indices: index n-1 is fixed, the others rotate */
static void rr_pair(int64_t n, int64_t s, int64_t u, int64_t* p, int64_t* q) {
  int64_t a, b;
  if (u == 0) { a = n - 1; b = s; }
  else { a = (s + u) % (n - 1); b = (s - u + (n - 1)) % (n - 1); }
  *p = a < b ? a : b;
  *q = a < b ? b : a;
}

int oracle_jacobi_eig(const double* G, int64_t m, double* lam, double* V, int max_sweeps) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* W = (double*)malloc(sizeof(double) * (size_t)(m * m)); /* W = V^T: row r = eigvec r */
  const int64_t n = (m % 2 == 0) ? m : m + 1;
  const int64_t half = n / 2;
  int64_t* pp = (int64_t*)malloc(sizeof(int64_t) * (size_t)half);
  int64_t* qq = (int64_t*)malloc(sizeof(int64_t) * (size_t)half);
  double* cc = (double*)malloc(sizeof(double) * (size_t)half);
  double* ss = (double*)malloc(sizeof(double) * (size_t)half);
  if (!A || !W || !pp || !qq || !cc || !ss) {
    free(A); free(W); free(pp); free(qq); free(cc); free(ss);
    return -1;
  }
  memcpy(A, G, sizeof(double) * (size_t)(m * m));
  double fro = 0.0;
  for (int64_t i = 0; i < m * m; ++i) fro = fro + A[i] * A[i];
  fro = sqrt(fro);
  const double abs_floor = 1e-300 + 1e-18 * fro; /* below this an off-diagonal is zero */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) W[i * m + j] = (i == j) ? 1.0 : 0.0;

  int sweep = 0;
  for (; sweep < max_sweeps && m > 1; ++sweep) {
    int64_t rotations = 0;
    for (int64_t s = 0; s < n - 1; ++s) {
      /* the rotations of this step, from the current A (sym.schur2) */
      for (int64_t u = 0; u < half; ++u) {
        int64_t p, q;
        rr_pair(n, s, u, &p, &q);
        pp[u] = p; qq[u] = q; cc[u] = 1.0; ss[u] = 0.0;
        if (q >= m) continue; /* the padding index of an odd m */
        const double apq = A[p * m + q], app = A[p * m + p], aqq = A[q * m + q];
        if (fabs(apq) <= abs_floor) continue;
        if (fabs(apq) <= 1e-15 * sqrt(fabs(app) * fabs(aqq))) continue;
        const double tau = (aqq - app) / (2.0 * apq);
        const double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                      : -1.0 / (-tau + sqrt(1.0 + tau * tau));
        const double c = 1.0 / sqrt(1.0 + t * t);
        cc[u] = c; ss[u] = t * c;
        ++rotations;
      }
      /* A <- J^T A (rows p, q of every rotating pair) and W <- J^T W */
#pragma omp parallel for schedule(static)
      for (int64_t u = 0; u < half; ++u) {
        if (ss[u] == 0.0) continue;
        const double c = cc[u], sn = ss[u];
        double* Ap = A + pp[u] * m; double* Aq = A + qq[u] * m;
        double* Wp = W + pp[u] * m; double* Wq = W + qq[u] * m;
        for (int64_t r = 0; r < m; ++r) {
          const double x = Ap[r], y = Aq[r];
          Ap[r] = c * x - sn * y;
          Aq[r] = sn * x + c * y;
          const double v = Wp[r], w = Wq[r];
          Wp[r] = c * v - sn * w;
          Wq[r] = sn * v + c * w;
        }
      }
      /* A <- A J (columns p, q of every rotating pair), one row at a time */
#pragma omp parallel for schedule(static)
      for (int64_t r = 0; r < m; ++r) {
        double* Ar = A + r * m;
        for (int64_t u = 0; u < half; ++u) {
          if (ss[u] == 0.0) continue;
          const double c = cc[u], sn = ss[u];
          const double x = Ar[pp[u]], y = Ar[qq[u]];
          Ar[pp[u]] = c * x - sn * y;
          Ar[qq[u]] = sn * x + c * y;
        }
      }
      /* the rotated pair's off-diagonal is zero by construction of (c, s) */
      for (int64_t u = 0; u < half; ++u)
        if (ss[u] != 0.0) { A[pp[u] * m + qq[u]] = 0.0; A[qq[u] * m + pp[u]] = 0.0; }
    }
    if (rotations == 0) break;
  }

  eig_pair* pr = (eig_pair*)malloc(sizeof(eig_pair) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) { pr[i].lam = A[i * m + i]; pr[i].idx = i; }
  qsort(pr, (size_t)m, sizeof(eig_pair), cmp_eig_desc);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < m; ++r) {
    const double* w = W + pr[r].idx * m;
    int64_t jmax = 0;
    for (int64_t j = 1; j < m; ++j)
      if (fabs(w[j]) > fabs(w[jmax])) jmax = j;
    double sg = (w[jmax] < 0.0) ? -1.0 : 1.0;
    lam[r] = pr[r].lam;
    for (int64_t j = 0; j < m; ++j) V[j * m + r] = sg * w[j];
  }
  free(pr); free(A); free(W); free(pp); free(qq); free(cc); free(ss);
  return sweep + 1;
}

/* Sign rule of DESIGN.md R8 applied to k given eigenvectors (V[j*k + r]), for eigenvectors
 * computed by another routine (the LAPACK step of oracle.decompose(eig="lapack")).          */
void oracle_sign_fix(double* V, int64_t m, int64_t k) {
  for (int64_t r = 0; r < k; ++r) {
    int64_t jmax = 0;
    for (int64_t j = 1; j < m; ++j)
      if (fabs(V[j * k + r]) > fabs(V[jmax * k + r])) jmax = j;
    if (V[jmax * k + r] < 0.0)
      for (int64_t j = 0; j < m; ++j) V[j * k + r] = -V[j * k + r];
  }
}

/* ------------------------------------------------------------------ */
/* 5. Outlier set E_top: entries ranked by |X_ij| descending           */
/*    (PAPER.md:21-22); ties by linear index i*m+j ascending, X_ij = 0 */
/*    excluded (R3, R4).  Output ascending by linear index.  */
/* ------------------------------------------------------------------ */
typedef struct { double a; int64_t idx; } abs_pair;
static int cmp_abs_desc(const void* pa, const void* pb) {
  const abs_pair* x = (const abs_pair*)pa;
  const abs_pair* y = (const abs_pair*)pb;
  if (x->a > y->a) return -1;
  if (x->a < y->a) return 1;
  return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}
static int cmp_i64(const void* pa, const void* pb) {
  int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  return (a < b) ? -1 : (a > b);
}

/* Full sort of all nonzero entries — the definition. Returns |E_top|. */
int64_t oracle_top_set_sort(const float* X, int64_t l, int64_t m, int64_t n_top, int64_t* idx) {
  int64_t n = l * m, nz = 0;
  abs_pair* pr = (abs_pair*)malloc(sizeof(abs_pair) * (size_t)(n > 0 ? n : 1));
  if (!pr) return -1;
  for (int64_t t = 0; t < n; ++t) {
    double a = fabs((double)X[t]);
    if (a == 0.0) continue;
    pr[nz].a = a; pr[nz].idx = t; ++nz;
  }
  qsort(pr, (size_t)nz, sizeof(abs_pair), cmp_abs_desc);
  int64_t cnt = nz < n_top ? nz : n_top;
  for (int64_t t = 0; t < cnt; ++t) idx[t] = pr[t].idx;
  free(pr);
  qsort(idx, (size_t)cnt, sizeof(int64_t), cmp_i64);
  return cnt;
}

/* Same set with a bounded min-heap of size n_top (for inputs too large to sort in RAM).
 * The heap's root is the "worst" kept entry under the same comparator. */
static int worse(const abs_pair* x, const abs_pair* y) { /* x ranks after y */
  return cmp_abs_desc(x, y) > 0;
}
int64_t oracle_top_set_heap(const float* X, int64_t l, int64_t m, int64_t n_top, int64_t* idx) {
  abs_pair* h = (abs_pair*)malloc(sizeof(abs_pair) * (size_t)(n_top > 0 ? n_top : 1));
  if (!h) return -1;
  int64_t sz = 0, n = l * m;
  for (int64_t t = 0; t < n; ++t) {
    double a = fabs((double)X[t]);
    if (a == 0.0) continue;
    abs_pair e = {a, t};
    if (sz < n_top) { /* sift up */
      int64_t c = sz++;
      h[c] = e;
      while (c > 0) {
        int64_t par = (c - 1) / 2;
        if (worse(&h[c], &h[par])) { abs_pair tmp = h[c]; h[c] = h[par]; h[par] = tmp; c = par; }
        else break;
      }
    } else if (sz > 0 && worse(&h[0], &e)) { /* e ranks before the worst kept: replace root */
      h[0] = e;
      int64_t c = 0;
      for (;;) {
        int64_t L = 2 * c + 1, R = L + 1, w = c;
        if (L < sz && worse(&h[L], &h[w])) w = L;
        if (R < sz && worse(&h[R], &h[w])) w = R;
        if (w == c) break;
        abs_pair tmp = h[c]; h[c] = h[w]; h[w] = tmp; c = w;
      }
    }
  }
  for (int64_t t = 0; t < sz; ++t) idx[t] = h[t].idx;
  free(h);
  qsort(idx, (size_t)sz, sizeof(int64_t), cmp_i64);
  return sz;
}

/* ------------------------------------------------------------------ */
/* 6. The whole pass.                                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n_top;             /* |E_top| actually selected (< request only if fewer nonzeros) */
  double energy_cf[4];       /* closed forms: total=sum x^2, mean=l||mu||^2, spike=sum_{r<=k} lam_r,
                                tail = tr(G) - sum_{r<=k} lam_r           */
  double energy_el[4];       /* elementwise: sum x^2, sum M^2, sum S^2, sum T^2                 */
  double cross_el[3];        /* <M,S>, <M,T>, <S,T> Frobenius inner products  */
  double colmean_absmax[2];  /* max_j |mean_i S_ij|, max_j |mean_i T_ij|          */
  double rho_mean_aggr[4];   /* mean over E_top of rho_mean, rho_spike, rho_tail, cross (R10)   */
  double rho_energy_aggr[3]; /* sum_E c^2 / sum_E x^2 for c = M, S, T                        */
  double sigma_next;         /* sigma_{k+1}, 0 if k = m                                          */
  double trace_g;            /* tr(G) = ||Xc||_F^2                                              */
  int32_t sweeps;            /* Jacobi sweeps                                                   */
  int32_t status;
} oracle_report;

/* Phase 1 of the pass: validation, mu and G = Xc^T Xc. */
int oracle_mean_gram(const float* X, int64_t l, int64_t m, int32_t k, double* mu, double* G) {
  /* validation (R1, R5) */
  if (l < 2 || m < 2 || k < 1 || k > (l < m ? l : m)) return ORACLE_EINVAL;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < m; ++j)
      if (!isfinite(X[i * m + j])) bad = 1;
  if (bad) return ORACLE_ENONFINITE;
  oracle_column_mean(X, l, m, mu);
  return oracle_gram_x(X, l, m, mu, G);
}

/* Phase 3 of the pass, given mu, the eigenvalues lam[0..k] of G (lam[k] only if k < m), the
 * eigenvectors V_k (V[j*k + r], sign rule applied) and tr(G):
 *   spike / tail row by row: p_i = xc_i V_k, S_i = p_i V_k^T, T_i = xc_i - S_i,
 *   elementwise and closed-form energies, E_top, rho and
 *   cross.
 * Row sums are taken over fixed blocks of rows (ORACLE_NB blocks, each summed in row order, the
 * block partials then added in block order), so the result does not depend on the thread count. */
#define ORACLE_NB 256
int oracle_finish(const float* X, int64_t l, int64_t m, int32_t k, int64_t n_top_req, int32_t use_heap,
                  const double* mu, const double* lam, const double* V, double trace, double* sigma,
                  int64_t* top_idx, double* rho, oracle_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (l < 2 || m < 2 || k < 1 || k > (l < m ? l : m) || n_top_req < 1) {
    rep->status = ORACLE_EINVAL; return ORACLE_EINVAL;
  }
  rep->trace_g = trace;
  double sum_lam_k = 0.0;
  for (int32_t r = 0; r < k; ++r) {
    double lr = lam[r] > 0.0 ? lam[r] : 0.0; /* DESIGN.md R9: sigma = sqrt(max(lam, 0)) */
    sigma[r] = sqrt(lr);
    sum_lam_k = sum_lam_k + lr;
  }
  rep->sigma_next = (k < m) ? sqrt(lam[k] > 0.0 ? lam[k] : 0.0) : 0.0;

  const int64_t nb = l < ORACLE_NB ? l : ORACLE_NB;
  double* P = (double*)malloc(sizeof(double) * (size_t)(l * k));
  double* part = (double*)calloc((size_t)(nb * 4), sizeof(double));
  double* csS = (double*)calloc((size_t)(nb * m), sizeof(double));
  double* csT = (double*)calloc((size_t)(nb * m), sizeof(double));
  if (!P || !part || !csS || !csT) {
    free(P); free(part); free(csS); free(csT);
    rep->status = ORACLE_ENOMEM; return ORACLE_ENOMEM;
  }
  int oom = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : oom)
  for (int64_t blk = 0; blk < nb; ++blk) {
    const int64_t i0 = l * blk / nb, i1 = l * (blk + 1) / nb;
    double* xc = (double*)malloc(sizeof(double) * (size_t)m);
    double* S_row = (double*)malloc(sizeof(double) * (size_t)m);
    if (!xc || !S_row) { free(xc); free(S_row); oom = 1; continue; }
    double sx2 = 0.0, sS2 = 0.0, sT2 = 0.0, sST = 0.0;
    double* cS = csS + blk * m;
    double* cT = csT + blk * m;
    for (int64_t i = i0; i < i1; ++i) {
      for (int64_t j = 0; j < m; ++j) xc[j] = (double)X[i * m + j] - mu[j];
      double* p = P + i * k;
      for (int32_t r = 0; r < k; ++r) {
        double s = 0.0;
        for (int64_t j = 0; j < m; ++j) s = s + xc[j] * V[j * k + r];
        p[r] = s;
      }
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int32_t r = 0; r < k; ++r) s = s + p[r] * V[j * k + r];
        S_row[j] = s;
      }
      for (int64_t j = 0; j < m; ++j) {
        double x = (double)X[i * m + j];
        double Sij = S_row[j];
        double Tij = xc[j] - Sij;
        sx2 = sx2 + x * x;
        sS2 = sS2 + Sij * Sij;
        sT2 = sT2 + Tij * Tij;
        sST = sST + Sij * Tij;
        cS[j] = cS[j] + Sij;
        cT[j] = cT[j] + Tij;
      }
    }
    part[blk * 4 + 0] = sx2; part[blk * 4 + 1] = sS2; part[blk * 4 + 2] = sT2; part[blk * 4 + 3] = sST;
    free(xc); free(S_row);
  }
  if (oom) {
    free(P); free(part); free(csS); free(csT);
    rep->status = ORACLE_ENOMEM; return ORACLE_ENOMEM;
  }
  double sum_x2 = 0.0, sum_S2 = 0.0, sum_T2 = 0.0, sum_ST = 0.0;
  for (int64_t blk = 0; blk < nb; ++blk) {
    sum_x2 = sum_x2 + part[blk * 4 + 0];
    sum_S2 = sum_S2 + part[blk * 4 + 1];
    sum_T2 = sum_T2 + part[blk * 4 + 2];
    sum_ST = sum_ST + part[blk * 4 + 3];
  }
  double sum_mu2 = 0.0, MS = 0.0, MT = 0.0, amS = 0.0, amT = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    double sS = 0.0, sT = 0.0;
    for (int64_t blk = 0; blk < nb; ++blk) { sS = sS + csS[blk * m + j]; sT = sT + csT[blk * m + j]; }
    sum_mu2 = sum_mu2 + mu[j] * mu[j];
    MS = MS + mu[j] * sS;
    MT = MT + mu[j] * sT;
    double a = fabs(sS / (double)l), b = fabs(sT / (double)l);
    if (a > amS) amS = a;
    if (b > amT) amT = b;
  }
  rep->energy_cf[0] = sum_x2;
  rep->energy_cf[1] = (double)l * sum_mu2;
  rep->energy_cf[2] = sum_lam_k;
  rep->energy_cf[3] = trace - sum_lam_k;
  rep->energy_el[0] = sum_x2;
  rep->energy_el[1] = (double)l * sum_mu2;
  rep->energy_el[2] = sum_S2;
  rep->energy_el[3] = sum_T2;
  rep->cross_el[0] = MS;
  rep->cross_el[1] = MT;
  rep->cross_el[2] = sum_ST;
  rep->colmean_absmax[0] = amS;
  rep->colmean_absmax[1] = amT;

  /* E_top and rho */
  int64_t n_top = use_heap ? oracle_top_set_heap(X, l, m, n_top_req, top_idx)
                           : oracle_top_set_sort(X, l, m, n_top_req, top_idx);
  rep->n_top = n_top;
  double* Sv = (double*)malloc(sizeof(double) * (size_t)(n_top > 0 ? 2 * n_top : 1));
  if (!Sv) {
    free(P); free(part); free(csS); free(csT);
    rep->status = ORACLE_ENOMEM; return ORACLE_ENOMEM;
  }
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n_top; ++t) {
    int64_t i = top_idx[t] / m, j = top_idx[t] % m;
    double x = (double)X[i * m + j];
    double M = mu[j];
    double Sij = 0.0;
    for (int32_t r = 0; r < k; ++r) Sij = Sij + P[i * k + r] * V[j * k + r];
    double Tij = (x - mu[j]) - Sij;
    double x2 = x * x;
    double rm = M * M / x2, rs = Sij * Sij / x2, rt = Tij * Tij / x2;
    double cr = 1.0 - (rm + rs + rt);
    rho[t * 4 + 0] = rm; rho[t * 4 + 1] = rs; rho[t * 4 + 2] = rt; rho[t * 4 + 3] = cr;
    Sv[2 * t] = Sij; Sv[2 * t + 1] = Tij;
  }
  double agg[4] = {0, 0, 0, 0}, eM = 0, eS = 0, eT = 0, eX = 0;
  for (int64_t t = 0; t < n_top; ++t) {
    int64_t j = top_idx[t] % m;
    double x = (double)X[top_idx[t]];
    double x2 = x * x;
    agg[0] = agg[0] + rho[t * 4 + 0]; agg[1] = agg[1] + rho[t * 4 + 1];
    agg[2] = agg[2] + rho[t * 4 + 2]; agg[3] = agg[3] + rho[t * 4 + 3];
    eM = eM + mu[j] * mu[j]; eS = eS + Sv[2 * t] * Sv[2 * t]; eT = eT + Sv[2 * t + 1] * Sv[2 * t + 1]; eX = eX + x2;
  }
  for (int c = 0; c < 4; ++c) rep->rho_mean_aggr[c] = n_top > 0 ? agg[c] / (double)n_top : 0.0;
  rep->rho_energy_aggr[0] = eX > 0 ? eM / eX : 0.0;
  rep->rho_energy_aggr[1] = eX > 0 ? eS / eX : 0.0;
  rep->rho_energy_aggr[2] = eX > 0 ? eT / eX : 0.0;

  free(P); free(part); free(csS); free(csT); free(Sv);
  rep->status = ORACLE_OK;
  return ORACLE_OK;
}

int oracle_decompose(const float* X, int64_t l, int64_t m, int32_t k, int64_t n_top_req,
                     int32_t use_heap, double* mu, double* V, double* sigma, double* lam_all,
                     int64_t* top_idx, double* rho, oracle_report* rep) {
  memset(rep, 0, sizeof(*rep));
  if (l < 2 || m < 2 || k < 1 || k > (l < m ? l : m) || n_top_req < 1) {
    rep->status = ORACLE_EINVAL; return ORACLE_EINVAL;
  }
  double* G = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* Vall = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* lam = (double*)malloc(sizeof(double) * (size_t)m);
  if (!G || !Vall || !lam) {
    free(G); free(Vall); free(lam);
    rep->status = ORACLE_ENOMEM; return ORACLE_ENOMEM;
  }
  /* mu, G */
  int st = oracle_mean_gram(X, l, m, k, mu, G);
  if (st != ORACLE_OK) { free(G); free(Vall); free(lam); rep->status = st; return st; }
  /* truncated SVD of Xc through the eigenpairs of G */
  const int sweeps = oracle_jacobi_eig(G, m, lam, Vall, 60);
  double trace = 0.0;
  for (int64_t j = 0; j < m; ++j) trace = trace + G[j * m + j];
  for (int64_t r = 0; r < m; ++r)
    if (lam_all) lam_all[r] = lam[r];
  for (int32_t r = 0; r < k; ++r)
    for (int64_t j = 0; j < m; ++j) V[j * k + r] = Vall[j * m + r];
  free(G); free(Vall);
  st = oracle_finish(X, l, m, k, n_top_req, use_heap, mu, lam, V, trace, sigma, top_idx, rho, rep);
  rep->sweeps = sweeps;
  free(lam);
  return st;
}
