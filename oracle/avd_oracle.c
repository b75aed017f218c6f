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
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC (see oracle/build.py).
 * OpenMP is used only across independent outputs; no summation order is changed by it.
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
 *    summed in row order i; computed for b >= a and mirrored (G is symmetric).
 *    XcT is the transpose of Xc (m x l) so each entry is one contiguous dot product. */
void oracle_gram(const double* Xc, int64_t l, int64_t m, double* G) {
  double* XcT = (double*)malloc(sizeof(double) * (size_t)(l * m));
  if (!XcT) return;
#pragma omp parallel for schedule(static)
  for (int64_t a = 0; a < m; ++a)
    for (int64_t i = 0; i < l; ++i) XcT[a * l + i] = Xc[i * m + a];
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t a = 0; a < m; ++a) {
    const double* xa = XcT + a * l;
    for (int64_t b = a; b < m; ++b) {
      const double* xb = XcT + b * l;
      double s = 0.0;
      for (int64_t i = 0; i < l; ++i) s = s + xa[i] * xb[i];
      G[a * m + b] = s;
      G[b * m + a] = s;
    }
  }
  free(XcT);
}

/* ------------------------------------------------------------------ */
/* 4. Symmetric eigendecomposition of G by cyclic-by-row Jacobi        */
/*    (Golub & Van Loan, "Matrix Computations", Alg. 8.5.2 sym.schur2  */
/*    + Alg. 8.5.3 cyclic Jacobi; Rutishauser's update formulas).      */
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

int oracle_jacobi_eig(const double* G, int64_t m, double* lam, double* V, int max_sweeps) {
  double* A = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* W = (double*)malloc(sizeof(double) * (size_t)(m * m)); /* W = V^T: row r = eigvec r */
  if (!A || !W) { free(A); free(W); return -1; }
  memcpy(A, G, sizeof(double) * (size_t)(m * m));
  double fro = 0.0;
  for (int64_t i = 0; i < m * m; ++i) fro = fro + A[i] * A[i];
  fro = sqrt(fro);
  const double abs_floor = 1e-300 + 1e-18 * fro; /* below this an off-diagonal is zero */
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) W[i * m + j] = (i == j) ? 1.0 : 0.0;

  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int64_t rotations = 0;
    for (int64_t p = 0; p < m - 1; ++p) {
      for (int64_t q = p + 1; q < m; ++q) {
        double apq = A[p * m + q];
        double app = A[p * m + p], aqq = A[q * m + q];
        if (fabs(apq) <= abs_floor) continue;
        if (fabs(apq) <= 1e-15 * sqrt(fabs(app) * fabs(aqq))) continue;
        /* sym.schur2: choose (c, s) so that J^T A J zeroes a_pq */
        double tau = (aqq - app) / (2.0 * apq);
        double t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                : -1.0 / (-tau + sqrt(1.0 + tau * tau));
        double c = 1.0 / sqrt(1.0 + t * t);
        double s = t * c;
        double* Ap = A + p * m;
        double* Aq = A + q * m;
        for (int64_t r = 0; r < m; ++r) {
          if (r == p || r == q) continue;
          double arp = Ap[r], arq = Aq[r];
          double np = c * arp - s * arq;
          double nq = s * arp + c * arq;
          Ap[r] = np; A[r * m + p] = np;
          Aq[r] = nq; A[r * m + q] = nq;
        }
        Ap[p] = app - t * apq;
        Aq[q] = aqq + t * apq;
        Ap[q] = 0.0; Aq[p] = 0.0;
        double* Wp = W + p * m;
        double* Wq = W + q * m;
        for (int64_t r = 0; r < m; ++r) {
          double vp = Wp[r], vq = Wq[r];
          Wp[r] = c * vp - s * vq;
          Wq[r] = s * vp + c * vq;
        }
        ++rotations;
      }
    }
    if (rotations == 0) break;
  }

  eig_pair* pr = (eig_pair*)malloc(sizeof(eig_pair) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) { pr[i].lam = A[i * m + i]; pr[i].idx = i; }
  qsort(pr, (size_t)m, sizeof(eig_pair), cmp_eig_desc);
  for (int64_t r = 0; r < m; ++r) {
    const double* w = W + pr[r].idx * m;
    int64_t jmax = 0;
    for (int64_t j = 1; j < m; ++j)
      if (fabs(w[j]) > fabs(w[jmax])) jmax = j;
    double sg = (w[jmax] < 0.0) ? -1.0 : 1.0;
    lam[r] = pr[r].lam;
    for (int64_t j = 0; j < m; ++j) V[j * m + r] = sg * w[j];
  }
  free(pr); free(A); free(W);
  return sweep + 1;
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

int oracle_decompose(const float* X, int64_t l, int64_t m, int32_t k, int64_t n_top_req,
                     int32_t use_heap, double* mu, double* V, double* sigma, double* lam_all,
                     int64_t* top_idx, double* rho, oracle_report* rep) {
  memset(rep, 0, sizeof(*rep));
  /* validation (R1, R5) */
  if (l < 2 || m < 2 || k < 1 || k > (l < m ? l : m) || n_top_req < 1) {
    rep->status = ORACLE_EINVAL; return ORACLE_EINVAL;
  }
  for (int64_t t = 0; t < l * m; ++t)
    if (!isfinite(X[t])) { rep->status = ORACLE_ENONFINITE; return ORACLE_ENONFINITE; }

  double* Xc = (double*)malloc(sizeof(double) * (size_t)(l * m));
  double* G = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* Vall = (double*)malloc(sizeof(double) * (size_t)(m * m));
  double* lam = (double*)malloc(sizeof(double) * (size_t)m);
  double* P = (double*)malloc(sizeof(double) * (size_t)(l * k));
  double* csS = (double*)calloc((size_t)m, sizeof(double));
  double* csT = (double*)calloc((size_t)m, sizeof(double));
  double* S_row = (double*)malloc(sizeof(double) * (size_t)m);
  if (!Xc || !G || !Vall || !lam || !P || !csS || !csT || !S_row) {
    free(Xc); free(G); free(Vall); free(lam); free(P); free(csS); free(csT); free(S_row);
    rep->status = ORACLE_ENOMEM; return ORACLE_ENOMEM;
  }

  /* mu, Xc */
  oracle_column_mean(X, l, m, mu);
  oracle_center(X, l, m, mu, Xc);

  /* truncated SVD of Xc through G = Xc^T Xc */
  oracle_gram(Xc, l, m, G);
  rep->sweeps = oracle_jacobi_eig(G, m, lam, Vall, 60);
  double trace = 0.0;
  for (int64_t j = 0; j < m; ++j) trace = trace + G[j * m + j];
  rep->trace_g = trace;
  for (int64_t r = 0; r < m; ++r)
    if (lam_all) lam_all[r] = lam[r];
  double sum_lam_k = 0.0;
  for (int32_t r = 0; r < k; ++r) {
    double lr = lam[r] > 0.0 ? lam[r] : 0.0; /* DESIGN.md R9: sigma = sqrt(max(lam, 0)) */
    sigma[r] = sqrt(lr);
    sum_lam_k = sum_lam_k + lr;
    for (int64_t j = 0; j < m; ++j) V[j * k + r] = Vall[j * m + r];
  }
  rep->sigma_next = (k < m) ? sqrt(lam[k] > 0.0 ? lam[k] : 0.0) : 0.0;

  /* spike / tail row by row: p_i = xc_i V_k, S_i = p_i V_k^T, T_i = xc_i - S_i */
  double sum_x2 = 0.0, sum_S2 = 0.0, sum_T2 = 0.0, sum_ST = 0.0;
  for (int64_t i = 0; i < l; ++i) {
    const double* xc = Xc + i * m;
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
      sum_x2 = sum_x2 + x * x;
      sum_S2 = sum_S2 + Sij * Sij;
      sum_T2 = sum_T2 + Tij * Tij;
      sum_ST = sum_ST + Sij * Tij;
      csS[j] = csS[j] + Sij;
      csT[j] = csT[j] + Tij;
    }
  }
  double sum_mu2 = 0.0, MS = 0.0, MT = 0.0, amS = 0.0, amT = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    sum_mu2 = sum_mu2 + mu[j] * mu[j];
    MS = MS + mu[j] * csS[j];
    MT = MT + mu[j] * csT[j];
    double a = fabs(csS[j] / (double)l), b = fabs(csT[j] / (double)l);
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
  double agg[4] = {0, 0, 0, 0}, eM = 0, eS = 0, eT = 0, eX = 0;
  for (int64_t t = 0; t < n_top; ++t) {
    int64_t i = top_idx[t] / m, j = top_idx[t] % m;
    double x = (double)X[i * m + j];
    double M = mu[j];
    double Sij = 0.0;
    for (int32_t r = 0; r < k; ++r) Sij = Sij + P[i * k + r] * V[j * k + r];
    double Tij = Xc[i * m + j] - Sij;
    double x2 = x * x;
    double rm = M * M / x2, rs = Sij * Sij / x2, rt = Tij * Tij / x2;
    double cr = 1.0 - (rm + rs + rt);
    rho[t * 4 + 0] = rm; rho[t * 4 + 1] = rs; rho[t * 4 + 2] = rt; rho[t * 4 + 3] = cr;
    agg[0] = agg[0] + rm; agg[1] = agg[1] + rs; agg[2] = agg[2] + rt; agg[3] = agg[3] + cr;
    eM = eM + M * M; eS = eS + Sij * Sij; eT = eT + Tij * Tij; eX = eX + x2;
  }
  for (int c = 0; c < 4; ++c) rep->rho_mean_aggr[c] = n_top > 0 ? agg[c] / (double)n_top : 0.0;
  rep->rho_energy_aggr[0] = eX > 0 ? eM / eX : 0.0;
  rep->rho_energy_aggr[1] = eX > 0 ? eS / eX : 0.0;
  rep->rho_energy_aggr[2] = eX > 0 ? eT / eX : 0.0;

  free(Xc); free(G); free(Vall); free(lam); free(P); free(csS); free(csT); free(S_row);
  rep->status = ORACLE_OK;
  return ORACLE_OK;
}
