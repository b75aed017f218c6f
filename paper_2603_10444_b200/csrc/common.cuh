// common.cuh — shared context, error handling and launch helpers of libavd (product code).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/avd.h"

namespace avd {

constexpr int kHistBins = 4096;   // first/second level: 12 key bits
constexpr int kHist3Bins = 128;   // third level: 7 key bits
constexpr int kGramTile = 128;    // Gram tile edge (rows of A / B panels)
constexpr int kGramK = 128;       // K rows per pipeline stage (one 128-byte swizzle row of int8)
constexpr int kMaxP = 112;        // subspace block size cap (two p x p fp64 matrices in smem)
constexpr int kRedRowsC = 128;    // rows per partial of the m-length p x p reductions (k_eig.cu)
constexpr int kEigCtlBytes = 256; // device-resident loop state of the eigensolver graph (k_eig.cu)
constexpr int kCtlBlocksU = 10;   // int index of EigCtl::blocks_u (then iters_u), read by the report
constexpr int kHostScratch = 8 * kMaxP;  // doubles of the pinned host scratch (eig_host)

// Device-side "plan2": values decided on the device after the stats exchange.
struct DevPlan {
  int64_t n_eff;        // min(n_top, #nonzero entries)
  int64_t cnt_gt;       // #entries with key strictly above the current bin prefix
  int64_t cand_count;   // candidates appended by K2
  int64_t nonfinite;    // #non-finite entries seen by K1
  int32_t b0;           // candidate threshold bin (from the row-sampled histogram)
  int32_t b1, b2;       // selected first/second level bins
  uint32_t T;           // exact 31-bit key threshold (n_top-th largest |x| bits)
  int32_t empty;        // 1 when n_eff == 0
  int64_t cnt_gt_T;     // #entries with key > T (global)
  int64_t q;            // ties (key == T) to take, globally
  int64_t ties_local;   // ties held by this rank
  int64_t quota;        // ties this rank takes
  int64_t sel_local;    // entries of E_top held by this rank
  int64_t top_offset;   // global position of this rank's first entry
  int32_t range_bits;   // max_j ceil(log2(max|y_j| / planned range)): bits an exact-range requant loses
  int32_t pad0;
};

struct Ctx {
  avd_config cfg;
  avd_plan_t plan;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t m_pad = 0;     // m rounded up to kGramTile
  int64_t l_pad = 0;     // l_local rounded up to kGramK
  int k = 0, p = 0, k_pad = 0;
  int nd = 3;
  int nd_max = 3;        // digit planes the workspace holds (3 when digits are automatic)
  bool auto_digits = false;
  bool escalate = false; // stage_gram must re-encode with nd = 3 (set by stage_eig)
  double prec_sigma = 0, prec_share = 0;  // a-posteriori quantisation-error bounds (run_eig)
  int64_t launches = 0;
  int stage = 0;         // last completed stage (ordering check)
  // K1
  int r1 = 1;                 // row chunks of the stats kernel
  double* colsum_part = nullptr;  // [r1][m]
  float* colmax_part = nullptr;   // [r1][m]
  float* colmin_part = nullptr;   // [r1][m]
  double* sq_part = nullptr;      // [r1 * ncb]
  double* stats = nullptr;        // [m + 4]: colsum[m], sum x^2 (set by the trace kernel from ysq), -, #nonzero, #overflowing columns (exchange)
  double* samp = nullptr;         // [m + 1]: row-sample column sums, #sampled rows (exchange SUM)
  float* smax = nullptr;          // [m] row-sample column max (exchange MAX)
  float* smin = nullptr;          // [m] row-sample column min (exchange MIN)
  float* qscale = nullptr;        // [m_pad] 2^shift (fp32)
  float* mu0 = nullptr;           // [m_pad] quantiser centre (fl32 of the sample mean)
  float* qoff = nullptr;          // [m_pad] -mu0 * 2^shift (fp32)
  long long* qsum_part = nullptr; // [r1][m] per-chunk integer column sums of q
  long long* qsum_local = nullptr;// [2 m]: this rank's column sums of q | sums of q^2
  long long* qsq_part = nullptr;  // [r1][m] per-chunk sums of q^2
  float* qerr_part = nullptr;     // [r1][m] per-chunk sums of the squared rounding errors
  double* qerr_local = nullptr;   // [m_pad] this rank's sums of squared rounding errors
  double* qerr = nullptr;         // [m_pad] (exchange SUM)
  double* ysq = nullptr;          // [m] sum_i (x_ij - mu0_j)^2, fp64 (exchange SUM): diag of G, ||X||^2
  unsigned long long* hist0 = nullptr;  // [4096] exact first-level histogram over candidates (exchange)
  float* colmax = nullptr;        // [m] max |x - mu0| (exchange MAX)
  float* colmin = nullptr;        // [m] (exchange MIN)
  unsigned long long* hist1 = nullptr;  // [4096] (exchange SUM)
  // prepare
  double* mu = nullptr;           // [m]
  float* mu_hl = nullptr;         // [2][m_pad]: mu = hi + lo (fp32 pair) for fp32 centring
  int32_t* shift = nullptr;       // [m_pad] digit scale exponent per column
  DevPlan* dplan = nullptr;
  DevPlan hplan{};
  // K2
  int8_t* digits = nullptr;       // [nd][m_pad][l_pad]
  uint32_t* cand_key = nullptr;   // [cand_cap]
  uint64_t* cand_idx = nullptr;   // [cand_cap]
  unsigned long long* cand_cnt = nullptr;
  int64_t cand_cap = 0;
  long long* cand_x = nullptr;    // [2] exchange SUM: candidate count, overflow flag
  bool cand_overflow = false;     // true -> K6 streams X instead of the candidate list
  bool requantised = false;       // the sampled digit scales overflowed: requantised with exact ranges
  // K3
  long long* gram_i = nullptr;    // [m_pad * m_pad] int64 (upper tiles) (exchange SUM)
  long long* gram_p = nullptr;    // world > 1: the upper 128-tiles packed [T(T+1)/2][128][128] (exchange SUM)
  double* G = nullptr;            // [m_pad][m_pad] fp64 symmetric (zero beyond m)
  float* G32 = nullptr;           // [m_pad][m_pad] fp32 copy (power steps of K4)
  long long* qsum = nullptr;      // [2 m] column sums of the quantised operand | of its squares (exchange SUM)
  CUtensorMap tmap_digits{};
  CUtensorMap tmap_digits_b{};    // 64-column SWIZZLE_64B boxes (B halves of the CTA-pair Gram)
  int gram_split = 1;
  // K4
  double *Q = nullptr, *Y = nullptr, *Z = nullptr, *U = nullptr;  // [m][p]
  double *H = nullptr, *W = nullptr, *theta = nullptr;          // [p][p], [p][p], [p]
  double* red_part = nullptr;     // [n_red_chunks][p*p]
  int n_red = 1;
  void* gemm_part = nullptr;      // split-K partials of Y = G Q [RB][KS][BM][p] + row-block tickets
  float *Q32 = nullptr, *Z32 = nullptr;  // [m][p] fp32 mirrors of Q, Z
  unsigned* ticket = nullptr;     // last-CTA ticket of the fused reductions
  double* gmax = nullptr;         // max |G| (fixed-point scale of the Y = G Q accumulation)
  void* eig_ctl = nullptr;        // [kEigCtlBytes] loop state of the eigensolver graph
  int8_t* gd = nullptr;           // [4][m_pad][m_pad] G in balanced base-128 digits (k_eig_i8.cu)
  double* gsc = nullptr;          // [m_pad] row scales of gd
  int8_t* qd = nullptr;           // [3][p][m_pad] the product's input block in digits (transposed)
  double* qsc = nullptr;          // [2 kMaxP] its column scales | column maxima (bit patterns)
  double* g8_part = nullptr;      // split-K partials of the int8 products
  unsigned* g8_tickets = nullptr; // [m_pad / 128] last-CTA tickets
  CUtensorMap tm_gd{}, tm_qd{};
  CUtensorMap* tm_dev = nullptr;  // [2] device copies of tm_gd, tm_qd (64-B aligned; graph kernels read them)
  bool tm_gd_ready = false;
  cudaGraphExec_t eig_exec = nullptr;   // subspace-iteration loop (built once per context)
  cudaGraphExec_t unc_exec = nullptr;   // uncentred power iteration loop (diagnostics)
  cudaStream_t cap_stream = nullptr;    // private stream the graphs are captured on
  cudaStream_t side_stream = nullptr;   // the uncentred loop runs here, concurrent with the eig
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int n_begin_nodes = 0, n_rr_nodes = 0, n_pow_nodes = 0, n_u_nodes = 0;  // kernels per graph body
  // mean-bias diagnostics: diag[0] = ||mu||, diag[4..4+m_pad) = q,
  // diag[4+m_pad..) = y of the uncentred power iteration
  double* diag = nullptr;
  double sigma1_u = 0, alpha1 = 0, cos_mu_v1 = 0, resid_u = 0;
  double* unc_topk = nullptr;     // [2 * kMaxP]: uncentred sigma_i | alpha_i, i < k (AVD_FLAG_MEAN_TOPK)
  int iters_uk = 0;
  double resid_uk = 0;
  int iters_u = 0;
  bool sign_valid = false;        // p_i signs available (tensor-core projection path)
  double* resid = nullptr;        // [p]
  double* trace = nullptr;        // [4]: tr(G), sum_a d_a^2 G_aa (precision bound), -, -
  double* prec = nullptr;         // [kMaxP]: t_r = sum_a d_a^2 v_ra^2 (quantisation step d_a)
  double* eig_host = nullptr;     // pinned: theta[p] + resid[p]
  cudaEvent_t ev_host = nullptr;  // host waits on this instead of the whole stream (stage_gram)
  double* V = nullptr;            // [m][k] output copy (row-major)
  double* sigma = nullptr;        // [k]
  float* V32 = nullptr;           // [m][k_pad] fp32 copy for K5/K8
  int iters = 0;
  int rr_count = 0;               // Rayleigh-Ritz checks in the last solve
  int jacobi_sweeps = 0;          // sweeps of the last Rayleigh-Ritz Jacobi
  double max_resid = 0;
  double sigma_next = 0;
  // K5/K8
  float* P = nullptr;             // [l_local][k_pad]
  int8_t* Pd = nullptr;           // [3][l_pad][128] P's spike columns in digits (K8 A operand)
  float* ps = nullptr;            // [l_pad] their row scales
  float* Vt_hl = nullptr;         // [2*k_pad][m_pad32] fp32 words; holds K5's int8 W digit planes [4][k_pad][m_pad]
  double* wsc = nullptr;          // [512]: K5 column scales t_r | corrections corr_r | (int) spiky columns at 384
  int8_t* Vd = nullptr;           // [3][m_pad][128] V_k in digits (K8 B operand)
  float* vs = nullptr;            // [m_pad] its row scales
  int64_t m_pad32 = 0;
  double* en_part = nullptr;      // [n_proj_ctas][4]
  double* colsumP_part = nullptr; // [n_proj_ctas][k_pad]
  int n_proj_ctas = 1;
  double* energy = nullptr;       // [4 + k_pad + m] exchange SUM: x^2, S^2, T^2, ST, colsumP[k_pad], colsumXc[m]
  // K6
  unsigned long long* hist2 = nullptr;  // [4096] (exchange)
  unsigned long long* hist3 = nullptr;  // [128] (exchange)
  long long* ties = nullptr;            // [world] (exchange)
  uint32_t* bm_sel = nullptr;           // bitmap [nwords]
  uint32_t* bm_tie = nullptr;
  int64_t nwords = 0;
  int64_t* blk_cnt = nullptr;           // [2 * nblk + 2] scan scratch
  int64_t nblk = 0;
  // K7
  double* agg = nullptr;                // [8] exchange: sum rho(4), sum_E M^2, S^2, T^2, X^2
  double* agg_part = nullptr;
  int n_gather_ctas = 1;
  // host path
  float* X_stage = nullptr;             // device copy for avd_decompose_host
  size_t ws_bytes = 0;
  // Gram-free products (AVD_FLAG_GRAM_FREE; k_gramfree.cu), allocated on first use
  bool gram_free = false;
  int8_t* gf_wd = nullptr;        // [4][KQ][m_pad] digits of 2^-s In
  double* gf_wsc = nullptr;       // [2 KQ]: column scales t_r | centring terms corr_r
  double* gf_tq = nullptr;        // [KQ] scales of P's digits
  unsigned* gf_pmax = nullptr;    // [KQ] column max |P| (fp32 bit patterns)
  long long* gf_zsum = nullptr;   // [KQ] column sums of P's integer codes
  float* gf_P = nullptr;          // [l_pad][KQ] P = Xhat In
  int8_t* gf_pd = nullptr;        // [4][l_pad][KQ] digits of P
  long long* gf_zi = nullptr;     // [m_pad][KQ] Xq^T Pd, high word (weight 2^28; reset after each product)
  long long* gf_zlo = nullptr;    // [m_pad][KQ] low word
  double* gf_dd = nullptr;        // [m_pad] exact minus quantised diagonal of Xhat^T Xhat
  long long* gf_qsq = nullptr;    // [m_pad] sum_i q_ij^2 of the digit planes
  CUtensorMap* gf_tm = nullptr;   // [3] device-resident tensor maps (X digits, W digits, P digits)
  std::vector<void*> gf_allocs;
};

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);

#define AVD_CUDA(call)                                                                \
  do {                                                                                \
    cudaError_t e__ = (call);                                                         \
    if (e__ != cudaSuccess) {                                                         \
      ::avd::set_error(std::string(#call) + " failed: " + cudaGetErrorString(e__) +   \
                       " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")");       \
      return AVD_ECUDA;                                                               \
    }                                                                                 \
  } while (0)

#define AVD_LAUNCHED(ctx)                                                             \
  do {                                                                                \
    (ctx)->launches++;                                                                \
    cudaError_t e__ = cudaGetLastError();                                             \
    if (e__ != cudaSuccess) {                                                         \
      ::avd::set_error(std::string("kernel launch failed: ") + cudaGetErrorString(e__) + \
                       " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")");       \
      return AVD_ECUDA;                                                               \
    }                                                                                 \
  } while (0)

#define AVD_TRY(expr)                        \
  do {                                       \
    avd_status s__ = (expr);                 \
    if (s__ != AVD_OK) return s__;           \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs more than it was last
// given (a host API call per launch costs microseconds; the eigensolver launches ~100 kernels)
cudaError_t smem_attr_impl(const void* fn, int bytes);
template <typename F>
inline cudaError_t smem_attr(F* fn, int bytes) { return smem_attr_impl(reinterpret_cast<const void*>(fn), bytes); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------- kernels (per file)
avd_status launch_sample(Ctx* c, const float* X);          // k_pass1.cu
avd_status launch_pass1(Ctx* c, const float* X, bool full); // k_pass1.cu
avd_status launch_finish(Ctx* c);                          // k_pass1.cu
avd_status launch_uncentred(Ctx* c);                       // k_eig.cu (mean-bias diagnostics, side stream)
avd_status join_uncentred(Ctx* c);                         // k_eig.cu
void destroy_graphs(Ctx* c);                               // k_eig.cu
avd_status run_uncentred_topk(Ctx* c, double* out);        // k_eig.cu (optional)
avd_status launch_sign_count(Ctx* c);                      // k_project.cu (mean-bias diagnostics)
avd_status launch_gram(Ctx* c, const double* skip = nullptr);  // k_gram.cu (skip: device gate)
avd_status gram_make_tmap(Ctx* c);                         // k_gram.cu
avd_status launch_gram_finalize(Ctx* c);                   // k_eig.cu
avd_status run_eig(Ctx* c);                                // k_eig.cu
avd_status run_eig_dist(Ctx* c, int rank, avd_exchange_fn fn, void* user);  // k_eig.cu
avd_status launch_gram_pack(Ctx* c, bool unpack);          // k_gram.cu (world > 1 exchange)
bool eig_i8_enabled(const Ctx* c);                         // k_eig_i8.cu
avd_status eig_i8_prepare(Ctx* c);                         // k_eig_i8.cu (once per solve)
avd_status gemm_i8(Ctx* c, const double* In, double* Y, float* Y32, const int* skip, int64_t r0, int64_t r1);
size_t gemm_i8_part_bytes(int64_t m_pad, int p, int num_sms);
void gemm_geometry(int64_t m, int64_t m_pad, int p, int num_sms, bool fp32, int* BM, int* KS, int* RB, int* KT);
size_t gemm_part_bytes(int64_t m, int64_t m_pad, int p, int num_sms);
avd_status launch_project(Ctx* c, const float* X);         // k_project.cu
avd_status launch_select0_speculative(Ctx* c);
avd_status launch_select(Ctx* c, const float* X, int level, int rank);  // k_select.cu
avd_status launch_gather(Ctx* c, const float* X, int rank, int64_t* top_idx, double* rho);
avd_status launch_project_reduce(Ctx* c);                  // k_project.cu
bool project_tc_supported(const Ctx* c, const float* X); // k_project_tc.cu
avd_status launch_project_tc(Ctx* c, const float* X);    // k_project_tc.cu
avd_status launch_agg_reduce(Ctx* c);                      // k_select.cu
avd_status gf_prepare(Ctx* c);                             // k_gramfree.cu
avd_status gf_product(Ctx* c, const double* In, double* Y, float* Y32, const int* skip);
avd_status gf_diag(Ctx* c);
avd_status launch_trace(Ctx* c);                           // k_eig.cu
avd_status gram_product(Ctx* c, const double* In, double* Y);  // k_eig.cu

}  // namespace avd
