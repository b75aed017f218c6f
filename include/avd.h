/*
 * avd.h — C ABI of the B200-native activation outlier-attribution pass
 * (arXiv 2603.10444, section "Mean Bias as the Dominant Source of Activation Outliers",
 * PAPER.md:1-27).  Library: paper_2603_10444_b200/libavd.so (sm_100a only).
 *
 * For an fp32 activation matrix X (l = b*s tokens x m hidden, row-major) the pass computes
 *   mu      = (1/l) X^T 1
 *   Xc      = X - 1 mu^T
 *   spike   = rank-k truncated SVD of Xc, k = floor(0.01 m)
 *             (V_k, sigma_k from the top-k eigenpairs of G = Xc^T Xc)
 *   tail    = Xc - spike
 *   energies ||X||^2 = ||M||^2 + ||spike||^2 + ||tail||^2
 *   E_top   = top 0.1% entries by |X_ij|
 *   rho     = M_ij^2/X_ij^2, spike_ij^2/X_ij^2, tail_ij^2/X_ij^2
 *   cross   = 1 - sum(rho)   (the "minor cross-terms")
 * Readings of the paper where it is silent are listed in DESIGN.md ("Readings" R1..R13).
 *
 * Conventions (all entry points):
 *   - Pointers named *_dev are CUDA device pointers on the context's device; *_host are host.
 *   - Every output buffer is caller-owned; the library keeps no caller pointer after return.
 *   - The library owns its workspace (device memory allocated in avd_create, freed in
 *     avd_destroy); avd_plan reports its size before creation.
 *   - All device work is stream-ordered on the context's stream.  Entry points that return
 *     host scalars synchronise that stream before returning.
 *   - Errors are status codes (never aborts or exceptions); avd_last_error() gives a
 *     thread-local message for the last failing call.
 *   - Results are deterministic for fixed (X, seed, world size): the Gram is accumulated
 *     exactly in integers, and every floating-point reduction has a fixed order.
 *   - Row sharding (world > 1): rank r owns rows [row_offset, row_offset + l_local) of the
 *     global matrix; linear indices are global (i * m + j).  Between the stage entry points
 *     the caller all-reduces the buffers avd_buffer() exposes (see paper_2603_10444_b200/
 *     distributed.py); with world == 1 avd_decompose runs the whole pass.
 */
#ifndef AVD_H_
#define AVD_H_
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AVD_OK = 0,
  AVD_EINVAL = 1,      /* bad sizes / fractions / pointers / alignment / workspace        */
  AVD_ENONFINITE = 2,  /* X contains NaN or Inf (R5)               */
  AVD_ENOCONV = 3,     /* eigensolver hit max_iters before eig_tol; outputs still written */
  AVD_ECUDA = 4,       /* a CUDA runtime / driver call failed                             */
  AVD_ENOMEM = 6,      /* device allocation failed                                       */
  AVD_ESTATE = 8,      /* stage called out of order                                      */
  AVD_EREPEAT = 9,     /* (stage API only) avd_stage_eig raised the Gram operand to 3 digits:
                          call avd_stage_gram again (exchange GRAM, QSUM, QERR), then
                          avd_stage_eig; avd_decompose handles this internally              */
  AVD_EEXCHANGE = 10   /* an exchange callback (avd_exchange_fn) returned nonzero            */
} avd_status;

/* Sizes derived from (l, m, fractions) — DESIGN.md R1, R2:
 *   k     = max(1, floor(k_frac * m))          ("k = floor(0.01 m)")
 *   n_top = max(1, floor(top_frac * l * m))    ("top 0.1%")
 * floor(f*n) is taken as round(f*n) when |f*n - round(f*n)| < 1e-9.                     */
typedef struct {
  int32_t k;               /* spike rank                                                    */
  int32_t p;               /* subspace-iteration block size = roundup16(k + 8)              */
  int64_t n_top;           /* |E_top| requested (global)                                    */
  int32_t digits;          /* int8 digit planes the Gram STARTS with (2 or 3; see avd_config) */
  size_t workspace_bytes;  /* device bytes avd_create will allocate                         */
} avd_plan_t;

typedef struct {
  int64_t l_global;        /* global rows l (>= 2)                                           */
  int64_t l_local;         /* rows held by this rank (== l_global when world == 1)           */
  int64_t row_offset;      /* first global row of this rank                                  */
  int64_t m;               /* columns (>= 2)                                                 */
  double k_frac;           /* 0.01; used when k_override == 0                  */
  double top_frac;         /* 0.001; used when n_top_override == 0             */
  int32_t k_override;      /* > 0: use this k                                                */
  int64_t n_top_override;  /* > 0: use this |E_top|                                          */
  uint64_t seed;           /* start block of the subspace iteration + Gram dither            */
  int32_t max_iters;       /* subspace iterations cap (0 -> 200)                             */
  double eig_tol;          /* Ritz residual tolerance relative to lambda_1 (0 -> 1e-6)       */
  int32_t digits;          /* Gram operand = centred X in int8 digit planes:
                              0 (default) = automatic: 2 digits (14 bits of each column's
                              range), raised to 3 (21 bits) when the a-posteriori bound of the
                              quantisation error on sigma_k or on the spike/tail energy shares
                              exceeds half the north-star tolerance (1e-4 on sigma, 1e-5 on
                              the shares; see precision_sigma / precision_share); 2 or 3 = fixed */
  int32_t world;           /* ranks sharing the rows (1 = single GPU)                        */
  int32_t device;          /* CUDA device ordinal                                            */
  void* stream;            /* cudaStream_t (NULL = legacy default stream)                    */
  int32_t flags;           /* AVD_FLAG_* bits (0 = defaults)                                 */
} avd_config;

/* avd_config.flags: select E_top by streaming X even when the candidate list would do (tests) */
#define AVD_FLAG_STREAM_SELECT 1
/* avd_config.flags: quantise the Gram operand with the exact column ranges (the fallback taken
 * when the row-sampled ranges overflow the digit range; forced here for tests)               */
#define AVD_FLAG_EXACT_SCALE 2
/* avd_config.flags (tests): with automatic digits, take the 3-digit escalation (AVD_EREPEAT and
 * the re-encoded Gram) whatever the precision bound says                                      */
#define AVD_FLAG_FORCE_ESCALATE 4
/* avd_config.flags (tests / profiling): run the eigensolver's loop from the host, one kernel
 * launch and one synchronisation per decision, instead of the device-resident CUDA graph (the
 * same kernels in the same order: bit-identical results; env AVD_EIG_NOGRAPH=1 does the same)  */
#define AVD_FLAG_EIG_HOST_LOOP 8
/* avd_config.flags: also compute the top-k singular pairs of the UNCENTRED X (eigenpairs of
 * X^T X = G + l mu mu^T) and alpha_i = |mu . v_i| into
 * avd_outputs.mean_sigma_dev / mean_alpha_dev — about one eigensolve of extra work          */
#define AVD_FLAG_MEAN_TOPK 16
/* Gram-free eigensolve: the m x m Gram is never
 * formed; every product G Q of the subspace iteration is evaluated as Xhat^T (Xhat Q) by two
 * streaming tensor-core passes over the Gram operand's digit planes.  Same outputs and tolerances.
 * Single GPU only (world 1; EINVAL otherwise); not combinable with AVD_FLAG_MEAN_TOPK, and the
 * uncentred top pair of the mean-bias diagnostics (cos_mu_v1, alpha1, sigma1_u, resid_u,
 * iters_u) is not computed (NaN). */
#define AVD_FLAG_GRAM_FREE 32

/* Outputs.  Device arrays caller-owned, sized from the plan (cap = n_top). */
typedef struct {
  double* mu_dev;          /* [m] feature-wise mean mu                          */
  double* V_dev;           /* [m*k] row-major: V[j*k + r] = component j of v_r */
  double* sigma_dev;       /* [k] singular values of Xc, descending                          */
  int64_t* top_idx_dev;    /* [n_top] global linear indices i*m+j of THIS rank's part of
                              E_top, ascending (ties by smaller index, zeros excluded; R3,R4)*/
  double* rho_dev;         /* [n_top*4]: rho_mean, rho_spike, rho_tail, cross per entry      */
  /* host scalars written on return */
  int64_t n_top_local;     /* entries of E_top owned by this rank                            */
  int64_t top_offset;      /* position of this rank's slice inside the global E_top          */
  int64_t n_top_global;    /* |E_top| (< requested only if X has fewer nonzeros)             */
  double energy_cf[4];     /* closed forms: total = sum x^2, mean = l||mu||^2,
                              spike = sum_{r<k} sigma_r^2, tail = tr(G) - spike*/
  double energy_el[4];     /* elementwise: sum x^2, sum M^2, sum spike^2, sum tail^2         */
  double cross_el[3];      /* <M,spike>, <M,tail>, <spike,tail> Frobenius inner products     */
  double colmean_absmax[2];/* max_j |mean_i spike_ij|, max_j |mean_i tail_ij|  */
  double rho_mean_aggr[4]; /* mean over E_top of rho_mean, rho_spike, rho_tail, cross (R10)  */
  double rho_energy_aggr[3]; /* sum_E c^2 / sum_E x^2, c = M, spike, tail                    */
  double sigma_next;       /* sigma_{k+1}: the (k+1)-th Ritz value of the converged p-column
                              subspace, a LOWER bound of sigma_{k+1} (Cauchy interlacing),
                              typically within a few % (its residual is not part of the
                              convergence test); 0 when unavailable                          */
  double trace_g;          /* tr(G) = ||Xc||_F^2                                             */
  int32_t iters;           /* subspace iterations used                                       */
  double max_resid;        /* max_r<k ||G v_r - lambda_r v_r|| / lambda_1                     */
  int32_t rr_checks;      /* Rayleigh-Ritz checks of the eigensolver (diagnostic)           */
  int32_t jacobi_sweeps;   /* total sweeps of the p x p Jacobi solves (diagnostic)           */
  int32_t requantised;     /* 1 if the Gram operand was re-quantised with exact column ranges */
  int32_t digits_used;     /* digit planes of the final Gram (3 after an automatic escalation) */
  double precision_sigma;  /* 5-sigma bound of the relative error of sigma_r (max over r < k)
                              from the operand's quantisation noise: the first-order
                              perturbation of lambda_r by the dithered rounding errors e_ia
                              (|E e| = 0, var e <= 1/4 in units of the column step d_a):
                              std(d lambda_r) <= sigma_r sqrt(sum_a d_a^2 v_ra^2)            */
  double precision_share;  /* 5-sigma bound of |d share| / share for the spike and tail shares:
                              std(d E_spike) <= sqrt(sum_a d_a^2 sum_r lambda_r v_ra^2)       */
  /* mean-bias diagnostics ("Mean bias phenomenon"; Eq. R):
   *   p_i = x_i^T mu_hat (mu_hat = mu / ||mu||); sign_fraction = max(#p_i > 0, #p_i < 0) / l
   *   (-1 when unavailable: m % 4 != 0 projection path; 0 when mu = 0);
   *   R = ||mu|| / sqrt(||X||_F^2 / l);  v_1, sigma_1 = top right singular pair of the UNCENTRED
   *   X (eigenpair of X^T X = G + l mu mu^T); alpha_1 = (sigma_1 / l) u_1^T 1 = mu . v_1 (sign of
   *   v_1 chosen so alpha_1 >= 0); cos_mu_v1 = |mu_hat . v_1| (0 when mu = 0)                    */
  double mean_R;
  double sign_fraction;
  int64_t p_pos, p_neg;
  double cos_mu_v1;
  double alpha1;
  double sigma1_u;
  double resid_u;          /* ||Gu v - lambda v|| / lambda of the uncentred power iteration     */
  int32_t iters_u;         /* its steps                                                         */
  /* AVD_FLAG_MEAN_TOPK: the top k uncentred pairs (caller-owned [k] arrays, device — host for
   * avd_decompose_host —, NULL = not wanted): sigma_i of X and alpha_i = |mu . v_i|, the
   * coefficients of mu = sum_i alpha_i v_i (cos(mu_hat, v_i) = alpha_i/||mu||) */
  double* mean_sigma_dev;
  double* mean_alpha_dev;
  int32_t iters_uk;        /* subspace steps of that solve (0 when not requested)              */
  double resid_uk;         /* its max_i<k ||Gu v_i - lambda_i v_i|| / lambda_1                  */
} avd_outputs;

typedef struct avd_ctx avd_ctx;

/* Sizes and workspace for a configuration (no device work).  AVD_EINVAL when l_global < 2,
 * m < 2, k > min(l, m), a fraction outside (0, 1], p > 112, or the row
 * shard is inconsistent.                                                                    */
avd_status avd_plan(const avd_config* cfg, avd_plan_t* plan);  /* k <= 95 */

/* Allocate the workspace on cfg->device and bind cfg->stream.  *ctx is NULL on failure.     */
avd_status avd_create(const avd_config* cfg, avd_ctx** ctx);
void avd_destroy(avd_ctx* ctx);
avd_status avd_get_plan(const avd_ctx* ctx, avd_plan_t* plan);

/* The whole pass on one GPU (cfg.world == 1).  X_dev: device, row-major l x m fp32, 16-byte
 * aligned, read only, not retained.  out: device arrays (see avd_outputs) + host scalars.
 * Blocks until outputs are ready.  AVD_ENONFINITE if X has NaN/Inf (outputs untouched);
 * AVD_ENOCONV if the eigensolver hit max_iters (outputs written, iters/max_resid tell).     */
avd_status avd_decompose(avd_ctx* ctx, const float* X_dev, avd_outputs* out);

/* Same pass from HOST memory: X_host (l x m fp32, pinned or pageable) is copied to an
 * internal device buffer (allocated on first use, freed by avd_destroy); out's array fields
 * are HOST pointers here and receive the results by device-to-host copy.                   */
avd_status avd_decompose_host(avd_ctx* ctx, const float* X_host, avd_outputs* out);

/* ---- stage entry points (row-sharded, world >= 1) -------------------------------------
 * Call in this order; after each stage the caller all-reduces (over all ranks, in place)
 * the buffers listed, then calls the next stage.  With world == 1 no exchange is needed.
 *   avd_stage_stats    (row sample, global rows i % s == 0, s = 16 at l >= 64k: column sums,
 *                       max, min, and on every 4th sampled row the |x| histogram bits 30:19;
 *                       they seed the quantiser centre / scale and the candidate bin b0)
 *       exchange: AVD_BUF_SAMPLE (f64, SUM), AVD_BUF_SMAX (f32, MAX), AVD_BUF_SMIN (f32, MIN),
 *                 AVD_BUF_HIST1 (i64, SUM)
 *   avd_stage_split    (the fused pass over X: fp64 column sums, sum x^2, #nonzero, the exact
 *                       column range about the quantiser centre, the centred int8 digit planes of
 *                       the Gram operand with their integer column sums and squared rounding
 *                       errors, the top-set candidates)
 *       exchange: AVD_BUF_STATS (f64, SUM), AVD_BUF_COLMAX (f32, MAX: max |x - quantiser centre|),
                 AVD_BUF_DIAG (f64, SUM: sum_i (x_ij - centre_j)^2, the exact diagonal of G)
 *   avd_stage_gram     (mu; AVD_ENONFINITE if X has NaN/Inf; re-quantisation with the exact
 *                       ranges if any rank's digits overflowed; K3 tcgen05 int8 Gram, exact int64;
 *                       with world > 1 its upper 128-tiles are also packed into AVD_BUF_GRAMP)
 *       exchange: AVD_BUF_GRAMP (i64, SUM; world > 1 — avd_stage_eig unpacks it),
 *                 AVD_BUF_CAND (i64, SUM), AVD_BUF_QSUM (i64, SUM), AVD_BUF_QERR (f64, SUM)
 *   avd_stage_eig      (exact centring of the Gram, K4 subspace iteration + Rayleigh-Ritz, and
 *                       the top eigenpair of the uncentred Gram G + l mu mu^T; replicated on every
 *                       rank)
 *   avd_stage_project  (K5+K8 projections P = Xc V_k and elementwise energies, counts of the
 *                       signs of p_i = x_i . mu_hat)
 *       exchange: AVD_BUF_ENERGY (f64, SUM)
 *   avd_stage_select(level 0)  (K6 exact |x| histogram, bits 30:19)  exchange: AVD_BUF_HIST0 (i64, SUM)
 *   avd_stage_select(level 1)  (K6 bits 18:7 inside bin b1)          exchange: AVD_BUF_HIST2 (i64, SUM)
 *   avd_stage_select(level 2)  (K6 bits 6:0 inside (b1, b2))         exchange: AVD_BUF_HIST3 (i64, SUM)
 *   avd_stage_select(level 3)  (K6 threshold T, mark, per-rank counts) exchange: AVD_BUF_TIES (i64, SUM)
 *   avd_stage_gather   (K6 ordered compaction with the rank's tie quota, K7 rho gather)
 *       exchange: AVD_BUF_AGG (f64, SUM)
 *   avd_stage_report   (host scalars into out)
 * The K6 histograms read the candidate list (entries with |x| bits >= bin b0 chosen from the
 * row-sampled histogram), or stream X itself when the exchanged candidate count does not cover
 * |E_top| or a rank overflowed its candidate capacity; both give the exact same E_top.        */
typedef enum {
  AVD_BUF_STATS = 0, AVD_BUF_COLMAX = 1, AVD_BUF_COLMIN = 2, AVD_BUF_HIST1 = 3,
  AVD_BUF_GRAM = 4, AVD_BUF_ENERGY = 5, AVD_BUF_HIST2 = 6, AVD_BUF_HIST3 = 7,
  AVD_BUF_TIES = 8, AVD_BUF_AGG = 9, AVD_BUF_HIST0 = 10, AVD_BUF_CAND = 11,
  AVD_BUF_SAMPLE = 12, AVD_BUF_SMAX = 13, AVD_BUF_SMIN = 14, AVD_BUF_QSUM = 15, AVD_BUF_QERR = 21,
  AVD_BUF_DIAG = 22,
  AVD_BUF_GRAMP = 25,  /* the Gram's upper 128-tiles, packed (i64, SUM): what world > 1 exchanges
                          after avd_stage_gram (half the bytes of AVD_BUF_GRAM)               */
  AVD_BUF_EIGZ = 23,   /* distributed eigensolve: Z = G Q, m x p f64 (SUM of row blocks)     */
  AVD_BUF_EIGY = 24,   /* distributed eigensolve: Y = G Z or G Q, m x p f64 (SUM of row blocks) */
  /* read-only views for tests / diagnostics (not exchanged) */
  AVD_BUF_MU = 16, AVD_BUF_G = 17, AVD_BUF_P = 18, AVD_BUF_DIGITS = 19, AVD_BUF_SCALE = 20
} avd_buffer_id;

/* Device pointer and byte size of a workspace buffer (valid until avd_destroy). */
avd_status avd_buffer(avd_ctx* ctx, int32_t which, void** dev_ptr, size_t* bytes);

avd_status avd_stage_stats(avd_ctx* ctx, const float* X_dev);
avd_status avd_stage_split(avd_ctx* ctx, const float* X_dev);
avd_status avd_stage_gram(avd_ctx* ctx, const float* X_dev);
avd_status avd_stage_eig(avd_ctx* ctx);
avd_status avd_stage_project(avd_ctx* ctx, const float* X_dev);
avd_status avd_stage_select(avd_ctx* ctx, const float* X_dev, int32_t level, int32_t rank);
avd_status avd_stage_gather(avd_ctx* ctx, const float* X_dev, int32_t rank, avd_outputs* out);
avd_status avd_stage_report(avd_ctx* ctx, avd_outputs* out);

/* ---- library-driven exchanges (row-sharded, world >= 1) --------------------------------
 * An exchange callback all-reduces IN PLACE, over all ranks, `count` elements of type `dtype`
 * at buf_dev (device; the workspace buffer `which`, avd_buffer_id) with `op`, stream-ordered
 * after the library's work on the context's stream (e.g. ncclAllReduce on that stream, or a
 * synchronous host-staged all-reduce).  Returns 0 on success; anything else aborts the call with
 * AVD_EEXCHANGE.                                                                              */
typedef enum { AVD_DT_F64 = 0, AVD_DT_F32 = 1, AVD_DT_I64 = 2 } avd_dtype;
typedef enum { AVD_OP_SUM = 0, AVD_OP_MAX = 1, AVD_OP_MIN = 2 } avd_op;
typedef int (*avd_exchange_fn)(int32_t which, void* buf_dev, int32_t dtype, int32_t op, size_t count,
                               void* user);

/* Distributed eigensolve: avd_stage_eig with every G Q product split by row
 * blocks over the ranks (rank r computes rows [r0, r1) of its share of the 128-row blocks); the
 * zero-padded products are exchanged through fn as SUMs (AVD_BUF_EIGZ, AVD_BUF_EIGY, both f64 —
 * i.e. all-gathers), twice per power step and once per Rayleigh-Ritz check; the p x p work is
 * replicated.  Same results as avd_stage_eig up to the row blocking of the GEMM partial sums.
 * world == 1 or fn == NULL: exactly avd_stage_eig.  May return AVD_EREPEAT like avd_stage_eig. */
avd_status avd_stage_eig_dist(avd_ctx* ctx, int32_t rank, avd_exchange_fn fn, void* user);

/* The whole row-sharded pass for a C caller: every stage in order, every exchange listed above
 * through fn (with world > 1 the Gram goes as AVD_BUF_GRAMP), the distributed eigensolve, the
 * 3-digit repeat.  X_dev: this rank's rows (cfg.l_local x m).  world == 1 with fn == NULL is
 * avd_decompose.                                                                              */
avd_status avd_decompose_sharded(avd_ctx* ctx, const float* X_dev, int32_t rank, avd_outputs* out,
                                 avd_exchange_fn fn, void* user);

/* A ready-made avd_exchange_fn over NCCL: user = &(avd_nccl_comm){comm, stream}, comm an
 * ncclComm_t of the `world` ranks in row order, stream the context's cudaStream_t.  Issues
 * ncclAllReduce(buf, buf, count, type, op, comm, stream) (libnccl.so.2 is loaded at first use;
 * returns nonzero when it cannot be loaded or the call fails).                                */
typedef struct { void* comm; void* stream; } avd_nccl_comm;
int avd_exchange_nccl(int32_t which, void* buf_dev, int32_t dtype, int32_t op, size_t count, void* user);

/* Tie quota of `rank` (R3): E_top takes the first q entries with key == T in global
 * linear order and rows are sharded in rank order, so rank r takes
 *   quota_r  = clamp(q - sum_{r'<r} tie_counts[r'], 0, tie_counts[r])
 *   offset_r = sum_{r'<r} (sel_counts[r'] + quota_r')   (position of its slice in E_top).
 * sel_counts / tie_counts: host arrays [world] of per-rank counts of key > T / key == T.
 * Host-only integer logic (no device work); used by avd_stage_gather.                       */
avd_status avd_tie_quota(const int64_t* sel_counts, const int64_t* tie_counts, int32_t world,
                         int32_t rank, int64_t q, int64_t* quota, int64_t* offset);

/* Y_dev = G In_dev for the context's Gram operand G = Xhat^T Xhat (Xhat: the quantised, exactly
 * centred matrix the eigensolve used): the formed fp64 G, or with
 * AVD_FLAG_GRAM_FREE the two streaming tensor-core passes Xhat^T (Xhat In).
 * In_dev, Y_dev: device fp64 row-major [m][p] (p from the plan), caller-owned.  Valid after the
 * eigen stage (or avd_decompose) of this context; synchronises.  ESTATE before that.  For checks
 * of the product itself (tests) and callers that reuse the operand for further subspace work. */
avd_status avd_gram_product(avd_ctx* ctx, const double* In_dev, double* Y_dev);

/* Number of kernels this context launched since creation (for the bench's gpu_launches). */
int64_t avd_launch_count(const avd_ctx* ctx);

const char* avd_strerror(avd_status s);
const char* avd_last_error(void); /* thread-local message of the last failing call */

#ifdef __cplusplus
}
#endif
#endif /* AVD_H_ */
