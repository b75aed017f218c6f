/*
 * avd_averis.h — C ABI of the Averis mean-residual NVFP4 forward GeMM, part of
 * paper_2603_10444_b200/libavd.so (sm_100a only; status codes and avd_last_error from avd.h).
 *
 * PAPER.md:391-429 (section "Averis", paragraph "Forward pass: activation mean--residual
 * splitting"), for activations X in R^{l x m} (l = b*s tokens) and weights W in R^{m x n}:
 *   mu_X   = (1/l) 1^T X
 *   X_R    = X - 1 mu_X
 *   mu_bar = Q_b(mu_X),  X_R_bar = Q_b(X_R),  W_bar = Q_b(W) PAPER.md:412-418
 *   Y_hat  = 1 (mu_bar W_bar) + X_R_bar W_bar              Eq. averis_forward
 * with Q_b = NVFP4: E2M1 values, one UE4M3 scale per 16 consecutive elements
 * along the contraction dimension m, one fp32 tensor scale g = amax / (6 * 448); the decision
 * arithmetic (fp32, in a fixed order) and the rounding rules are DESIGN.md readings A1-A8.
 * AVD_AVERIS_VANILLA computes the paper's baseline Q_b(X) Q_b(W) instead.
 *
 * Conventions: as avd.h.  *_dev pointers are device pointers on the context's device; every
 * output buffer is caller-owned; the library owns its workspace (allocated in
 * avd_averis_create, freed in avd_averis_destroy); device work is ordered on the context's
 * stream; errors are status codes with a thread-local message (avd_last_error).
 */
#ifndef AVD_AVERIS_H_
#define AVD_AVERIS_H_
#include <stddef.h>
#include <stdint.h>

#include "avd.h"

#ifdef __cplusplus
extern "C" {
#endif

/* flags */
#define AVD_AVERIS_STOCHASTIC 1 /* stochastic rounding of the E2M1 codes ("SR is applied
                                   by default"; A3: counter hash of (seed, tensor, index));
                                   default: nearest, ties to the even grid index */
#define AVD_AVERIS_VANILLA 2    /* no split: Y = Q_b(X) Q_b(W) (the paper's "Vanilla FP4")          */
#define AVD_AVERIS_TIMING 4     /* record CUDA events at the stage boundaries of each forward
                                   (read with avd_averis_stage_ms)                                  */
#define AVD_AVERIS_BF16_OUT 8   /* Y in bf16 (round to nearest even of the fp32 epilogue value: the
                                   output type of the paper's FP4 training GeMMs); default fp32     */

typedef struct {
  int64_t l;       /* tokens (rows of X and Y), >= 1                                     */
  int64_t m;       /* contraction dimension (columns of X, rows of W); multiple of 32     */
  int64_t n;       /* output features (columns of W and Y); multiple of 16                */
  int32_t flags;   /* AVD_AVERIS_* */
  uint64_t seed;   /* stochastic-rounding seed (ignored for nearest rounding)              */
  int32_t device;  /* CUDA device ordinal; must be sm_100                                  */
  void* stream;    /* cudaStream_t the work is ordered on (NULL: the legacy default stream) */
} avd_averis_config;

typedef struct avd_averis_ctx* avd_averis_handle;

/* Allocate the workspace (codes and scales of X_R and W, mu, partial sums; about
 * (l + n) * m * 0.5625 bytes + 48 * ceil(l / 148) * m bytes).  EINVAL: l < 1, m % 32, n % 16,
 * m < 32, n < 16; ECUDA: not an sm_100 device or allocation failed. */
avd_status avd_averis_create(const avd_averis_config* cfg, avd_averis_handle* out);
avd_status avd_averis_destroy(avd_averis_handle h);

/* W_bar = Q_b(W) from W_dev (fp32, row-major [m][n], 16-byte aligned; read only, not retained).
 * Must precede avd_averis_forward; call again whenever W changes.  Returns before the device
 * work completes (stream-ordered). */
avd_status avd_averis_set_weight(avd_averis_handle h, const float* W_dev);

/* Y_dev (row-major [l][n], fp32 — or bf16 with AVD_AVERIS_BF16_OUT —, caller-owned) = Eq.
 * averis_forward for X_dev (fp32, row-major [l][m], 16-byte aligned, finite).  Stream-ordered,
 * returns without synchronising.  ESTATE: no weight set. */
avd_status avd_averis_forward(avd_averis_handle h, const float* X_dev, void* Y_dev);

/* The same from host memory: copies X_host (l*m fp32) in, runs avd_averis_forward, copies Y
 * (l*n fp32 or bf16) out to Y_host; synchronises the stream before returning.  Pinned host
 * buffers are copied asynchronously, pageable ones synchronously. */
avd_status avd_averis_forward_host(avd_averis_handle h, const float* X_host, void* Y_host);

/* Workspace buffers for checks (device pointer and byte size; valid until destroy):
 *   AVD_AV_MU      f64 [m]   mu_X (zero with AVD_AVERIS_VANILLA)
 *   AVD_AV_XCODES  u8  [l_pad][m/2]  E2M1 codes of X_R, element k of a row in nibble k%2 of
 *                                    byte k/2 (even k: low nibble); code = sign<<3 | grid index
 *   AVD_AV_XSF     u8  UE4M3 block scales of X_R in the tensor-core layout: the scale of row r,
 *                      block b (elements 16b..16b+15) is at byte
 *                      ((r/128) * KB4 + b/4) * 512 + (r%32) * 16 + ((r%128)/32) * 4 + b%4,
 *                      KB4 = 4 * ceil(m / 256)
 *   AVD_AV_WCODES  u8  [n_pad][m/2]  codes of W, row j = column j of W (blocks along m)
 *   AVD_AV_WSF     u8  scales of W, same layout as XSF with r = j
 *   AVD_AV_MUCODES u8  [m/2]     codes of mu_bar (same nibble order)
 *   AVD_AV_MUSF    u8  [m/16]    UE4M3 scales of mu_bar, plain order
 *   AVD_AV_GSCALE  f32 [4]       g of X_R, W, mu_bar, and the tensor amax of X_R
 *   AVD_AV_BIAS    f32 [n]       mu_bar W_bar (zero with AVD_AVERIS_VANILLA)
 * l_pad = 256 * ceil(l / 256), n_pad = 256 * ceil(n / 256).  EINVAL: unknown id. */
#define AVD_AV_MU 0
#define AVD_AV_XCODES 1
#define AVD_AV_XSF 2
#define AVD_AV_WCODES 3
#define AVD_AV_WSF 4
#define AVD_AV_MUCODES 5
#define AVD_AV_MUSF 6
#define AVD_AV_GSCALE 7
#define AVD_AV_BIAS 8
avd_status avd_averis_buffer(avd_averis_handle h, int32_t which, void** dev, size_t* bytes);

/* Kernels this context has launched so far (for the bench's gpu_launches). */
int64_t avd_averis_launch_count(avd_averis_handle h);

/* Stage times of the last avd_averis_forward (needs AVD_AVERIS_TIMING; waits for its end), ms:
 * ms[0] column statistics + mu_bar + bias, ms[1] quantisation of X_R, ms[2] the NVFP4 GeMM.
 * EINVAL: no AVD_AVERIS_TIMING. */
avd_status avd_averis_stage_ms(avd_averis_handle h, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* AVD_AVERIS_H_ */
