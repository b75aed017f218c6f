// avd.cu — C ABI (include/avd.h): plan, workspace, stage orchestration and the one-call pass.
// Every numerical step runs in the kernels of k_*.cu; this file only validates arguments,
// carves the workspace, launches, and copies the final scalars.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <unordered_map>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "common.cuh"

namespace avd {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

cudaError_t smem_attr_impl(const void* fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> set;  // one process drives one device
  std::lock_guard<std::mutex> lk(mu);
  int& cur = set[fn];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

namespace {

int64_t floor_frac(double f, int64_t n) {
  const double v = f * (double)n;
  const double r = std::nearbyint(v);
  return std::fabs(v - r) < 1e-9 ? (int64_t)r : (int64_t)std::floor(v);
}

struct Layout {
  // byte offsets inside the single workspace allocation
  size_t off[128];
  size_t total = 0;
  int n = 0;
  size_t add(size_t bytes) {
    if (n >= 128) return (size_t)n;  // make_plan checks n against the bound below
    total = (total + 255) & ~size_t(255);
    off[n] = total;
    total += bytes;
    return (size_t)n++;
  }
};

avd_status make_plan(const avd_config* cfg, avd_plan_t* plan, Ctx* c, Layout* lay) {
  if (!cfg || !plan) { set_error("null argument"); return AVD_EINVAL; }
  const int64_t l = cfg->l_global, m = cfg->m;
  if (l < 2 || m < 2) { set_error("l and m must be >= 2 (SPEC.md:225)"); return AVD_EINVAL; }
  const int world = cfg->world <= 0 ? 1 : cfg->world;
  if (cfg->l_local < 1 || cfg->row_offset < 0 || cfg->row_offset + cfg->l_local > l ||
      (world == 1 && (cfg->l_local != l || cfg->row_offset != 0))) {
    set_error("inconsistent row shard");
    return AVD_EINVAL;
  }
  if (cfg->k_override <= 0 && !(cfg->k_frac > 0.0 && cfg->k_frac <= 1.0)) { set_error("k_frac must be in (0,1]"); return AVD_EINVAL; }
  if (cfg->n_top_override <= 0 && !(cfg->top_frac > 0.0 && cfg->top_frac <= 1.0)) { set_error("top_frac must be in (0,1]"); return AVD_EINVAL; }
  const int64_t k = cfg->k_override > 0 ? cfg->k_override : std::max<int64_t>(1, floor_frac(cfg->k_frac, m));
  if (k > std::min(l, m)) { set_error("k > min(l, m) (SPEC.md:227)"); return AVD_EINVAL; }
  const int64_t p = ((k + 8 + 15) / 16) * 16;
  if (p > kMaxP || k > 95) { set_error("k too large for this build (p <= 112, k <= 95)"); return AVD_EINVAL; }
  const int64_t n_top = cfg->n_top_override > 0 ? cfg->n_top_override : std::max<int64_t>(1, floor_frac(cfg->top_frac, l * m));
  const int nd = cfg->digits == 0 ? 2 : cfg->digits;
  if (nd != 2 && nd != 3) { set_error("digits must be 0 (automatic), 2 or 3"); return AVD_EINVAL; }
  const int nd_max = cfg->digits == 0 ? 3 : nd;
  if ((cfg->flags & AVD_FLAG_GRAM_FREE) && (world > 1 || (cfg->flags & AVD_FLAG_MEAN_TOPK))) {
    set_error("AVD_FLAG_GRAM_FREE needs world == 1 and excludes AVD_FLAG_MEAN_TOPK");
    return AVD_EINVAL;
  }
  plan->k = (int32_t)k;
  plan->p = (int32_t)p;
  plan->n_top = n_top;
  plan->digits = nd;

  Ctx tmp;
  Ctx* C = c ? c : &tmp;
  C->cfg = *cfg;
  C->cfg.world = world;
  C->k = (int)k;
  C->p = (int)p;
  C->k_pad = (int)(((k + 1 + 15) / 16) * 16);  // + one column: the mean direction (diagnostics)
  C->nd = nd;
  C->nd_max = nd_max;
  C->auto_digits = cfg->digits == 0;
  C->gram_free = (cfg->flags & AVD_FLAG_GRAM_FREE) != 0;
  C->m_pad = round_up(m, kGramTile);
  C->m_pad32 = round_up(m, 32);
  C->l_pad = round_up(cfg->l_local, kGramK);
  const int64_t ll = cfg->l_local;
  const int ncb = (int)ceil_div(m, 256LL * ((m % 4 == 0) ? 4 : 1));
  C->r1 = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(4LL * C->num_sms, ncb), ceil_div(ll, 4)));
  C->r1 = (int)std::max<int64_t>(C->r1, ceil_div(ll, 65536));  // int32 per-chunk sums of q (k_pass1.cu)
  // + room for the holes of the per-warp slot blocks (k_pass1.cu kCandBlk)
  C->cand_cap = std::min<int64_t>(ll * m, std::max<int64_t>(4 * n_top, 1 << 20) + (1 << 18));
  C->n_red = (int)ceil_div(m, kRedRowsC);  // partials of the m-length p x p reductions
  C->n_proj_ctas = (int)ceil_div(ll, 32);
  C->nwords = ceil_div(ll * m, 32);
  C->nblk = ceil_div(C->nwords, 1024);
  C->n_gather_ctas = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_top, 256), 4LL * C->num_sms));

  Layout L;
  L.add(sizeof(double) * C->r1 * m);            // 0 colsum_part
  L.add(sizeof(float) * C->r1 * m);             // 1 colmax_part
  L.add(sizeof(float) * C->r1 * m);             // 2 colmin_part
  L.add(sizeof(double) * C->r1 * ncb);          // 3 sq_part
  L.add(sizeof(double) * (m + 4));              // 4 stats
  L.add(sizeof(float) * m);                     // 5 colmax
  L.add(sizeof(float) * m);                     // 6 colmin
  L.add(sizeof(unsigned long long) * kHistBins);// 7 hist1
  L.add(sizeof(double) * m);                    // 8 mu
  L.add(sizeof(int32_t) * C->m_pad);            // 9 shift
  L.add(sizeof(DevPlan));                       // 10 dplan
  L.add((size_t)nd_max * C->m_pad * C->l_pad);  // 11 digits
  L.add(sizeof(uint32_t) * C->cand_cap);        // 12 cand_key
  L.add(sizeof(uint64_t) * C->cand_cap);        // 13 cand_idx
  L.add(2 * sizeof(unsigned long long));        // 14 cand_cnt [slot cursor, real count]
  L.add(sizeof(long long) * C->m_pad * C->m_pad);// 15 gram_i
  L.add(sizeof(double) * C->m_pad * C->m_pad);  // 16 G
  L.add(sizeof(double) * m * p);                // 17 Q
  L.add(sizeof(double) * m * p);                // 18 Y
  L.add(sizeof(double) * m * p);                // 19 Z
  L.add(sizeof(double) * m * p);                // 20 U
  L.add(sizeof(double) * p * p);                // 21 H
  L.add(sizeof(double) * p * p);                // 22 W
  L.add(sizeof(double) * 2 * p);                // 23 theta
  L.add(sizeof(double) * C->n_red * p * p);     // 24 red_part
  L.add(sizeof(double) * (4 * p + 8));          // 25 resid (+ flags, + scratch of the uncentred top-k)
  L.add(sizeof(double) * 4);                    // 26 trace
  L.add(sizeof(double) * m * k);                // 27 V
  L.add(sizeof(double) * k);                    // 28 sigma
  L.add(sizeof(float) * m * C->k_pad);          // 29 V32
  L.add(sizeof(float) * ll * C->k_pad);         // 30 P
  L.add(sizeof(double) * C->n_proj_ctas * 4);   // 31 en_part
  L.add(sizeof(double) * C->n_proj_ctas * C->k_pad);  // 32 colsumP_part
  L.add(sizeof(double) * (6 + C->k_pad));       // 33 energy (+ #p_i > 0, #p_i < 0)
  L.add(sizeof(unsigned long long) * kHistBins);// 34 hist2
  L.add(sizeof(unsigned long long) * kHist3Bins);// 35 hist3
  L.add(sizeof(long long) * 2 * world);         // 36 ties
  L.add(sizeof(uint32_t) * C->nwords);          // 37 bm_sel
  L.add(sizeof(uint32_t) * C->nwords);          // 38 bm_tie
  L.add(sizeof(int64_t) * (2 * C->nblk + 2));   // 39 blk_cnt
  L.add(sizeof(double) * 8);                    // 40 agg
  L.add(sizeof(double) * 8 * C->n_gather_ctas); // 41 agg_part
  L.add(sizeof(double) * 16);                   // 42 report
  L.add(sizeof(unsigned long long) * kHistBins);// 43 hist0
  L.add(sizeof(long long) * 2);                 // 44 cand_x
  L.add(gemm_part_bytes(m, C->m_pad, (int)p, C->num_sms));  // 45 gemm_part
  L.add((size_t)3 * C->l_pad * 128);                                     // 46 Pd
  L.add(std::max<size_t>(sizeof(float) * 2 * C->k_pad * round_up(m, 32), (size_t)4 * C->k_pad * C->m_pad));  // 47 Vt_hl / W digits
  L.add((size_t)3 * C->m_pad * 128);                                     // 48 Vd
  L.add(sizeof(float) * 2 * C->m_pad);                                   // 49 mu_hl
  L.add(sizeof(float) * C->m_pad * C->m_pad);                            // 50 G32
  L.add(sizeof(long long) * 2 * C->m_pad);                               // 51 qsum
  L.add(sizeof(float) * m * p);                                          // 52 Q32
  L.add(sizeof(float) * m * p);                                          // 53 Z32
  L.add(sizeof(unsigned) * 4);                                           // 54 ticket
  L.add(sizeof(double));                                                 // 55 gmax
  L.add(sizeof(double) * (m + 1));                                       // 56 samp
  L.add(sizeof(float) * m);                                              // 57 smax
  L.add(sizeof(float) * m);                                              // 58 smin
  L.add(sizeof(float) * C->m_pad);                                       // 59 qscale
  L.add(sizeof(float) * C->m_pad);                                       // 60 qoff
  L.add(sizeof(long long) * C->r1 * m);                                  // 61 qsum_part
  L.add(sizeof(long long) * 2 * C->m_pad);                               // 62 qsum_local
  L.add(sizeof(float) * C->r1 * m);                                      // 63 qerr_part
  L.add(sizeof(double) * C->m_pad);                                      // 64 qerr_local
  L.add(sizeof(double) * C->m_pad);                                      // 65 qerr
  L.add(sizeof(float) * C->m_pad);                                       // 66 mu0
  L.add(sizeof(long long) * C->r1 * m);                                  // 67 qsq_part
  L.add(sizeof(double) * (4 + 2 * C->m_pad));                            // 68 diag: |mu|, scratch, q, y
  L.add(sizeof(double) * kMaxP);                                         // 69 prec
  L.add(sizeof(double) * m);                                             // 70 ysq
  L.add(kEigCtlBytes);                                                   // 71 eig_ctl
  L.add(sizeof(double) * 512);                                           // 72 wsc (+ spiky list at 384)
  {
    const int64_t T = C->m_pad / 128;
    L.add(world > 1 ? sizeof(long long) * (size_t)(T * (T + 1) / 2) * 128 * 128 : 0);  // 73 gram_p
  }
  L.add((size_t)4 * C->m_pad * C->m_pad);                               // 74 gd
  L.add(sizeof(double) * C->m_pad);                                      // 75 gsc
  L.add((size_t)3 * kMaxP * C->m_pad);                                   // 76 qd
  L.add(sizeof(double) * 2 * kMaxP);                                     // 77 qsc (+ column maxima)
  L.add(gemm_i8_part_bytes(C->m_pad, (int)p, C->num_sms));               // 78 g8_part
  L.add(sizeof(unsigned) * (size_t)(C->m_pad / 128 + 1));                // 79 g8_tickets
  L.add(2 * sizeof(CUtensorMap));                                        // 80 tm_dev
  L.add(sizeof(double) * 2 * kMaxP);                                     // 81 unc_topk
  L.add(sizeof(float) * C->l_pad);                                       // 82 ps
  L.add(sizeof(float) * C->m_pad);                                       // 83 vs
  if (L.n >= 128) { set_error("workspace layout table overflow"); return AVD_EINVAL; }
  plan->workspace_bytes = L.total;
  if (lay) *lay = L;
  return AVD_OK;
}

// colmean maxima and <M,spike>, <M,tail>, l||mu||^2: one thread per column, per-CTA partials
// (fixed order) + a one-CTA finish
__global__ void report_part_kernel(const double* __restrict__ energy, const double* __restrict__ stats,
                                   const double* __restrict__ mu, const double* __restrict__ V, int64_t m, int k,
                                   int64_t l_global, double* __restrict__ part) {
  __shared__ double sh[5][256];
  const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double ms = 0, mt = 0, as = 0, at = 0, mu2 = 0;
  if (j < m) {
    const double inv_l = 1.0 / (double)l_global;
    double cs = 0.0;  // sum_i spike_ij = sum_r (1^T P)_r V_jr
    for (int r = 0; r < k; ++r) cs = fma(energy[4 + r], V[j * k + r], cs);
    const double cxc = stats[j] - (double)l_global * mu[j];  // sum_i xc_ij
    const double ct = cxc - cs;                              // sum_i tail_ij
    ms = mu[j] * cs;
    mt = mu[j] * ct;
    as = fabs(cs * inv_l);
    at = fabs(ct * inv_l);
    mu2 = mu[j] * mu[j];
  }
  sh[0][threadIdx.x] = ms; sh[1][threadIdx.x] = mt; sh[2][threadIdx.x] = as; sh[3][threadIdx.x] = at;
  sh[4][threadIdx.x] = mu2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + o];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + o];
      sh[2][threadIdx.x] = fmax(sh[2][threadIdx.x], sh[2][threadIdx.x + o]);
      sh[3][threadIdx.x] = fmax(sh[3][threadIdx.x], sh[3][threadIdx.x + o]);
      sh[4][threadIdx.x] += sh[4][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x < 5) part[(int64_t)blockIdx.x * 5 + threadIdx.x] = sh[threadIdx.x][0];
}
__global__ void report_final_kernel(const double* __restrict__ part, int nparts, int64_t l_global,
                                    double* __restrict__ rep) {
  if (threadIdx.x != 0) return;
  double a = 0, b = 0, c = 0, d = 0, e = 0;
  for (int q = 0; q < nparts; ++q) {
    a += part[q * 5]; b += part[q * 5 + 1]; c = fmax(c, part[q * 5 + 2]); d = fmax(d, part[q * 5 + 3]);
    e += part[q * 5 + 4];
  }
  rep[0] = a; rep[1] = b; rep[2] = c; rep[3] = d; rep[4] = (double)l_global * e;
}

// assemble the user's device outputs
__global__ void copy_outputs_kernel(const double* __restrict__ mu, const double* __restrict__ V,
                                    const double* __restrict__ sigma, int64_t m, int k, double* __restrict__ mu_o,
                                    double* __restrict__ V_o, double* __restrict__ sigma_o) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu_o && t < m) mu_o[t] = mu[t];
  if (V_o && t < m * k) V_o[t] = V[t];
  if (sigma_o && t < k) sigma_o[t] = sigma[t];
}

// gather the report's scalars into one contiguous block (one D2H copy instead of nine):
// [0,5) report, [8,16) agg, [16,20) energy, 20 sum x^2, 21 trace, [22,24) sign counts,
// 24 ||mu||, [32, 32+k) sigma, then the DevPlan words
constexpr int kPackHead = 32;
constexpr int kPlanWords = (int)((sizeof(DevPlan) + 7) / 8);
__global__ void report_pack_kernel(const double* __restrict__ report, const double* __restrict__ agg,
                                   const double* __restrict__ energy, const double* __restrict__ stats,
                                   const double* __restrict__ trace, const double* __restrict__ diag,
                                   const double* __restrict__ sigma, const DevPlan* __restrict__ dp,
                                   const double* __restrict__ jstats, const int* __restrict__ uctl, int64_t m,
                                   int k, int k_pad, double* __restrict__ pack) {
  const int t = threadIdx.x;
  if (t < 5) pack[t] = report[t];
  if (t < 8) pack[8 + t] = agg[t];
  if (t < 4) pack[16 + t] = energy[t];
  if (t == 0) { pack[20] = stats[m]; pack[21] = trace[0]; pack[24] = diag[0]; }
  if (t < 3) pack[25 + t] = diag[1 + t];  // uncentred lambda_1, residual, mu . v_1
  if (t < 2) pack[28 + t] = (double)uctl[t];  // blocks, steps of the uncentred power iteration
  if (t < 2) pack[22 + t] = energy[4 + k_pad + t];
  for (int r = t; r < k; r += blockDim.x) pack[kPackHead + r] = sigma[r];
  const unsigned long long* pw = reinterpret_cast<const unsigned long long*>(dp);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(pack + kPackHead + k);
  if (t < (int)(sizeof(DevPlan) / 8)) dst[t] = pw[t];
  if (t < 8) pack[kPackHead + k + kPlanWords + t] = jstats[t];  // 16 int sweep counts (run_eig)
}

}  // namespace
}  // namespace avd

using namespace avd;

struct avd_ctx : public Ctx {
  void* ws = nullptr;
  // device outputs for the host path
  double *o_mu = nullptr, *o_V = nullptr, *o_sigma = nullptr, *o_rho = nullptr;
  int64_t* o_idx = nullptr;
  double* report = nullptr;
};

extern "C" {

const char* avd_strerror(avd_status s) {
  switch (s) {
    case AVD_OK: return "ok";
    case AVD_EINVAL: return "invalid argument";
    case AVD_ENONFINITE: return "input contains NaN or Inf";
    case AVD_ENOCONV: return "eigensolver did not converge";
    case AVD_ECUDA: return "CUDA error";
    case AVD_ENOMEM: return "out of device memory";
    case AVD_ESTATE: return "stage called out of order";
    case AVD_EREPEAT: return "repeat avd_stage_gram: the Gram operand was raised to 3 digits";
    case AVD_EEXCHANGE: return "exchange callback failed";
  }
  return "unknown status";
}

const char* avd_last_error(void) { return avd::g_err.c_str(); }

avd_status avd_plan(const avd_config* cfg, avd_plan_t* plan) { return make_plan(cfg, plan, nullptr, nullptr); }

avd_status avd_create(const avd_config* cfg, avd_ctx** out) {
  if (!out) { set_error("null ctx pointer"); return AVD_EINVAL; }
  *out = nullptr;
  avd_ctx* c = new (std::nothrow) avd_ctx();
  if (!c) return AVD_ENOMEM;
  AVD_CUDA(cudaSetDevice(cfg ? cfg->device : 0));
  int dev = 0, sms = 148, major = 0, minor = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    set_error("libavd is built for sm_100a (B200); device is sm_" + std::to_string(major) + std::to_string(minor));
    delete c;
    return AVD_ECUDA;
  }
  c->num_sms = sms;
  Layout L;
  avd_status st = make_plan(cfg, &c->plan, c, &L);
  if (st != AVD_OK) { delete c; return st; }
  c->stream = (cudaStream_t)cfg->stream;
  if (cudaMalloc(&c->ws, L.total) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc of " + std::to_string(L.total) + " workspace bytes failed");
    delete c;
    return AVD_ENOMEM;
  }
  c->ws_bytes = L.total;
  char* b = (char*)c->ws;
  int i = 0;
#define BIND(field, T) c->field = reinterpret_cast<T>(b + L.off[i++])
  BIND(colsum_part, double*); BIND(colmax_part, float*); BIND(colmin_part, float*); BIND(sq_part, double*);
  BIND(stats, double*); BIND(colmax, float*); BIND(colmin, float*); BIND(hist1, unsigned long long*);
  BIND(mu, double*); BIND(shift, int32_t*); BIND(dplan, DevPlan*); BIND(digits, int8_t*);
  BIND(cand_key, uint32_t*); BIND(cand_idx, uint64_t*); BIND(cand_cnt, unsigned long long*);
  BIND(gram_i, long long*); BIND(G, double*); BIND(Q, double*); BIND(Y, double*); BIND(Z, double*); BIND(U, double*);
  BIND(H, double*); BIND(W, double*); BIND(theta, double*); BIND(red_part, double*); BIND(resid, double*);
  BIND(trace, double*); BIND(V, double*); BIND(sigma, double*); BIND(V32, float*); BIND(P, float*);
  BIND(en_part, double*); BIND(colsumP_part, double*); BIND(energy, double*); BIND(hist2, unsigned long long*);
  BIND(hist3, unsigned long long*); BIND(ties, long long*); BIND(bm_sel, uint32_t*); BIND(bm_tie, uint32_t*);
  BIND(blk_cnt, int64_t*); BIND(agg, double*); BIND(agg_part, double*); BIND(report, double*); BIND(hist0, unsigned long long*); BIND(cand_x, long long*); BIND(gemm_part, void*);
  BIND(Pd, int8_t*); BIND(Vt_hl, float*); BIND(Vd, int8_t*); BIND(mu_hl, float*);
  BIND(G32, float*); BIND(qsum, long long*); BIND(Q32, float*); BIND(Z32, float*); BIND(ticket, unsigned*); BIND(gmax, double*);
  BIND(samp, double*); BIND(smax, float*); BIND(smin, float*); BIND(qscale, float*); BIND(qoff, float*);
  BIND(qsum_part, long long*); BIND(qsum_local, long long*); BIND(qerr_part, float*); BIND(qerr_local, double*);
  BIND(qerr, double*); BIND(mu0, float*); BIND(qsq_part, long long*); BIND(diag, double*);
  BIND(prec, double*); BIND(ysq, double*); BIND(eig_ctl, void*); BIND(wsc, double*); BIND(gram_p, long long*);
  BIND(gd, int8_t*); BIND(gsc, double*); BIND(qd, int8_t*); BIND(qsc, double*); BIND(g8_part, double*);
  BIND(g8_tickets, unsigned*); BIND(tm_dev, CUtensorMap*); BIND(unc_topk, double*);
  BIND(ps, float*); BIND(vs, float*);
  if (c->cfg.world <= 1) c->gram_p = nullptr;
#undef BIND
  if (cudaMallocHost(&c->eig_host, sizeof(double) * kHostScratch) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(c->ws);
    delete c;
    set_error("cudaMallocHost failed");
    return AVD_ENOMEM;
  }
  if (cudaEventCreateWithFlags(&c->ev_host, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(c->ws);
    cudaFreeHost(c->eig_host);
    delete c;
    set_error("cudaEventCreate failed");
    return AVD_ECUDA;
  }
  cudaMemset(c->Pd, 0, (size_t)3 * c->l_pad * 128);  // K padding bytes of K8's operands stay zero
  cudaMemset(c->ps, 0, sizeof(float) * c->l_pad);
  cudaMemset(c->g8_tickets, 0, sizeof(unsigned) * (size_t)(c->m_pad / 128 + 1));
  st = gram_make_tmap(c);
  if (st != AVD_OK) { cudaFree(c->ws); cudaFreeHost(c->eig_host); cudaEventDestroy(c->ev_host); delete c; return st; }
  c->stage = 0;
  *out = c;
  return AVD_OK;
}

void avd_destroy(avd_ctx* c) {
  if (!c) return;
  destroy_graphs(c);
  cudaFree(c->ws);
  cudaFreeHost(c->eig_host);
  if (c->ev_host) cudaEventDestroy(c->ev_host);
  cudaFree(c->X_stage);
  cudaFree(c->o_mu); cudaFree(c->o_V); cudaFree(c->o_sigma); cudaFree(c->o_rho); cudaFree(c->o_idx);
  for (void* q : c->gf_allocs) cudaFree(q);
  delete c;
}

avd_status avd_get_plan(const avd_ctx* c, avd_plan_t* plan) {
  if (!c || !plan) return AVD_EINVAL;
  *plan = c->plan;
  return AVD_OK;
}

int64_t avd_launch_count(const avd_ctx* c) { return c ? c->launches : 0; }

avd_status avd_tie_quota(const int64_t* sel_counts, const int64_t* tie_counts, int32_t world, int32_t rank,
                         int64_t q, int64_t* quota, int64_t* offset) {
  if (!sel_counts || !tie_counts || !quota || !offset || world < 1 || rank < 0 || rank >= world || q < 0) {
    set_error("avd_tie_quota: bad arguments");
    return AVD_EINVAL;
  }
  int64_t rem = q, off = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t qr = std::min<int64_t>(std::max<int64_t>(rem, 0), tie_counts[r]);
    if (r == rank) { *quota = qr; *offset = off; return AVD_OK; }
    off += sel_counts[r] + qr;
    rem -= tie_counts[r];
  }
  return AVD_OK;
}

avd_status avd_buffer(avd_ctx* c, int32_t which, void** ptr, size_t* bytes) {
  if (!c || !ptr || !bytes) return AVD_EINVAL;
  const int64_t m = c->cfg.m;
  switch (which) {
    case AVD_BUF_STATS: *ptr = c->stats; *bytes = sizeof(double) * (m + 4); break;
    case AVD_BUF_SAMPLE: *ptr = c->samp; *bytes = sizeof(double) * (m + 1); break;
    case AVD_BUF_SMAX: *ptr = c->smax; *bytes = sizeof(float) * m; break;
    case AVD_BUF_SMIN: *ptr = c->smin; *bytes = sizeof(float) * m; break;
    case AVD_BUF_QSUM: *ptr = c->qsum; *bytes = sizeof(long long) * 2 * m; break;
    case AVD_BUF_QERR: *ptr = c->qerr; *bytes = sizeof(double) * m; break;
    case AVD_BUF_DIAG: *ptr = c->ysq; *bytes = sizeof(double) * m; break;
    case AVD_BUF_HIST0: *ptr = c->hist0; *bytes = sizeof(long long) * kHistBins; break;
    case AVD_BUF_CAND: *ptr = c->cand_x; *bytes = sizeof(long long) * 2; break;
    case AVD_BUF_COLMAX: *ptr = c->colmax; *bytes = sizeof(float) * m; break;
    case AVD_BUF_COLMIN: *ptr = c->colmin; *bytes = sizeof(float) * m; break;
    case AVD_BUF_HIST1: *ptr = c->hist1; *bytes = sizeof(long long) * kHistBins; break;
    case AVD_BUF_GRAM: *ptr = c->gram_i; *bytes = sizeof(long long) * c->m_pad * c->m_pad; break;
    case AVD_BUF_ENERGY: *ptr = c->energy; *bytes = sizeof(double) * (6 + c->k_pad); break;
    case AVD_BUF_HIST2: *ptr = c->hist2; *bytes = sizeof(long long) * kHistBins; break;
    case AVD_BUF_HIST3: *ptr = c->hist3; *bytes = sizeof(long long) * kHist3Bins; break;
    case AVD_BUF_TIES: *ptr = c->ties; *bytes = sizeof(long long) * 2 * c->cfg.world; break;
    case AVD_BUF_AGG: *ptr = c->agg; *bytes = sizeof(double) * 8; break;
    case AVD_BUF_MU: *ptr = c->mu; *bytes = sizeof(double) * m; break;
    case AVD_BUF_G: *ptr = c->G; *bytes = sizeof(double) * c->m_pad * c->m_pad; break;
    case AVD_BUF_P: *ptr = c->P; *bytes = sizeof(float) * c->cfg.l_local * c->k_pad; break;
    case AVD_BUF_DIGITS: *ptr = c->digits; *bytes = (size_t)c->nd_max * c->m_pad * c->l_pad; break;
    case AVD_BUF_SCALE: *ptr = c->shift; *bytes = sizeof(int32_t) * c->m_pad; break;
    case AVD_BUF_GRAMP: {
      if (!c->gram_p) { set_error("AVD_BUF_GRAMP exists with world > 1 only"); return AVD_EINVAL; }
      const int64_t T = c->m_pad / 128;
      *ptr = c->gram_p;
      *bytes = sizeof(long long) * (size_t)(T * (T + 1) / 2) * 128 * 128;
      break;
    }
    case AVD_BUF_EIGZ: *ptr = c->Z; *bytes = sizeof(double) * m * c->p; break;
    // diagnostic views of K8's digit operands (not exchanged)
    case 30: *ptr = c->Pd; *bytes = (size_t)3 * c->l_pad * 128; break;
    case 31: *ptr = c->ps; *bytes = sizeof(float) * c->l_pad; break;
    case 32: *ptr = c->Vd; *bytes = (size_t)3 * c->m_pad * 128; break;
    case 33: *ptr = c->vs; *bytes = sizeof(float) * c->m_pad; break;
    case AVD_BUF_EIGY: *ptr = c->Y; *bytes = sizeof(double) * m * c->p; break;
    default: set_error("unknown buffer id"); return AVD_EINVAL;
  }
  return AVD_OK;
}

#define STAGE_CHECK(c, want)                                                              \
  do {                                                                                    \
    if (!(c)) { set_error("null ctx"); return AVD_EINVAL; }                               \
    if ((c)->stage != (want)) {                                                           \
      set_error("stage order: expected stage " + std::to_string(want) + ", ctx is at " +  \
                std::to_string((c)->stage));                                              \
      return AVD_ESTATE;                                                                  \
    }                                                                                     \
  } while (0)

avd_status avd_stage_stats(avd_ctx* c, const float* X) {
  if (!c || !X) { set_error("null argument"); return AVD_EINVAL; }
  c->stage = 0;  // a new pass may start at any time
  c->nd = c->plan.digits;  // an automatic escalation lasts for one pass
  c->escalate = false;
  AVD_TRY(launch_sample(c, X));
  c->stage = 1;
  return AVD_OK;
}

avd_status avd_stage_split(avd_ctx* c, const float* X) {
  STAGE_CHECK(c, 1);
  if (!X) { set_error("null argument"); return AVD_EINVAL; }
  AVD_TRY(launch_pass1(c, X, true));
  c->stage = 2;
  return AVD_OK;
}

avd_status avd_stage_gram(avd_ctx* c, const float* X) {
  STAGE_CHECK(c, 2);
  if (!X) { set_error("null argument"); return AVD_EINVAL; }
  if (c->escalate) {
    // raised to 3 digits by avd_stage_eig: re-encode with the exact column ranges of the fused
    // pass (already exchanged) and redo the Gram; every other statistic stands
    c->escalate = false;
    AVD_TRY(launch_pass1(c, X, false));
    AVD_CUDA(cudaMemcpyAsync(c->qsum, c->qsum_local, sizeof(long long) * 2 * c->cfg.m, cudaMemcpyDeviceToDevice,
                             c->stream));
    AVD_CUDA(cudaMemcpyAsync(c->qerr, c->qerr_local, sizeof(double) * c->m_pad, cudaMemcpyDeviceToDevice, c->stream));
    if (!c->gram_free) AVD_TRY(launch_gram(c));
    if (c->gram_p) AVD_TRY(launch_gram_pack(c, false));  // world > 1: the exchanged form
    c->requantised = true;
    c->stage = 3;
    return AVD_OK;
  }
  AVD_TRY(launch_finish(c));
  double* hs = c->eig_host;  // pinned scratch
  AVD_CUDA(cudaMemcpyAsync(hs, c->stats + c->cfg.m + 3, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaMemcpyAsync(hs + 1, c->dplan, sizeof(DevPlan), cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaEventRecord(c->ev_host, c->stream));
  // speculative: the Gram of the digits as they stand is queued before the host reads the flags,
  // so the GPU does not idle through the round trip; a requant (or an error) redoes / drops it
  auto gram = [&]() -> avd_status {
    AVD_CUDA(cudaMemcpyAsync(c->qsum, c->qsum_local, sizeof(long long) * 2 * c->cfg.m, cudaMemcpyDeviceToDevice,
                             c->stream));
    AVD_CUDA(cudaMemcpyAsync(c->qerr, c->qerr_local, sizeof(double) * c->m_pad, cudaMemcpyDeviceToDevice, c->stream));
    return c->gram_free ? AVD_OK : launch_gram(c);  // Gram-free: no Gram
  };
  const bool force_exact = (c->cfg.flags & AVD_FLAG_EXACT_SCALE) != 0;
  if (!force_exact) {  // gated on the device: skipped when an entry overflowed the sampled range
    AVD_CUDA(cudaMemcpyAsync(c->qsum, c->qsum_local, sizeof(long long) * 2 * c->cfg.m, cudaMemcpyDeviceToDevice,
                             c->stream));
    AVD_CUDA(cudaMemcpyAsync(c->qerr, c->qerr_local, sizeof(double) * c->m_pad, cudaMemcpyDeviceToDevice, c->stream));
    if (!c->gram_free) AVD_TRY(launch_gram(c, c->stats + c->cfg.m + 3));
  }
  AVD_CUDA(cudaEventSynchronize(c->ev_host));
  const double ovf = hs[0];
  std::memcpy(&c->hplan, hs + 1, sizeof(DevPlan));
  if (c->hplan.nonfinite > 0) {
    set_error("X has non-finite entries (" + std::to_string(c->hplan.nonfinite) + " non-finite column sums)");
    c->stage = 0;
    return AVD_ENONFINITE;
  }
  c->requantised = ovf > 0.0 || force_exact;
  if (c->requantised) {
    // automatic digits: an exact-range requant that costs a column >= 3 bits of its planned
    // 14-bit resolution (a massive activation the row sample missed) goes to
    // 3 digits at once instead of through a 2-digit Gram and the a-posteriori escalation
    if (c->auto_digits && c->nd == 2 && c->hplan.range_bits >= 3) c->nd = 3;
    AVD_TRY(launch_pass1(c, X, false));  // exact column ranges (k_pass1.cu)
    AVD_TRY(gram());
  }
  if (c->gram_p) AVD_TRY(launch_gram_pack(c, false));  // world > 1: the exchanged form
  c->stage = 3;
  return AVD_OK;
}

static avd_status stage_eig_impl(avd_ctx* c, int32_t rank, avd_exchange_fn fn, void* user) {
  STAGE_CHECK(c, 3);
  avd_status st;
  if (c->gram_free) {  // no Gram; tr(G) and diag(G) from the fused pass's sums
    AVD_TRY(gf_prepare(c));
    AVD_TRY(gf_diag(c));
    AVD_TRY(launch_trace(c));
    st = run_eig(c);
  } else {
    if (c->gram_p) AVD_TRY(launch_gram_pack(c, true));  // the exchanged packed tiles back into G_int
    AVD_TRY(launch_gram_finalize(c));
    AVD_TRY(launch_uncentred(c));  // mean-bias diagnostics, side stream
    st = fn ? run_eig_dist(c, rank, fn, user) : run_eig(c);
    AVD_TRY(join_uncentred(c));    // (stream order only; G32 is not rewritten before the join)
  }
  if (st != AVD_OK && st != AVD_ENOCONV) return st;
  // automatic digits (avd_config.digits == 0): the quantisation-error bound decides whether the
  // 2-digit operand meets half the north-star tolerances; if not, redo the Gram with 3 digits.
  // The decision uses only replicated values (G, V_k, shifts), so every rank takes it alike.
  const bool force = (c->cfg.flags & AVD_FLAG_FORCE_ESCALATE) != 0;
  if (c->auto_digits && c->nd == 2 && (force || c->prec_sigma > 5e-5 || c->prec_share > 5e-6)) {
    c->nd = 3;
    c->escalate = true;
    c->stage = 2;
    set_error("Gram operand raised to 3 digits: call avd_stage_gram again");
    return AVD_EREPEAT;
  }
  if (c->cfg.flags & AVD_FLAG_MEAN_TOPK) AVD_TRY(run_uncentred_topk(c, c->unc_topk));
  c->stage = 4;
  return st;
}

avd_status avd_stage_eig(avd_ctx* c) { return stage_eig_impl(c, 0, nullptr, nullptr); }

avd_status avd_stage_eig_dist(avd_ctx* c, int32_t rank, avd_exchange_fn fn, void* user) {
  if (!c) { set_error("null ctx"); return AVD_EINVAL; }
  return stage_eig_impl(c, rank, c->cfg.world > 1 ? fn : nullptr, user);
}

avd_status avd_stage_project(avd_ctx* c, const float* X) {
  STAGE_CHECK(c, 4);
  AVD_TRY(launch_project(c, X));
  c->stage = 5;
  return AVD_OK;
}

avd_status avd_stage_select(avd_ctx* c, const float* X, int32_t level, int32_t rank) {
  STAGE_CHECK(c, 5 + level);
  if (level < 0 || level > 3 || rank < 0 || rank >= c->cfg.world) { set_error("bad level/rank"); return AVD_EINVAL; }
  if (level == 0) {
    // local count + globally exchanged [count, overflow] -> same decision on every rank
    long long* hs = reinterpret_cast<long long*>(c->eig_host);  // pinned scratch
    AVD_CUDA(cudaMemcpyAsync(hs, c->cand_cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaMemcpyAsync(hs + 1, c->cand_x, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    AVD_CUDA(cudaEventRecord(c->ev_host, c->stream));
    AVD_TRY(launch_select0_speculative(c));  // runs while the host reads the counts
    AVD_CUDA(cudaEventSynchronize(c->ev_host));
    const unsigned long long cnt = (unsigned long long)hs[0];
    const long long gx[2] = {hs[1], hs[2]};
    c->hplan.cand_count = (int64_t)cnt;
    // the candidate list is used only if it holds >= n_top entries (then |E_top| = n_top)
    c->cand_overflow = gx[1] > 0 || gx[0] < c->plan.n_top || (c->cfg.flags & AVD_FLAG_STREAM_SELECT);
  }
  if (level != 0 || c->cand_overflow) AVD_TRY(launch_select(c, X, level, rank));  // level 0 from X
  c->stage = 6 + level;
  return AVD_OK;
}

avd_status avd_stage_gather(avd_ctx* c, const float* X, int32_t rank, avd_outputs* out) {
  STAGE_CHECK(c, 9);
  if (!out || !out->top_idx_dev || !out->rho_dev) { set_error("null output arrays"); return AVD_EINVAL; }
  AVD_TRY(launch_gather(c, X, rank, out->top_idx_dev, out->rho_dev));
  c->stage = 10;
  return AVD_OK;
}

avd_status avd_gram_product(avd_ctx* c, const double* In, double* Y) {
  if (!c || !In || !Y) { set_error("null argument"); return AVD_EINVAL; }
  if (c->stage < 4) { set_error("avd_gram_product needs a completed eigen stage (or avd_decompose)"); return AVD_ESTATE; }
  AVD_TRY(gram_product(c, In, Y));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  return AVD_OK;
}

avd_status avd_stage_report(avd_ctx* c, avd_outputs* out) {
  STAGE_CHECK(c, 10);
  if (!out) { set_error("null outputs"); return AVD_EINVAL; }
  const int64_t m = c->cfg.m;
  const int k = c->k;
  const int nrep = (int)ceil_div(m, 256);
  report_part_kernel<<<nrep, 256, 0, c->stream>>>(c->energy, c->stats, c->mu, c->V, m, k, c->cfg.l_global,
                                                  c->red_part);  // eig scratch is free here
  AVD_LAUNCHED(c);
  report_final_kernel<<<1, 32, 0, c->stream>>>(c->red_part, nrep, c->cfg.l_global, c->report);
  AVD_LAUNCHED(c);
  if (c->cfg.flags & AVD_FLAG_MEAN_TOPK) {  // uncentred sigma_i, alpha_i (i < k)
    if (out->mean_sigma_dev)
      AVD_CUDA(cudaMemcpyAsync(out->mean_sigma_dev, c->unc_topk, sizeof(double) * k, cudaMemcpyDeviceToDevice, c->stream));
    if (out->mean_alpha_dev)
      AVD_CUDA(cudaMemcpyAsync(out->mean_alpha_dev, c->unc_topk + k, sizeof(double) * k, cudaMemcpyDeviceToDevice,
                               c->stream));
  }
  if (out->mu_dev || out->V_dev || out->sigma_dev) {
    copy_outputs_kernel<<<(unsigned)ceil_div(std::max<int64_t>(m * k, m), 256), 256, 0, c->stream>>>(
        c->mu, c->V, c->sigma, m, k, out->mu_dev, out->V_dev, out->sigma_dev);
    AVD_LAUNCHED(c);
  }
  // one packed D2H copy (pageable copies cost ~10 us each); the tail of the eig scratch is free
  const int64_t npack = kPackHead + k + kPlanWords + 8;
  double* pack = c->red_part + ((int64_t)c->n_red * c->p * c->p - npack);
  report_pack_kernel<<<1, 128, 0, c->stream>>>(c->report, c->agg, c->energy, c->stats, c->trace, c->diag, c->sigma,
                                               c->dplan, c->theta + c->p,
                                               reinterpret_cast<const int*>(c->eig_ctl) + kCtlBlocksU, m, k,
                                               c->k_pad, pack);
  AVD_LAUNCHED(c);
  static_assert(kPackHead + 96 + kPlanWords + 8 <= 4 * kMaxP, "pinned scratch too small for the report pack");
  const double* h = c->eig_host;  // pinned scratch (k <= 95)
  AVD_CUDA(cudaMemcpyAsync(c->eig_host, pack, sizeof(double) * npack, cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  std::memcpy(&c->hplan, h + kPackHead + k, sizeof(DevPlan));
  {
    int sw[16];
    std::memcpy(sw, h + kPackHead + k + kPlanWords, sizeof(sw));
    c->jacobi_sweeps = 0;
    for (int q = 0; q < std::min(c->rr_count, 16); ++q) c->jacobi_sweeps += sw[q];  // over all RR solves
  }
  const double* sig = h + kPackHead;
  double spike = 0.0;
  for (int r = 0; r < k; ++r) spike += sig[r] * sig[r];
  const double total = h[20], trace = h[21];
  out->energy_cf[0] = total;
  out->energy_cf[1] = h[4];
  out->energy_cf[2] = spike;
  out->energy_cf[3] = trace - spike;
  out->energy_el[0] = total;
  out->energy_el[1] = h[4];
  out->energy_el[2] = h[16];
  out->energy_el[3] = h[17];
  out->cross_el[0] = h[0];
  out->cross_el[1] = h[1];
  out->cross_el[2] = h[18];
  out->colmean_absmax[0] = h[2];
  out->colmean_absmax[1] = h[3];
  const double nt = (double)c->hplan.n_eff;
  for (int q = 0; q < 4; ++q) out->rho_mean_aggr[q] = nt > 0 ? h[8 + q] / nt : 0.0;
  for (int q = 0; q < 3; ++q) out->rho_energy_aggr[q] = h[15] > 0 ? h[12 + q] / h[15] : 0.0;
  out->sigma_next = c->sigma_next;
  out->trace_g = trace;
  out->iters = c->iters;
  out->max_resid = c->max_resid;
  out->rr_checks = c->rr_count;
  out->jacobi_sweeps = c->jacobi_sweeps;
  out->requantised = c->requantised ? 1 : 0;
  out->digits_used = c->nd;
  out->precision_sigma = c->prec_sigma;
  out->precision_share = c->prec_share;
  // mean-bias diagnostics
  const double lg = (double)c->cfg.l_global;
  out->mean_R = (total > 0.0) ? h[24] / std::sqrt(total / lg) : 0.0;
  out->p_pos = (int64_t)h[22];
  out->p_neg = (int64_t)h[23];
  out->sign_fraction = c->sign_valid ? (double)std::max(out->p_pos, out->p_neg) / lg : -1.0;
  {  // uncentred top pair (k_eig.cu launch_uncentred): diag[0] = ||mu||, lambda_1, residual, mu . v_1
    const double nmu = h[24];
    c->sigma1_u = std::sqrt(std::max(h[25], 0.0));
    c->alpha1 = std::fabs(h[27]);
    c->cos_mu_v1 = nmu > 0.0 ? std::min(1.0, std::fabs(h[27]) / nmu) : 0.0;
    c->resid_u = h[26];
    c->iters_u = (int)h[29];
    if (!c->gram_free) c->launches += (int64_t)c->n_u_nodes * (int64_t)h[28];
    if (c->gram_free) {  // the uncentred pair needs G (not formed)
      c->sigma1_u = c->alpha1 = c->cos_mu_v1 = c->resid_u = std::nan("");
      c->iters_u = 0;
    }
  }
  out->cos_mu_v1 = c->cos_mu_v1;
  out->alpha1 = c->alpha1;
  out->sigma1_u = c->sigma1_u;
  out->resid_u = c->resid_u;
  out->iters_u = c->iters_u;
  out->iters_uk = (c->cfg.flags & AVD_FLAG_MEAN_TOPK) ? c->iters_uk : 0;
  out->resid_uk = (c->cfg.flags & AVD_FLAG_MEAN_TOPK) ? c->resid_uk : 0.0;
  out->n_top_local = c->hplan.sel_local;
  out->top_offset = c->hplan.top_offset;
  out->n_top_global = c->hplan.n_eff;
  c->stage = 11;
  return AVD_OK;
}

avd_status avd_decompose(avd_ctx* c, const float* X, avd_outputs* out) {
  if (!c || !X || !out) { set_error("null argument"); return AVD_EINVAL; }
  if (c->cfg.world != 1) { set_error("avd_decompose needs world == 1 (use the stage API)"); return AVD_EINVAL; }
  if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) { set_error("X must be 16-byte aligned"); return AVD_EINVAL; }
  AVD_TRY(avd_stage_stats(c, X));
  AVD_TRY(avd_stage_split(c, X));
  AVD_TRY(avd_stage_gram(c, X));
  avd_status eig = avd_stage_eig(c);
  if (eig == AVD_EREPEAT) {  // automatic digits: 3-digit Gram
    AVD_TRY(avd_stage_gram(c, X));
    eig = avd_stage_eig(c);
  }
  if (eig != AVD_OK && eig != AVD_ENOCONV) return eig;
  AVD_TRY(avd_stage_project(c, X));
  for (int lv = 0; lv < 4; ++lv) AVD_TRY(avd_stage_select(c, X, lv, 0));
  AVD_TRY(avd_stage_gather(c, X, 0, out));
  AVD_TRY(avd_stage_report(c, out));
  return eig;
}

// The exchange table of the stage API (include/avd.h), in call order
namespace {
struct Exch { int32_t which, dtype, op; };
avd_status run_exchanges(avd_ctx* c, const Exch* tab, int n, avd_exchange_fn fn, void* user) {
  for (int i = 0; i < n; ++i) {
    void* ptr = nullptr;
    size_t bytes = 0;
    AVD_TRY(avd_buffer(c, tab[i].which, &ptr, &bytes));
    const size_t es = tab[i].dtype == AVD_DT_F32 ? 4 : 8;
    if (fn(tab[i].which, ptr, tab[i].dtype, tab[i].op, bytes / es, user) != 0) {
      set_error("exchange callback failed (buffer " + std::to_string(tab[i].which) + ")");
      return AVD_EEXCHANGE;
    }
  }
  return AVD_OK;
}
}  // namespace

avd_status avd_decompose_sharded(avd_ctx* c, const float* X, int32_t rank, avd_outputs* out, avd_exchange_fn fn,
                                 void* user) {
  if (!c || !X || !out) { set_error("null argument"); return AVD_EINVAL; }
  if (c->cfg.world == 1 && !fn) return avd_decompose(c, X, out);
  if (!fn) { set_error("world > 1 needs an exchange callback"); return AVD_EINVAL; }
  const bool w = c->cfg.world > 1;
  static const Exch kStats[] = {{AVD_BUF_SAMPLE, AVD_DT_F64, AVD_OP_SUM}, {AVD_BUF_SMAX, AVD_DT_F32, AVD_OP_MAX},
                                {AVD_BUF_SMIN, AVD_DT_F32, AVD_OP_MIN}, {AVD_BUF_HIST1, AVD_DT_I64, AVD_OP_SUM}};
  static const Exch kSplit[] = {{AVD_BUF_STATS, AVD_DT_F64, AVD_OP_SUM}, {AVD_BUF_COLMAX, AVD_DT_F32, AVD_OP_MAX},
                                {AVD_BUF_DIAG, AVD_DT_F64, AVD_OP_SUM}};
  static const Exch kGram[] = {{AVD_BUF_GRAMP, AVD_DT_I64, AVD_OP_SUM}, {AVD_BUF_CAND, AVD_DT_I64, AVD_OP_SUM},
                               {AVD_BUF_QSUM, AVD_DT_I64, AVD_OP_SUM}, {AVD_BUF_QERR, AVD_DT_F64, AVD_OP_SUM}};
  static const Exch kRegram[] = {{AVD_BUF_GRAMP, AVD_DT_I64, AVD_OP_SUM}, {AVD_BUF_QSUM, AVD_DT_I64, AVD_OP_SUM},
                                 {AVD_BUF_QERR, AVD_DT_F64, AVD_OP_SUM}};
  static const Exch kProj[] = {{AVD_BUF_ENERGY, AVD_DT_F64, AVD_OP_SUM}};
  static const Exch kSel[4] = {{AVD_BUF_HIST0, AVD_DT_I64, AVD_OP_SUM}, {AVD_BUF_HIST2, AVD_DT_I64, AVD_OP_SUM},
                               {AVD_BUF_HIST3, AVD_DT_I64, AVD_OP_SUM}, {AVD_BUF_TIES, AVD_DT_I64, AVD_OP_SUM}};
  static const Exch kAgg[] = {{AVD_BUF_AGG, AVD_DT_F64, AVD_OP_SUM}};
  AVD_TRY(avd_stage_stats(c, X));
  AVD_TRY(run_exchanges(c, kStats, 4, fn, user));
  AVD_TRY(avd_stage_split(c, X));
  AVD_TRY(run_exchanges(c, kSplit, 3, fn, user));
  AVD_TRY(avd_stage_gram(c, X));
  if (w) AVD_TRY(run_exchanges(c, kGram, 4, fn, user));
  else AVD_TRY(run_exchanges(c, kGram + 1, 3, fn, user));
  avd_status eig = avd_stage_eig_dist(c, rank, fn, user);
  if (eig == AVD_EREPEAT) {
    AVD_TRY(avd_stage_gram(c, X));
    if (w) AVD_TRY(run_exchanges(c, kRegram, 3, fn, user));
    else AVD_TRY(run_exchanges(c, kRegram + 1, 2, fn, user));
    eig = avd_stage_eig_dist(c, rank, fn, user);
  }
  if (eig != AVD_OK && eig != AVD_ENOCONV) return eig;
  AVD_TRY(avd_stage_project(c, X));
  AVD_TRY(run_exchanges(c, kProj, 1, fn, user));
  for (int lv = 0; lv < 4; ++lv) {
    AVD_TRY(avd_stage_select(c, X, lv, rank));
    AVD_TRY(run_exchanges(c, kSel + lv, 1, fn, user));
  }
  AVD_TRY(avd_stage_gather(c, X, rank, out));
  AVD_TRY(run_exchanges(c, kAgg, 1, fn, user));
  AVD_TRY(avd_stage_report(c, out));
  return eig;
}

// ---- NCCL exchange (libnccl.so.2 loaded at first use; types from nccl.h)
typedef ncclResult_t (*nccl_allreduce_t)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                         cudaStream_t);
int avd_exchange_nccl(int32_t which, void* buf, int32_t dtype, int32_t op, size_t count, void* user) {
  (void)which;
  static nccl_allreduce_t fn = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce")) : nullptr;
  }();
  const avd_nccl_comm* nc = static_cast<const avd_nccl_comm*>(user);
  if (!fn || !nc || !nc->comm) return 1;
  const ncclDataType_t t = dtype == AVD_DT_F64 ? ncclFloat64 : (dtype == AVD_DT_F32 ? ncclFloat32 : ncclInt64);
  const ncclRedOp_t o = op == AVD_OP_MAX ? ncclMax : (op == AVD_OP_MIN ? ncclMin : ncclSum);
  return fn(buf, buf, count, t, o, static_cast<ncclComm_t>(nc->comm), static_cast<cudaStream_t>(nc->stream)) ==
                 ncclSuccess
             ? 0
             : 1;
}

avd_status avd_decompose_host(avd_ctx* c, const float* X_host, avd_outputs* out) {
  if (!c || !X_host || !out) { set_error("null argument"); return AVD_EINVAL; }
  const int64_t l = c->cfg.l_local, m = c->cfg.m, k = c->k, n = c->plan.n_top;
  if (!c->X_stage) {
    AVD_CUDA(cudaMalloc(&c->X_stage, sizeof(float) * l * m));
    AVD_CUDA(cudaMalloc(&c->o_mu, sizeof(double) * m));
    AVD_CUDA(cudaMalloc(&c->o_V, sizeof(double) * m * k));
    AVD_CUDA(cudaMalloc(&c->o_sigma, sizeof(double) * k));
    AVD_CUDA(cudaMalloc(&c->o_idx, sizeof(int64_t) * n));
    AVD_CUDA(cudaMalloc(&c->o_rho, sizeof(double) * 4 * n));
  }
  AVD_CUDA(cudaMemcpyAsync(c->X_stage, X_host, sizeof(float) * l * m, cudaMemcpyHostToDevice, c->stream));
  avd_outputs d = *out;
  d.mu_dev = c->o_mu; d.V_dev = c->o_V; d.sigma_dev = c->o_sigma; d.top_idx_dev = c->o_idx; d.rho_dev = c->o_rho;
  d.mean_sigma_dev = nullptr; d.mean_alpha_dev = nullptr;  // host arrays here: copied below
  const avd_status st = avd_decompose(c, c->X_stage, &d);
  if (st != AVD_OK && st != AVD_ENOCONV) return st;
  if (out->mu_dev) AVD_CUDA(cudaMemcpyAsync(out->mu_dev, c->o_mu, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
  if (out->V_dev) AVD_CUDA(cudaMemcpyAsync(out->V_dev, c->o_V, sizeof(double) * m * k, cudaMemcpyDeviceToHost, c->stream));
  if (out->sigma_dev) AVD_CUDA(cudaMemcpyAsync(out->sigma_dev, c->o_sigma, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
  if (out->top_idx_dev) AVD_CUDA(cudaMemcpyAsync(out->top_idx_dev, c->o_idx, sizeof(int64_t) * d.n_top_local, cudaMemcpyDeviceToHost, c->stream));
  if (out->rho_dev) AVD_CUDA(cudaMemcpyAsync(out->rho_dev, c->o_rho, sizeof(double) * 4 * d.n_top_local, cudaMemcpyDeviceToHost, c->stream));
  if ((c->cfg.flags & AVD_FLAG_MEAN_TOPK) && out->mean_sigma_dev)
    AVD_CUDA(cudaMemcpyAsync(out->mean_sigma_dev, c->unc_topk, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
  if ((c->cfg.flags & AVD_FLAG_MEAN_TOPK) && out->mean_alpha_dev)
    AVD_CUDA(cudaMemcpyAsync(out->mean_alpha_dev, c->unc_topk + k, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
  AVD_CUDA(cudaStreamSynchronize(c->stream));
  double* keep[6] = {out->mu_dev, out->V_dev, out->sigma_dev, out->rho_dev, out->mean_sigma_dev, out->mean_alpha_dev};
  int64_t* keep_idx = out->top_idx_dev;
  *out = d;
  out->mu_dev = keep[0]; out->V_dev = keep[1]; out->sigma_dev = keep[2]; out->rho_dev = keep[3];
  out->mean_sigma_dev = keep[4]; out->mean_alpha_dev = keep[5];
  out->top_idx_dev = keep_idx;
  return st;
}

}  // extern "C"
