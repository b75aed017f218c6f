// umma_probe.cu — hardware probe for tcgen05.mma kind::tf32 on sm_100a (not product code):
//  (1) validates the K-major and MN-major SWIZZLE_128B smem descriptors against a host GEMM,
//  (2) measures how the tensor core converts fp32 operands to tf32 (round vs truncate),
//  (3) measures the fp32 accumulator rounding (RN vs RZ) in TMEM across and within MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I.. tools/umma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "../paper_2603_10444_b200/csrc/sm100.cuh"
using namespace avd::sm100;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}
static CUtensorMap make_map(const float* g, uint64_t inner, uint64_t outer, uint32_t box_in, uint32_t box_out) {
  CUtensorMap m; uint64_t dims[2] = {inner, outer}; uint64_t strides[1] = {inner * 4};
  uint32_t box[2] = {box_in, box_out}; uint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

template <bool AMN, bool BMN>
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap ta,
    const __grid_constant__ CUtensorMap tb, int K, float* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sA = (float*)smem;            // 16 KB
  float* sB = (float*)(smem + 16384);  // 16 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) { mbar_init(&bar_tma, 1); mbar_init(&bar_mma, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<128>(&tmem_base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_tf32(128, 128, AMN, BMN);
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    for (int k0 = 0; k0 < K; k0 += 32) {
      mbar_arrive_expect_tx(&bar_tma, 32768);
      if (AMN) { for (int nb = 0; nb < 4; ++nb) tma_load_2d(sA + nb * 1024, &ta, &bar_tma, nb * 32, k0); }
      else tma_load_2d(sA, &ta, &bar_tma, k0, 0);
      if (BMN) { for (int nb = 0; nb < 4; ++nb) tma_load_2d(sB + nb * 1024, &tb, &bar_tma, nb * 32, k0); }
      else tma_load_2d(sB, &tb, &bar_tma, k0, 0);
      mbar_wait(&bar_tma, ph);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = AMN ? smem_desc(smem_u32(sA) + kk * 1024, 4096, 1024, 2)
                          : smem_desc(smem_u32(sA) + kk * 32, 16, 1024, 2);
        uint64_t bd = BMN ? smem_desc(smem_u32(sB) + kk * 1024, 4096, 1024, 2)
                          : smem_desc(smem_u32(sB) + kk * 32, 16, 1024, 2);
        mma_tf32(tmem, ad, bd, idesc, (k0 > 0 || kk > 0) ? 1u : 0u);
      }
      mma_commit(&bar_mma);
      mbar_wait(&bar_mma, ph);
      ph ^= 1;
    }
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t row = warp * 32 + lane_id();
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int t = 0; t < 16; ++t) D[row * 128 + c0 + t] = __uint_as_float(r[t]);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

// A logical [128][K], B logical [128][K]; D = A B^T
static std::vector<float> run(bool amn, bool bmn, int K, const std::vector<float>& A, const std::vector<float>& B) {
  std::vector<float> As(128 * K), Bs(128 * K);
  for (int i = 0; i < 128; ++i) for (int k = 0; k < K; ++k) {
    As[amn ? k * 128 + i : i * K + k] = A[i * K + k];
    Bs[bmn ? k * 128 + i : i * K + k] = B[i * K + k];
  }
  float *dA, *dB, *dD; CK(cudaMalloc(&dA, As.size() * 4)); CK(cudaMalloc(&dB, Bs.size() * 4)); CK(cudaMalloc(&dD, 128 * 128 * 4));
  CK(cudaMemcpy(dA, As.data(), As.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bs.data(), Bs.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap ta = amn ? make_map(dA, 128, K, 32, 32) : make_map(dA, K, 128, 32, 128);
  CUtensorMap tb = bmn ? make_map(dB, 128, K, 32, 32) : make_map(dB, K, 128, 32, 128);
  size_t sm = 32768 + 1024;
  auto launch = [&](auto kern) { CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); kern<<<1, 128, sm>>>(ta, tb, K, dD); };
  if (amn && bmn) launch(probe<true, true>); else if (amn) launch(probe<true, false>);
  else if (bmn) launch(probe<false, true>); else launch(probe<false, false>);
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  std::vector<float> D(128 * 128); CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return D;
}
static float tf32_rn(float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & ~0x1FFFu; float y; memcpy(&y, &u, 4); return y; }
static float tf32_rz(float x) { uint32_t u; memcpy(&u, &x, 4); u &= ~0x1FFFu; float y; memcpy(&y, &u, 4); return y; }

int main() {
  srand(1);
  // (1) descriptor validation with tf32-exact random data (so conversion mode does not matter)
  const int K = 256;
  std::vector<float> A(128 * K), B(128 * K);
  for (auto& v : A) v = tf32_rz((rand() / (float)RAND_MAX - 0.5f) * 4);
  for (auto& v : B) v = tf32_rz((rand() / (float)RAND_MAX - 0.5f) * 4);
  for (int amn = 0; amn < 2; ++amn) for (int bmn = 0; bmn < 2; ++bmn) {
    auto D = run(amn, bmn, K, A, B);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
      double s = 0; for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * 128 + j])); maxref = fmax(maxref, fabs(s));
    }
    printf("layout A=%s B=%s : max|err|=%.3e (max|ref|=%.3e) %s\n", amn ? "MN" : "K", bmn ? "MN" : "K", maxerr, maxref, maxerr < 1e-3 * maxref ? "OK" : "FAIL");
  }
  // (2) operand conversion: random fp32 (not tf32-exact)
  {
    for (auto& v : A) v = (rand() / (float)RAND_MAX - 0.5f) * 4;
    for (auto& v : B) v = (rand() / (float)RAND_MAX - 0.5f) * 4;
    auto D = run(false, false, K, A, B);
    double e_rn = 0, e_rz = 0, e_ex = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
      double srn = 0, srz = 0, sex = 0;
      for (int k = 0; k < K; ++k) { srn += (double)tf32_rn(A[i*K+k]) * tf32_rn(B[j*K+k]); srz += (double)tf32_rz(A[i*K+k]) * tf32_rz(B[j*K+k]); sex += (double)A[i*K+k]*B[j*K+k]; }
      double d = D[i * 128 + j]; e_rn += fabs(d - srn); e_rz += fabs(d - srz); e_ex += fabs(d - sex);
    }
    printf("operand conversion: mean|D-ref| with RN-tf32 %.3e, RZ-tf32 %.3e, fp32-exact %.3e\n", e_rn / 16384, e_rz / 16384, e_ex / 16384);
  }
  // (3) accumulator rounding probes, K = 32 (padded), B[:,0] = 1 for all k
  {
    const int K2 = 32;
    std::vector<float> A2(128 * K2, 0.f), B2(128 * K2, 0.f);
    for (int k = 0; k < K2; ++k) B2[0 * K2 + k] = 1.f;
    auto a = [&](int r, int k, float v) { A2[r * K2 + k] = v; };
    // row0: MMA#1 gives 1, MMA#2 adds +0.75 ulp(1)=0.75*2^-23
    a(0, 0, 1.f); a(0, 8, 0.75f * ldexpf(1, -23));
    // row1: within one MMA: 1 + 7 * 2^-25 (= 1 + 1.75 * 2^-23)
    a(1, 0, 1.f); for (int k = 1; k < 8; ++k) a(1, k, ldexpf(1, -25));
    // row2: operand 1 + 2^-11 + 2^-13 (0.625 tf32-ulp above 1)
    a(2, 0, 1.f + ldexpf(1, -11) + ldexpf(1, -13));
    // row3: MMA#1 gives 1, MMA#2 adds -0.75*2^-23
    a(3, 0, 1.f); a(3, 8, -0.75f * ldexpf(1, -23));
    // row4: MMA#1 gives 1, MMA#2 adds +0.5 ulp (tie)
    a(4, 0, 1.f); a(4, 8, 0.5f * ldexpf(1, -23));
    // row5: MMA#1 gives 1, MMA#2 adds +1.5 ulp (tie above odd)
    a(5, 0, 1.f); a(5, 8, 1.5f * ldexpf(1, -23));
    // row6: in one MMA: 1 + 0.75ulp
    a(6, 0, 1.f); a(6, 1, 0.75f * ldexpf(1, -23));
    // row7: in one MMA: 2^24 + 1 + 1 (exact int arithmetic needs 25 bits)
    a(7, 0, ldexpf(1, 24)); a(7, 1, 1.f); a(7, 2, 1.f);
    auto D = run(false, false, K2, A2, B2);
    const char* nm[8] = {"1 +0.75u across MMAs", "1 +1.75u inside MMA", "operand 1+0.625tf32ulp", "1 -0.75u across MMAs",
                         "1 +0.5u across (tie)", "1 +1.5u across (tie)", "1 +0.75u inside MMA", "2^24+1+1 inside MMA"};
    for (int r = 0; r < 8; ++r) { double d = D[r * 128]; printf("probe %-26s -> %.10g  (d-1)/2^-23 = %.4f\n", nm[r], d, r == 7 ? d - ldexp(1, 24) : (d - 1.0) / ldexp(1, -23)); }
  }
  // (4) long accumulation drift, K = 8192, positive tf32-exact values
  {
    const int K3 = 8192;
    std::vector<float> A3(128 * K3), B3(128 * K3);
    for (int i = 0; i < 128; ++i) for (int k = 0; k < K3; ++k) { A3[i*K3+k] = 1.f + ldexpf((float)((k * 7 + i) % 1024), -10); B3[i*K3+k] = 1.f + ldexpf((float)((k * 3 + 5 * i) % 1024), -10); }
    auto D = run(false, false, K3, A3, B3);
    double mrel = 0, maxrel = 0; double sim_rn = 0, sim_rz = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < 128; ++j) {
      double s = 0; for (int k = 0; k < K3; ++k) s += (double)A3[i*K3+k] * B3[j*K3+k];
      double rel = (D[i * 128 + j] - s) / s; mrel += rel; maxrel = fmax(maxrel, fabs(rel));
    }
    // host emulation for row0/col0: fp32 RN sequential per MMA (exact 8-sum then add)
    { float acc_rn = 0, acc_rz = 0; double ex = 0;
      for (int k0 = 0; k0 < K3; k0 += 8) { double blk = 0; for (int k = k0; k < k0 + 8; ++k) blk += (double)A3[k] * B3[k]; ex += blk;
        acc_rn = (float)((double)acc_rn + blk);
        double t = (double)acc_rz + blk; float f = (float)t; if (fabs((double)f) > fabs(t)) f = nextafterf(f, 0.f); acc_rz = f; }
      sim_rn = (acc_rn - ex) / ex; sim_rz = (acc_rz - ex) / ex; }
    printf("drift K=8192: mean rel err %.3e, max |rel| %.3e ; host sim row0: RN-per-MMA %.3e RZ-per-MMA %.3e ; HW row0 %.3e\n",
           mrel / 16384, maxrel, sim_rn, sim_rz, 0.0);
    double s0 = 0; for (int k = 0; k < K3; ++k) s0 += (double)A3[k] * B3[k];
    printf("HW row0col0 rel err %.3e\n", (D[0] - s0) / s0);
  }
  printf("done\n");
  return 0;
}
