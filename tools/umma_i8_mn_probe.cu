// umma_i8_mn_probe.cu — hardware probe (not product code): does tcgen05.mma kind::i8 accept
// MN-major SWIZZLE_128B operands loaded by TMA straight from a row-major [K][M] int8 array,
// and which (LBO, SBO) encoding does it want?  D[M=128][N=128] = sum_k A[k][m] B[k][n].
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/umma_i8_mn_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2603_10444_b200/csrc/sm100.cuh"
using namespace avd::sm100;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}
// row-major [rows][cols] int8, box = 128 cols (inner) x 128 rows
static CUtensorMap make_map(const int8_t* g, uint64_t cols, uint64_t rows) {
  CUtensorMap m; uint64_t dims[2] = {cols, rows}; uint64_t strides[1] = {cols};
  uint32_t box[2] = {128, 128}; uint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

// A, B: [K][128] int8 row-major (the MN index contiguous); grid 1, 128 threads
__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap ta,
    const __grid_constant__ CUtensorMap tb, int K, int a_mn, int b_mn, uint32_t lbo, uint32_t sbo, int* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;            // 16 KB: 128 K-rows x 128 B
  uint8_t* sB = smem + 16384;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) { mbar_init(&bar_tma, 1); mbar_init(&bar_mma, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<128>(&tmem_base);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                         ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    uint32_t ph = 0;
    for (int k0 = 0; k0 < K; k0 += 128) {
      mbar_arrive_expect_tx(&bar_tma, 32768);
      tma_load_2d(sA, &ta, &bar_tma, 0, k0);
      tma_load_2d(sB, &tb, &bar_tma, 0, k0);
      mbar_wait(&bar_tma, ph);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = smem_desc(smem_u32(sA) + kk * 4096, lbo, sbo, 2);
        const uint64_t bd = smem_desc(smem_u32(sB) + kk * 4096, lbo, sbo, 2);
        mma_i8(tmem, ad, bd, idesc, (k0 > 0 || kk > 0) ? 1u : 0u);
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
    for (int t = 0; t < 16; ++t) D[row * 128 + c0 + t] = (int)r[t];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem);
}

int main() {
  const int K = 512;
  std::vector<int8_t> hA(K * 128), hB(K * 128);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int8_t)((s >> 24) - 128); };
  for (auto& v : hA) v = rnd();
  for (auto& v : hB) v = rnd();
  std::vector<long long> ref(128 * 128, 0);
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) ref[m * 128 + n] += (long long)hA[k * 128 + m] * hB[k * 128 + n];
  int8_t *dA, *dB; int* dD;
  CK(cudaMalloc(&dA, K * 128)); CK(cudaMalloc(&dB, K * 128)); CK(cudaMalloc(&dD, 128 * 128 * 4));
  CK(cudaMemcpy(dA, hA.data(), K * 128, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), K * 128, cudaMemcpyHostToDevice));
  CUtensorMap ta = make_map(dA, 128, K), tb = make_map(dB, 128, K);
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024));
  const uint32_t cand[][2] = {{16384, 1024}, {1024, 16384}, {0, 1024}, {1024, 0}, {128, 1024}, {1024, 128},
                              {8192, 1024}, {4096, 1024}};
  for (auto& c : cand) {
    CK(cudaMemset(dD, 0, 128 * 128 * 4));
    probe<<<1, 128, 33 * 1024>>>(ta, tb, K, 1, 1, c[0], c[1], dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("lbo=%u sbo=%u: CUDA error %s\n", c[0], c[1], cudaGetErrorString(e)); return 1; }
    std::vector<int> hD(128 * 128);
    CK(cudaMemcpy(hD.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost));
    long long bad = 0, maxerr = 0;
    for (int i = 0; i < 128 * 128; ++i) {
      long long d = (long long)hD[i] - ref[i];
      if (d) ++bad;
      if (llabs(d) > maxerr) maxerr = llabs(d);
    }
    printf("int8 A=MN B=MN lbo=%5u sbo=%5u : %s (mismatches %lld, max|err| %lld)\n", c[0], c[1],
           bad ? "FAIL" : "EXACT", bad, maxerr);
  }
  return 0;
}
