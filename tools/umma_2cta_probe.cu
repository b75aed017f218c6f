// umma_2cta_probe.cu — hardware probe (not product code): a CTA pair (cluster of 2) runs
// tcgen05.mma.cta_group::2.kind::i8 with M = 256 (128 A-rows per CTA) and N = 128 (64 B-rows
// per CTA), MN-major operands loaded by TMA straight from row-major [K][M] / [K][N] int8 arrays
// (A: SWIZZLE_128B box 128 x 128, B: SWIZZLE_64B box 64 x 128).  Checks D = A^T B exactly.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/umma_2cta_probe.cu -o tools/umma_2cta_probe -lcuda
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
static CUtensorMap make_map(const int8_t* g, uint64_t cols, uint64_t rows, uint32_t box_cols, CUtensorMapSwizzle sw) {
  CUtensorMap m; uint64_t dims[2] = {cols, rows}; uint64_t strides[1] = {cols};
  uint32_t box[2] = {box_cols, 128}; uint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
  return m;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank)); return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's smem, completion bytes counted on the mbarrier at cluster address `bar`
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t bar, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar),
               "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_2sm(uint64_t* bar) {  // arrive on `bar` (same offset) in both CTAs
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int K, int lbo_b, int* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;            // 16 KB: 128 K-rows x 128 B
  uint8_t* sB = smem + 16384;    // 8 KB: 128 K-rows x 64 B
  __shared__ __align__(8) uint64_t bar_full, bar_done;
  __shared__ uint32_t tmem_base;
  const uint32_t rank = cluster_rank();
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) { mbar_init(&bar_full, 1); mbar_init(&bar_done, 1); fence_mbar_init(); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  const uint32_t full_leader = mapa(smem_u32(&bar_full), 0);
  // idesc: S32 accum, s8 x s8, A and B MN-major, N = 128, M = 256
  const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) |
                         ((256u >> 4) << 24);
  uint32_t ph = 0;
  for (int k0 = 0; k0 < K; k0 += 128, ph ^= 1) {
    if (threadIdx.x == 0) {
      if (rank == 0) mbar_arrive_expect_tx(&bar_full, 2 * (16384 + 8192));
      tma_load_2d_2sm(sA, &ta, full_leader, (int32_t)(128 * rank), k0);
      tma_load_2d_2sm(sB, &tb, full_leader, (int32_t)(64 * rank), k0);
    }
    if (rank == 0 && threadIdx.x == 0) {
      mbar_wait(&bar_full, ph);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = smem_desc(smem_u32(sA) + kk * 4096, 16384, 1024, 2);          // SW128
        const uint64_t bd = smem_desc(smem_u32(sB) + kk * 2048, (uint32_t)lbo_b, 512, 4);  // SW64
        mma_i8_2sm(tmem, ad, bd, idesc, (k0 > 0 || kk > 0) ? 1u : 0u);
      }
      commit_2sm(&bar_done);
    }
    mbar_wait(&bar_done, ph);  // both CTAs: MMA finished reading this stage
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t row = warp * 32 + lane_id();
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t r[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int t = 0; t < 16; ++t) D[(128 * rank + row) * 128 + c0 + t] = (int)r[t];
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

int main() {
  const int K = 512;
  std::vector<int8_t> hA(K * 256), hB(K * 128);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int8_t)((s >> 24) - 128); };
  for (auto& v : hA) v = rnd();
  for (auto& v : hB) v = rnd();
  std::vector<long long> ref(256 * 128, 0);
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < 128; ++n) ref[m * 128 + n] += (long long)hA[k * 256 + m] * hB[k * 128 + n];
  int8_t *dA, *dB; int* dD;
  CK(cudaMalloc(&dA, K * 256)); CK(cudaMalloc(&dB, K * 128)); CK(cudaMalloc(&dD, 256 * 128 * 4));
  CK(cudaMemcpy(dA, hA.data(), K * 256, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), K * 128, cudaMemcpyHostToDevice));
  CUtensorMap ta = make_map(dA, 256, K, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap tb = make_map(dB, 128, K, 64, CU_TENSOR_MAP_SWIZZLE_64B);
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 25 * 1024 + 1024));
  for (int lbo : {8192, 0}) {
    CK(cudaMemset(dD, 0, 256 * 128 * 4));
    probe<<<2, 128, 25 * 1024 + 1024>>>(ta, tb, K, lbo, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("lbo_b=%d: CUDA error %s\n", lbo, cudaGetErrorString(e)); return 1; }
    std::vector<int> hD(256 * 128);
    CK(cudaMemcpy(hD.data(), dD, 256 * 128 * 4, cudaMemcpyDeviceToHost));
    long long bad = 0, bad0 = 0, bad1 = 0;
    for (int i = 0; i < 256 * 128; ++i)
      if ((long long)hD[i] != ref[i]) { ++bad; if (i < 128 * 128) ++bad0; else ++bad1; }
    printf("2-CTA int8 M=256 N=128 (A SW128 MN, B SW64 MN lbo=%d): %s (mismatches %lld: rank0 %lld rank1 %lld) D[0]=%d ref %lld\n",
           lbo, bad ? "FAIL" : "EXACT", bad, bad0, bad1, hD[0], ref[0]);
  }
  return 0;
}
