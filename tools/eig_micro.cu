// eig_micro.cu — micro-benchmark of the K4 building blocks (not product code): times the fused
// m-length reduction kernels of k_eig.cu in isolation (sum only / + Cholesky / + Jacobi, and the
// one-CTA tail alone) and the stream-K GEMMs, with CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo tools/eig_micro.cu -o tools/eig_micro
#define AVD_EIG_PROBE 1
#include "../paper_2603_10444_b200/csrc/k_eig.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace avd {
void set_error(const std::string&) {}
}
using namespace avd;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int MODE>
float time_atb(const double* A, const double* B, int64_t m, int grid, double* part, unsigned* ticket, double* o0,
               double* o1, int* ib, int* st, int reps) {
  constexpr int PC = 3;
  constexpr int p = 48;
  const size_t sm = std::max<size_t>(2 * RedCfg<PC>::chunk * p, (size_t)p * (p + 1) + (size_t)p * p) * sizeof(double);
  CK(cudaFuncSetAttribute(atb_fused_kernel<MODE, PC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) atb_fused_kernel<MODE, PC><<<grid, RedCfg<PC>::threads, sm>>>(A, B, m, part, ticket, o0, o1, ib, st, nullptr);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) atb_fused_kernel<MODE, PC><<<grid, RedCfg<PC>::threads, sm>>>(A, B, m, part, ticket, o0, o1, ib, st, nullptr);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  long long clk[16];
  CK(cudaMemcpyFromSymbol(clk, g_probe_clk, sizeof(clk)));
  printf("    [mode %d grid %d] cycles: partial %lld, ticket %lld, sum %lld, prep %lld, solve %lld | jac phase1 %lld, bar1 %lld\n", MODE, grid,
         clk[1] - clk[0], clk[2] - clk[1], clk[3] - clk[2], MODE ? clk[4] - clk[3] : 0, MODE ? clk[5] - clk[4] : 0, clk[8], clk[9]);
  long long z[16] = {0};
  CK(cudaMemcpyToSymbol(g_probe_clk, z, sizeof(z)));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return 1000.f * ms / reps;
}

int main() {
  const int64_t m = 4096;
  const int p = 48;
  std::vector<double> h(m * p);
  uint32_t s = 1;
  for (auto& v : h) { s = s * 1664525u + 1013904223u; v = ((s >> 8) / 16777216.0) - 0.5; }
  double *A, *part, *o0, *o1;
  unsigned* ticket;
  int *ib, *st;
  CK(cudaMalloc(&A, m * p * 8));
  CK(cudaMalloc(&part, 64 * p * p * 8));
  CK(cudaMalloc(&o0, p * p * 8));
  CK(cudaMalloc(&o1, p * 8));
  CK(cudaMalloc(&ticket, 16));
  CK(cudaMalloc(&ib, p * 4));
  CK(cudaMalloc(&st, 64));
  CK(cudaMemset(ticket, 0, 16));
  CK(cudaMemcpy(A, h.data(), m * p * 8, cudaMemcpyHostToDevice));
  const int grid = (int)ceil_div(m, kRedRows);
  printf("fused reduction, m=%ld p=%d, %d CTAs x %d threads\n", (long)m, p, grid, RedCfg<3>::threads);
  printf("  sum only      : %8.2f us\n", time_atb<0>(A, A, m, grid, part, ticket, o0, o1, ib, st, 50));
  printf("  + Cholesky    : %8.2f us\n", time_atb<1>(A, A, m, grid, part, ticket, o0, o1, ib, st, 50));
  printf("  + Jacobi      : %8.2f us\n", time_atb<2>(A, A, m, grid, part, ticket, o0, o1, ib, st, 10));
  int sw = 0;
  CK(cudaMemcpy(&sw, st, 4, cudaMemcpyDeviceToHost));
  printf("    (jacobi sweeps %d)\n", sw);
  printf("one CTA (m=128): sum %8.2f us, chol %8.2f us, jacobi %8.2f us\n",
         time_atb<0>(A, A, 128, 1, part, ticket, o0, o1, ib, st, 50),
         time_atb<1>(A, A, 128, 1, part, ticket, o0, o1, ib, st, 50),
         time_atb<2>(A, A, 128, 1, part, ticket, o0, o1, ib, st, 10));
  CK(cudaMemcpy(&sw, st, 4, cudaMemcpyDeviceToHost));
  printf("    (jacobi sweeps %d)\n", sw);
  return 0;
}
