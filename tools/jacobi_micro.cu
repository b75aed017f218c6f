// jacobi_micro.cu — cycles per sweep step of the RR Jacobi (k_eig.cu jacobi_onesided) in one CTA,
// for several block sizes, plus an empty barrier loop as the floor.  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/jacobi_micro.cu -o /tmp/jm && /tmp/jm
#include "../paper_2603_10444_b200/csrc/k_eig.cu"
#include <cstdio>
#include <vector>
#include <random>
namespace avd {
void set_error(const std::string&) {}
cudaError_t smem_attr_impl(const void* fn, int bytes) { return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); }
}
using namespace avd;

template <int P>
__global__ void jk(const double* Ain, int cap, long long* clk, int* sw) {
  __shared__ double A[P * (P + 1)];
  __shared__ double Vt[P * P];
  __shared__ int fl[2];
  for (int t = threadIdx.x; t < P * P; t += blockDim.x) {
    A[(t / P) * (P + 1) + t % P] = Ain[t];
    Vt[t] = (t / P == t % P) ? 1.0 : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
  int s = jacobi_onesided<P, P + 1>(A, Vt, fl, cap, P);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { clk[0] = t1 - t0; sw[0] = s; }
}
__global__ void bar_only(int steps, long long* clk) {
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
}

int main2();
int main() {
  main2();
  constexpr int P = 48;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> B(P * P), H(P * P, 0.0);
  for (auto& x : B) x = nd(g);
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) {
      double s = 0;
      for (int k = 0; k < P; ++k) s += B[k * P + i] * B[k * P + j] * (1.0 + 10.0 * (k < 8));
      H[i * P + j] = s / 100.0;
    }
  double* dA; long long* clk; int* sw;
  cudaMalloc(&dA, P * P * 8); cudaMalloc(&clk, 8); cudaMalloc(&sw, 4);
  cudaMemcpy(dA, H.data(), P * P * 8, cudaMemcpyHostToDevice);
  for (int nt : {1024, 768, 384, 256, 128}) {
    for (int cap : {1, 3, 40}) {
      jk<P><<<1, nt>>>(dA, cap, clk, sw);
      long long c; int s;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&s, sw, 4, cudaMemcpyDeviceToHost);
      printf("threads %4d cap %2d: sweeps %d  cycles %lld  per step %.0f\n", nt, cap, s, c, (double)c / (s * (P - 1)));
    }
    bar_only<<<1, nt>>>(1000, clk);
    long long c;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d: empty barrier %.1f cycles\n", nt, c / 1000.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
// ---- phase probe: a copy of one step of jacobi_onesided with clock64 stamps (warp 0)
template <int P, int LDA>
__global__ void jk_probe(const double* Ain, long long* ph) {
  __shared__ double A[P * LDA];
  __shared__ double Vt[P * P];
  __shared__ int fl[2];
  for (int t = threadIdx.x; t < P * P; t += blockDim.x) { A[(t / P) * LDA + t % P] = Ain[t]; Vt[t] = (t / P == t % P); }
  __syncthreads();
  constexpr int half = P / 2, E = (P + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  for (int step = 0; step < P - 1; ++step) {
    long long c0 = clock64(), c1 = c0, c2 = c0, c3 = c0, c4 = c0;
    for (int u = warp; u < half; u += nwarps) {
      int pc, qc;
      rr_pair(P, step, u, pc, qc);
      double ap[E], aq[E], al = 0, be = 0, ga = 0;
#pragma unroll
      for (int t = 0; t < E; ++t) {
        const int i = lane + 32 * t;
        ap[t] = i < P ? A[i * LDA + pc] : 0.0;
        aq[t] = i < P ? A[i * LDA + qc] : 0.0;
        al = fma(ap[t], ap[t], al); be = fma(aq[t], aq[t], be); ga = fma(ap[t], aq[t], ga);
      }
      c1 = clock64();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xFFFFFFFFu, al, o);
        be += __shfl_xor_sync(0xFFFFFFFFu, be, o);
        ga += __shfl_xor_sync(0xFFFFFFFFu, ga, o);
      }
      c2 = clock64();
      double c, sn; bool rot;
      jacobi_rotation(al, be, ga, c, sn, rot, 1e-20);
      c3 = clock64();
      if (rot) {
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int i = lane + 32 * t;
          if (i < P) {
            A[i * LDA + pc] = c * ap[t] - sn * aq[t];
            A[i * LDA + qc] = sn * ap[t] + c * aq[t];
            const double vp = Vt[pc * P + i], vq = Vt[qc * P + i];
            Vt[pc * P + i] = c * vp - sn * vq;
            Vt[qc * P + i] = sn * vp + c * vq;
          }
        }
      }
      c4 = clock64();
    }
    __syncthreads();
    long long c5 = clock64();
    acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3; acc[4] += c5 - c4; acc[5] += c5 - c0;
  }
  if (threadIdx.x == 0) for (int i = 0; i < 6; ++i) ph[i] = acc[i] / (P - 1);
  if (threadIdx.x == 0) fl[0] = 0;
}
int main2() {
  constexpr int P = 48;
  std::vector<double> H(P * P);
  std::mt19937_64 g(2); std::normal_distribution<double> nd;
  for (int i = 0; i < P; ++i) for (int j = 0; j <= i; ++j) { double v = nd(g); H[i * P + j] = H[j * P + i] = (i == j) ? 10 + v : v; }
  double* dA; long long* ph;
  cudaMalloc(&dA, P * P * 8); cudaMalloc(&ph, 64);
  cudaMemcpy(dA, H.data(), P * P * 8, cudaMemcpyHostToDevice);
  for (int nt : {768, 256}) {
    jk_probe<P, P + 1><<<1, nt>>>(dA, ph);
    long long h[6]; cudaMemcpy(h, ph, 48, cudaMemcpyDeviceToHost);
    printf("probe threads %d: load %lld, shfl %lld, rot %lld, write %lld, barrier-wait %lld, step %lld cycles\n", nt, h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  return 0;
}
