// lat_micro.cu — dependent-chain latency (cycles per op) of a few instructions on this GPU.
#include <cstdio>
__global__ void k(double* out, long long* clk, int n) {
  double x = out[0], y = out[1];
  float f = (float)out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);             // DFMA chain
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) f = __fmaf_rn(f, 0.999f, 0.5f); // FFMA chain
  long long t2 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = (double)(float)z * 1.0000001; // F2F x2 + DMUL
  long long t3 = clock64();
  double w = z;
  for (int i = 0; i < n; ++i) w += __shfl_xor_sync(0xFFFFFFFFu, w, 1); // SHFL x2 + DADD
  long long t4 = clock64();
  float r = f;
  for (int i = 0; i < n; ++i) r = rsqrtf(r + 1.0f);            // MUFU + FADD
  long long t5 = clock64();
  double q = w;
  for (int i = 0; i < n; ++i) q = sqrt(q + 1.0);               // fp64 sqrt (software)
  long long t6 = clock64();
  out[3] = x + f + z + w + r + q;
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; clk[4] = t5 - t4; clk[5] = t6 - t5; }
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  double h[4] = {1.0, 0.999, 1.0, 0};
  cudaMemcpy(o, h, 32, cudaMemcpyHostToDevice);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n);
  k<<<1, 32>>>(o, c, n);
  long long r[6];
  cudaMemcpy(r, c, 48, cudaMemcpyDeviceToHost);
  const char* nm[6] = {"DFMA", "FFMA", "F2F.F32.F64+F2F.F64.F32+DMUL", "SHFL.f64+DADD", "MUFU.RSQ+FADD", "sqrt f64"};
  for (int i = 0; i < 6; ++i) printf("%-32s %.1f cycles/iter\n", nm[i], (double)r[i] / n);
}
