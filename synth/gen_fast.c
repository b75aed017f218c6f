/* gen_fast.c — the SAME seeded generator as synth/gen.py, in C, for filling host matrices of
 * bench scale quickly (c5 = 8.6e9 entries) on the oracle side.  Holds none of the method's
 * arithmetic.  Every floating operation is the IEEE fp64 op the torch version issues, in the same
 * order (-ffp-contract=off), so the output is bit-identical (tests/test_oracle_pins.py pins it
 * against synth.gen.generate).  The planted parameters (Walsh codes a_r, b_r, c_r, mu) come from
 * synth.gen.planted. */
#include <stdint.h>
#include <stdlib.h>

static inline uint32_t h32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}
static inline double walsh(int64_t a, int64_t i) { return __builtin_parityll((unsigned long long)(a & i)) ? -1.0 : 1.0; }

int synth_fill(float* out, int64_t row0, int64_t rows, int64_t m, const double* mu, int32_t ks,
               const int64_t* a, const int64_t* b, const double* c, int32_t tail, double sigma_t,
               uint32_t seed_mix) {
  uint32_t* hj = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)m);
  double* hb = (double*)malloc(sizeof(double) * (size_t)(ks > 0 ? ks : 1) * (size_t)m);
  if (!hj || !hb) { free(hj); free(hb); return 1; }
  for (int64_t j = 0; j < m; ++j) {
    hj[j] = h32((uint32_t)((uint64_t)j ^ (uint64_t)seed_mix));
    for (int32_t r = 0; r < ks; ++r) hb[(int64_t)r * m + j] = walsh(b[r], j);
  }
  uint32_t kt[12];
  for (int t = 0; t < 12; ++t) kt[t] = (uint32_t)(0x632BE5ABull * (uint64_t)(t + 1));
#pragma omp parallel for schedule(static)
  for (int64_t rr = 0; rr < rows; ++rr) {
    const int64_t i = row0 + rr;
    double ha[128];
    for (int32_t r = 0; r < ks && r < 128; ++r) ha[r] = walsh(a[r], i) * c[r];
    const uint32_t hi = h32((uint32_t)((uint64_t)i ^ 0x3C6EF372ull));
    float* o = out + rr * m;
    for (int64_t j = 0; j < m; ++j) {
      double acc = mu[j];
      for (int32_t r = 0; r < ks; ++r) {
        if (c[r] == 0.0) continue;
        acc = acc + ha[r] * hb[(int64_t)r * m + j];
      }
      if (tail) {
        const uint32_t base = h32(hi ^ hj[j]);
        double z = 0.0;
        for (int t = 0; t < 12; ++t) z = z + (double)(h32(base ^ kt[t]) >> 8);
        z = z / 16777216.0 - 6.0;
        acc = acc + sigma_t * z;
      }
      o[j] = (float)acc;
    }
  }
  free(hj);
  free(hb);
  return 0;
}
