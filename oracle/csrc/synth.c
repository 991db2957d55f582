/*
 * C copy of the bench's synthetic corpus generator (tools/synth.py, "iso"
 * family) — TEST INFRASTRUCTURE / CPU ARMS ONLY.
 *
 * The CPU baseline and the `bench.py --impl reference` arm need the same 10M x
 * 1024 corpus the GPU arm searches, on the host, in seconds; torch's CPU
 * elementwise path takes minutes.  Every step below is exact integer
 * arithmetic or a correctly rounded IEEE operation, in the same order as
 * tools/synth.py, so the rows are bit-identical to the torch (CPU or CUDA)
 * generator (pinned by tests/test_synth.py and tests/test_gpu_synth.py).
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp, no -ffast-math: IEEE div/sqrt).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ROW_KEY 0xA5A5A5A5u
#define COL_KEY 0x5BD1E995u

static inline uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

static inline float to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u); /* finite inputs only (|x| <= 1) */
  u &= 0xFFFF0000u;
  memcpy(&f, &u, 4);
  return f;
}

/* rows [row0, row0 + nrows) of seed `seed` as float32 (bf16-rounded when
 * bf16 != 0) into out[nrows][d]. */
int synth_rows(int64_t row0, int64_t nrows, int d, uint32_t seed, int bf16, float* out, int nthreads) {
  if (d <= 0 || d > 65536 || nrows < 0) return 1;
  const uint32_t key = mix32(seed ^ ROW_KEY);
  uint32_t hc[2 * 65536];
  for (int j = 0; j < 2 * d; ++j) hc[j] = mix32((uint32_t)j ^ COL_KEY);
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) if (nthreads != 1)
  for (int64_t r = 0; r < nrows; ++r) {
    int32_t v[65536];
    const uint32_t hr = mix32((uint32_t)(row0 + r) ^ key);
    int64_t s = 0;
    for (int j = 0; j < d; ++j) {
      uint32_t h0 = mix32(hr ^ hc[2 * j]), h1 = mix32(hr ^ hc[2 * j + 1]);
      int32_t x = (int32_t)((h0 & 0xFFFFu) + (h0 >> 16) + (h1 & 0xFFFFu) + (h1 >> 16)) - 131070;
      v[j] = x;
      s += (int64_t)x * x;
    }
    const double nrm = sqrt((double)s);
    float* o = out + r * (int64_t)d;
    for (int j = 0; j < d; ++j) {
      float f = (float)((double)v[j] / nrm);
      o[j] = bf16 ? to_bf16_rne(f) : f;
    }
  }
  return 0;
}
