// Dependent-chain latency of the FP64 scalar operations the small Cholesky kernels sit on
// (one thread, clock64 around N dependent operations).  nvcc -O3 -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

#define N 256
__global__ void lat(double* out, long long* cyc, double seed) {
  double x = seed, y = seed * 0.5;
  long long t0, t1;
  // DFMA
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64(); cyc[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[1] = t1 - t0;
  // sqrt (correctly rounded)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = sqrt(x) + 0.5;
  t1 = clock64(); cyc[2] = t1 - t0;
  // rsqrt
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); cyc[3] = t1 - t0;
  // division
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); cyc[4] = t1 - t0;
  // MUFU.RCP64H approximation (__drcp_rn is correctly rounded; use it)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 0.5;
  t1 = clock64(); cyc[5] = t1 - t0;
  // shfl of a double (dependent)
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31) + 1.0;
  t1 = clock64(); cyc[6] = t1 - t0;
  // DADD
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = x + 1e-3;
  t1 = clock64(); cyc[7] = t1 - t0;
  // __dsqrt_rn
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) x = __dsqrt_rn(x) + 0.25;
  t1 = clock64(); cyc[8] = t1 - t0;
  // float sqrt approx (MUFU) for reference
  float f = (float)seed;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) f = __fsqrt_rn(f) + 0.5f;
  t1 = clock64(); cyc[9] = t1 - t0;
  out[threadIdx.x] = x + y + f;
}

int main() {
  double* o; long long* c; long long h[10];
  cudaMalloc(&o, 32 * sizeof(double)); cudaMalloc(&c, 10 * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) {
    lat<<<1, 32>>>(o, c, 1.7);
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  }
  const char* nm[10] = {"dfma", "dmul", "sqrt", "rsqrt", "div", "drcp_rn", "shfl.f64+dadd", "dadd", "dsqrt_rn", "fsqrt_rn"};
  printf("{");
  for (int i = 0; i < 10; ++i) printf("%s\"%s\": %.1f", i ? ", " : "", nm[i], (double)h[i] / N);
  printf("}\n");
  return 0;
}
