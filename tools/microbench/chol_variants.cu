// Variants of the b x b (b = 16, 32) warp Cholesky for the cluster kernel, timed with clock64.
#include <cstdio>
#include <cuda_runtime.h>

// V1: registers + shuffles (current cl_chol_reg)
template <int B>
__device__ void v1(double* U, double* dinv) {
  const int lane = threadIdx.x;
  double x[B];
#pragma unroll
  for (int i = 0; i < B; ++i) x[i] = (lane < B && i <= lane) ? U[i + lane * B] : 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const double d = __shfl_sync(0xffffffffu, x[k], k);
    const double r = rsqrt(d), ukk = d * r;
    if (lane > k) x[k] *= r;
    if (lane == k) { x[k] = ukk; dinv[k] = r; }
#pragma unroll
    for (int i = k + 1; i < B; ++i) {
      const double uki = __shfl_sync(0xffffffffu, x[k], i);
      if (lane >= i) x[i] = fma(-uki, x[k], x[i]);
    }
  }
  if (lane < B)
#pragma unroll
    for (int i = 0; i < B; ++i) U[i + lane * B] = i <= lane ? x[i] : 0.0;
}

// V2: registers for the own column; row k broadcast through shared memory
template <int B>
__device__ void v2(double* U, double* dinv, double* row) {
  const int lane = threadIdx.x;
  double x[B];
#pragma unroll
  for (int i = 0; i < B; ++i) x[i] = (lane < B && i <= lane) ? U[i + lane * B] : 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    if (lane == k) row[k] = x[k];
    __syncwarp();
    const double d = row[k];
    const double r = rsqrt(d), ukk = d * r;
    const double ukj = lane == k ? ukk : x[k] * r;
    x[k] = lane >= k ? ukj : x[k];
    if (lane == k) dinv[k] = r;
    if (lane > k && lane < B) row[lane] = ukj;
    __syncwarp();
#pragma unroll
    for (int i = k + 1; i < B; ++i)
      if (lane >= i) x[i] = fma(-row[i], ukj, x[i]);
    __syncwarp();
  }
  if (lane < B)
#pragma unroll
    for (int i = 0; i < B; ++i) U[i + lane * B] = i <= lane ? x[i] : 0.0;
}

// V3: smem only (lane j owns column j), loop not unrolled
template <int B>
__device__ void v3(double* U, double* dinv) {
  const int lane = threadIdx.x;
  for (int k = 0; k < B; ++k) {
    const double d = U[k + k * B];
    const double r = rsqrt(d);
    __syncwarp();
    double ukj = 0.0;
    if (lane > k && lane < B) { ukj = U[k + lane * B] * r; U[k + lane * B] = ukj; }
    if (lane == k) { U[k + k * B] = d * r; dinv[k] = r; }
    __syncwarp();
    if (lane > k && lane < B) {
#pragma unroll 4
      for (int i = k + 1; i <= lane; ++i) U[i + lane * B] = fma(-U[k + i * B], ukj, U[i + lane * B]);
    }
    __syncwarp();
  }
}

template <int B, int V>
__global__ void bench(const double* W, double* out, long long* cyc) {
  __shared__ double U[B * B], dinv[B], row[B];
  long long tot = 0;
  for (int rep = 0; rep < 8; ++rep) {
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) U[e] = W[e];
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x < 32) {
      if (V == 1) v1<B>(U, dinv);
      if (V == 2) v2<B>(U, dinv, row);
      if (V == 3) v3<B>(U, dinv);
    }
    __syncthreads();
    long long t1 = clock64();
    if (rep) tot += t1 - t0;
  }
  if (threadIdx.x == 0) cyc[0] = tot / 7;
  for (int e = threadIdx.x; e < B * B; e += blockDim.x) out[e] = U[e];
}

template <int B, int V>
void run(double* ref) {
  double h[B * B];
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < B; ++j) h[i + j * B] = (i == j ? B + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *W, *o; long long* c; long long hc;
  cudaMalloc(&W, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&c, 8);
  cudaMemcpy(W, h, sizeof(h), cudaMemcpyHostToDevice);
  bench<B, V><<<1, 256>>>(W, o, c);
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  double md = 0;
  if (ref) for (int e = 0; e < B * B; ++e) md = fmax(md, fabs(h[e] - ref[e]));
  if (ref && V == 1) for (int e = 0; e < B * B; ++e) ref[e] = h[e];
  printf("\"b%d_v%d\": [%lld, %.1e], ", B, V, hc, md);
}

int main() {
  static double r16[256], r32[1024];
  printf("{");
  run<16, 1>(r16); run<16, 2>(r16); run<16, 3>(r16);
  run<32, 1>(r32); run<32, 2>(r32); run<32, 3>(r32);
  printf("\"end\": 0}\n");
  return 0;
}
