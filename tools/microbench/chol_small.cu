// Latency of the cluster kernel's b x b Cholesky variants (one CTA, clock64 per call).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2405_04237_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>
#include "cluster_small.cuh"
using namespace tsqr;

template <int B>
__global__ void bench(const double* W, double* out, long long* cyc, int* status) {
  __shared__ double red[B * B], dinv[2 * B];
  __shared__ int flag[4];
  ClusterSmem<B> s{};
  s.red = red; s.dinv = dinv; s.flag = flag;
  long long tot = 0;
  for (int rep = 0; rep < 8; ++rep) {
    for (int e = threadIdx.x; e < B * B; e += blockDim.x) red[e] = W[e];
    __syncthreads();
    long long t0 = clock64();
    bool ok = cl_chol<B>(s, status, 1, 1, 1, true);
    long long t1 = clock64();
    if (rep) tot += t1 - t0;
    if (!ok) break;
  }
  if (threadIdx.x == 0) cyc[0] = tot / 7;
  for (int e = threadIdx.x; e < B * B; e += blockDim.x) out[e] = red[e];
}

template <int B>
void run() {
  double h[B * B];
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < B; ++j) h[i + j * B] = (i == j ? B + 1.0 : 0.0) + 1.0 / (1 + i + j);
  double *W, *o; long long* c; int* st; long long hc;
  cudaMalloc(&W, sizeof(h)); cudaMalloc(&o, sizeof(h)); cudaMalloc(&c, 8); cudaMalloc(&st, 64);
  cudaMemset(st, 0, 64);
  cudaMemcpy(W, h, sizeof(h), cudaMemcpyHostToDevice);
  bench<B><<<1, CL_NT>>>(W, o, c, st);
  cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("\"chol%d\": %lld%s", B, hc, B == 64 ? "" : ", ");
}

int main() {
  printf("{");
  run<16>(); run<32>(); run<64>();
  printf("}\n");
  return 0;
}
