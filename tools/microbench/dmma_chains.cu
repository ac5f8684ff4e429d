// DMMA.8x8x4 throughput vs independent accumulator chains per warp and warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_chains dmma_chains.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chains(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}

// same with A/B fragments loaded from shared memory every step (like the real kernels)
template <int ILP>
__global__ void chains_lds(double* out, int iters) {
  __shared__ double sm[64 * 68];
  for (int i = threadIdx.x; i < 64 * 68; i += blockDim.x) sm[i] = i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
    const int k0 = (it & 15) * 4 + tig;
    double fa[ILP], fb = sm[gid * 68 + k0];
#pragma unroll
    for (int i = 0; i < ILP; ++i) fa[i] = sm[k0 * 68 + (i & 7) * 8 + gid];
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(fa[i]), "d"(fb));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters) {
  double* out;
  cudaMalloc(&out, 64);
  kern<<<blocks, threads>>>(out, iters);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaFree(out);
  return best;
}

int main() {
  const int sms = 148, iters = 4096;
  printf("{");
  bool first = true;
  auto rep = [&](const char* name, int ilp, int wps, float ms) {
    // wps = warps per SMSP -> blocks of 128*wps threads, one block per SM
    double fl = 2.0 * 256 * ilp * (double)iters * sms * 4 * wps;
    printf("%s\"%s_ilp%d_w%d\": %.2f", first ? "" : ", ", name, ilp, wps, fl / ms / 1e9);
    first = false;
  };
  for (int wps : {1, 2, 3, 4}) {
    rep("reg", 2, wps, run(chains<2>, sms, 128 * wps, iters));
    rep("reg", 4, wps, run(chains<4>, sms, 128 * wps, iters));
    rep("reg", 8, wps, run(chains<8>, sms, 128 * wps, iters));
    rep("reg", 16, wps, run(chains<16>, sms, 128 * wps, iters));
    rep("lds", 4, wps, run(chains_lds<4>, sms, 128 * wps, iters));
    rep("lds", 8, wps, run(chains_lds<8>, sms, 128 * wps, iters));
    rep("lds", 16, wps, run(chains_lds<16>, sms, 128 * wps, iters));
  }
  printf("}\n");
  return 0;
}
