// FP64 peak microbenchmarks for B200 (sm_100a): DFMA register loop, mma.sync f64
// (DMMA) shapes, and an HBM copy. Writes one JSON object to stdout.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double s) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], s, 1e-9);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += acc[i];
  if (r == 12345.678) out[0] = r;
}

// m8n8k4: A 1, B 1, C 2 doubles per lane
template <int ILP>
__global__ void dmma_m8n8k4(double* out, int iters) {
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

template <int ILP>
__global__ void dmma_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

template <int ILP>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0; b[1] = 0.5;
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

template <int ILP>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 / (i + 1);
  double c[ILP][4];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

__global__ void copy_kernel(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) dst[i] = src[i];
}

template <typename F>
static float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a); cudaEventDestroy(b);
  return best;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  printf("{\"sms\": %d", sms);
  const int iters = 4096;
  // DFMA: 8 warps per block, several blocks per SM
  for (int bpsm : {2, 4, 8}) {
    int blocks = sms * bpsm, threads = 256;
    float ms = time_it([&] { dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999999); }, 5);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_ilp8_bpsm%d_tflops\": %.3f", bpsm, fl / ms / 1e9);
  }
  auto mma_run = [&](const char* name, auto kern, double flops_per_mma, int ilp) {
    for (int bpsm : {1, 2, 4}) {
      int blocks = sms * bpsm, threads = 256;
      float ms = time_it([&] { kern<<<blocks, threads>>>(out, iters); }, 5);
      double fl = flops_per_mma * ilp * iters * (double)blocks * (threads / 32);
      printf(", \"%s_bpsm%d_tflops\": %.3f", name, bpsm, fl / ms / 1e9);
    }
  };
  mma_run("dmma_m8n8k4_ilp8", dmma_m8n8k4<8>, 2.0 * 8 * 8 * 4, 8);
  mma_run("dmma_m16n8k4_ilp4", dmma_m16n8k4<4>, 2.0 * 16 * 8 * 4, 4);
  mma_run("dmma_m16n8k8_ilp4", dmma_m16n8k8<4>, 2.0 * 16 * 8 * 8, 4);
  mma_run("dmma_m16n8k16_ilp4", dmma_m16n8k16<4>, 2.0 * 16 * 8 * 16, 4);
  mma_run("dmma_m16n8k16_ilp2", dmma_m16n8k16<2>, 2.0 * 16 * 8 * 16, 2);
  // HBM copy, 4 GiB each side
  size_t bytes = (size_t)4 << 30;
  double2 *s, *d;
  CK(cudaMalloc(&s, bytes)); CK(cudaMalloc(&d, bytes));
  CK(cudaMemset(s, 0, bytes));
  size_t n2 = bytes / sizeof(double2);
  for (int bpsm : {4, 8}) {
    float ms = time_it([&] { copy_kernel<<<sms * bpsm, 512>>>(s, d, n2); }, 5);
    printf(", \"copy_bpsm%d_gbs\": %.1f", bpsm, 2.0 * bytes / ms / 1e6);
  }
  float ms = time_it([&] { cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice); }, 5);
  printf(", \"memcpy_d2d_gbs\": %.1f", 2.0 * bytes / ms / 1e6);
  // sustained DMMA for ~4 s
  {
    int blocks = sms * 2, threads = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int n = 0; float total = 0;
    cudaEventRecord(a);
    while (total < 4000.f) {
      for (int r = 0; r < 20; ++r) dmma_m16n8k16<4><<<blocks, threads>>>(out, iters);
      n += 20;
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&total, a, b);
    }
    double fl = 2.0 * 16 * 8 * 16 * 4 * iters * (double)blocks * (threads / 32) * n;
    printf(", \"dmma_m16n8k16_sustained_tflops\": %.3f", fl / total / 1e9);
  }
  {
    int blocks = sms * 4, threads = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int n = 0; float total = 0;
    cudaEventRecord(a);
    while (total < 4000.f) {
      for (int r = 0; r < 20; ++r) dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999999);
      n += 20;
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&total, a, b);
    }
    double fl = 2.0 * 8 * iters * (double)blocks * threads * n;
    printf(", \"dfma_sustained_tflops\": %.3f", fl / total / 1e9);
  }
  printf("}\n");
  return 0;
}
