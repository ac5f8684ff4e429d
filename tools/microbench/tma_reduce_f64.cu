// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_reduce_f64 tma_reduce_f64.cu
// Result on B200 (round 1): FLOAT64 tensor-map reduce-add works (h[0]=1.5 h[1]=2.5 h[16]=0.5 ...)
// does cp.reduce.async.bulk.tensor .add work for FLOAT64 tensor maps on sm_100a?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
__global__ void k(const __grid_constant__ CUtensorMap map, int rows) {
  __shared__ alignas(128) double s[16 * 16];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s[i] = 1.0 + i;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(0), "r"((unsigned)__cvta_generic_to_shared(s))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}
int main() {
  const int rows = 64, cols = 16;
  std::vector<double> h(rows * cols);
  for (int i = 0; i < rows * cols; ++i) h[i] = 0.5;
  double* d; cudaMalloc(&d, sizeof(double) * rows * cols);
  cudaMemcpy(d, h.data(), sizeof(double) * rows * cols, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)rows * 8};
  cuuint32_t box[2] = {16, 16}, es[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 128>>>(map, rows);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(h.data(), d, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost);
  printf("h[0]=%g h[1]=%g h[16]=%g h[64]=%g h[17*64]=%g\n", h[0], h[1], h[16], h[64], h[15*64+15]);
  return 0;
}
