// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I$NCCL/include -o nccl_lsa_allreduce nccl_lsa_allreduce.cu -L$NCCL/lib -l:libnccl.so.2
// Result on 2 B200 (round 1): correct for 5 iterations, 9.5 us per fused call (8 CTAs, 4096 doubles)
// standalone check of the NCCL 2.28 device API (symmetric window + LSA barrier) on 2 GPUs:
// every rank writes its vector into slot[rank] of every peer's window, LSA barrier per CTA,
// then sums the slots in rank order.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r != ncclSuccess) { printf("NCCL %s @%d: %s\n", #x, __LINE__, ncclGetErrorString(r)); return 1; } } while (0)

constexpr int G = 8;  // CTAs = barrier indices

__global__ void k_fused(ncclDevComm dc, ncclWindow_t win, int n, int nranks, int rank, double* out, int iter) {
  // this CTA owns elements e = blockIdx.x + G * t
  const int buf = iter & 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += G * blockDim.x) {
    const double v = 1000.0 * rank + e + 0.5 * iter;
    for (int peer = 0; peer < nranks; ++peer) {
      double* dst = (double*)ncclGetLsaPointer(win, sizeof(double) * ((size_t)(buf * nranks + rank) * n), peer);
      dst[e] = v;
    }
  }
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  const double* mine = (const double*)ncclGetLocalPointer(win, sizeof(double) * ((size_t)buf * nranks * n));
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += G * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += mine[(size_t)r * n + e];
    out[e] = s;
  }
}

int main() {
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  const int P = ndev >= 2 ? 2 : 1;
  std::vector<ncclComm_t> comms(P);
  std::vector<int> devs(P);
  for (int i = 0; i < P; ++i) devs[i] = i;
  NK(ncclCommInitAll(comms.data(), P, devs.data()));
  const int n = 4096;
  const size_t bytes = sizeof(double) * 2 * P * n;
  std::vector<void*> bufs(P);
  std::vector<ncclWindow_t> wins(P);
  std::vector<ncclDevComm_t> dcs(P);
  std::vector<double*> outs(P);
  std::vector<cudaStream_t> sts(P);
  for (int i = 0; i < P; ++i) {
    CK(cudaSetDevice(i));
    NK(ncclMemAlloc(&bufs[i], bytes < 4096 ? 4096 : bytes));
    CK(cudaMalloc(&outs[i], sizeof(double) * n));
    CK(cudaStreamCreate(&sts[i]));
  }
  NK(ncclGroupStart());
  for (int i = 0; i < P; ++i) NK(ncclCommWindowRegister(comms[i], bufs[i], bytes, &wins[i], NCCL_WIN_COLL_SYMMETRIC));
  NK(ncclGroupEnd());
  ncclDevCommRequirements_t req = {};
  req.lsaBarrierCount = G;
  NK(ncclGroupStart());
  for (int i = 0; i < P; ++i) NK(ncclDevCommCreate(comms[i], &req, &dcs[i]));
  NK(ncclGroupEnd());
  printf("setup ok P=%d\n", P);
  for (int iter = 0; iter < 5; ++iter) {
    for (int i = 0; i < P; ++i) {
      CK(cudaSetDevice(i));
      k_fused<<<G, 256, 0, sts[i]>>>(dcs[i], wins[i], n, P, i, outs[i], iter);
      CK(cudaGetLastError());
    }
    for (int i = 0; i < P; ++i) { CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(sts[i])); }
    int bad = 0;
    for (int i = 0; i < P; ++i) {
      std::vector<double> h(n);
      CK(cudaSetDevice(i));
      CK(cudaMemcpy(h.data(), outs[i], sizeof(double) * n, cudaMemcpyDeviceToHost));
      for (int e = 0; e < n; ++e) {
        double ex = 0; for (int r = 0; r < P; ++r) ex += 1000.0 * r + e + 0.5 * iter;
        if (h[e] != ex) { if (bad < 3) printf("rank %d e %d got %g want %g\n", i, e, h[e], ex); ++bad; }
      }
    }
    printf("iter %d bad %d\n", iter, bad);
  }
  // timing: 200 back-to-back calls
  cudaEvent_t a, b; CK(cudaSetDevice(0)); CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, sts[0]));
  for (int iter = 0; iter < 200; ++iter)
    for (int i = 0; i < P; ++i) { CK(cudaSetDevice(i)); k_fused<<<G, 256, 0, sts[i]>>>(dcs[i], wins[i], n, P, i, outs[i], iter); }
  CK(cudaSetDevice(0)); CK(cudaEventRecord(b, sts[0]));
  for (int i = 0; i < P; ++i) { CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(sts[i])); }
  float ms; CK(cudaEventElapsedTime(&ms, a, b)); printf("fused call: %.2f us\n", 1000.0 * ms / 200);
  // NCCL allreduce of the same size for comparison
  CK(cudaSetDevice(0)); CK(cudaEventRecord(a, sts[0]));
  for (int iter = 0; iter < 200; ++iter) {
    NK(ncclGroupStart());
    for (int i = 0; i < P; ++i) NK(ncclAllReduce(outs[i], outs[i], n, ncclFloat64, ncclSum, comms[i], sts[i]));
    NK(ncclGroupEnd());
  }
  CK(cudaSetDevice(0)); CK(cudaEventRecord(b, sts[0]));
  for (int i = 0; i < P; ++i) { CK(cudaSetDevice(i)); CK(cudaStreamSynchronize(sts[i])); }
  CK(cudaEventElapsedTime(&ms, a, b)); printf("ncclAllReduce: %.2f us\n", 1000.0 * ms / 200);
  return 0;
}
