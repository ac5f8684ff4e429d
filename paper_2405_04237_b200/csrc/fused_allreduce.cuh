// fused_allreduce.cuh -- the split-row reduction fused with the cross-GPU sum (SURVEY §8(e),
// NEXT-f1's "fold the cross-GPU reduce into the reduce kernel"), over NVLink peer memory with
// the NCCL 2.28 device API: a symmetric window (ncclMemAlloc + ncclCommWindowRegister) holds
// one p x q slot per rank on every GPU, and LSA barriers synchronise CTAs of the same index
// across the ranks.
//
// k_reduce_allreduce (one launch replaces k_reduce + ncclAllReduce of Alg. 2 l.3 P:154,
// Alg. 7 l.3/l.8 P:345/Alg. 8 l.3/l.7):
//   1. every CTA forms the local sum of the split-row partials of its 32-element groups (the
//      fixed order of k_reduce) and stores it into slot[parity][rank] of EVERY rank's window;
//   2. LSA barrier (acq_rel, per CTA index): all ranks' slots of these groups have landed;
//   3. out = slot[parity][0] + ... + slot[parity][P-1] in rank order from the local window --
//      a fixed order, so every rank gets the same bits (R is replicated bitwise) and
//      the result is run-to-run deterministic (unlike a library allreduce).
// parity = the barrier's epoch (number of completed syncs of this CTA index: the same on every
// rank, persistent across CUDA-graph replays) & 1.  The window layout does NOT depend on the
// call's p x q: half h holds nranks slots of `cap` doubles each (cap = b*n, the largest block
// any call sums), element e of rank r's slot sits at h*nranks*cap + r*cap + e, and element e
// is written AND read by CTA index (e/32) mod gridDim in every call.  So a fast rank's next
// call (other half) never touches what this call reads, and its call after that (same half)
// reaches its write phase only after passing the intermediate barrier of the same CTA index,
// which every rank's CTA enters only after finishing this call's reads -- one barrier per call.
// (A layout sized by the current call's p*q would let consecutive calls with different block
// shapes overlap across halves.)
// Every rank executes the barrier even after a breakdown (the status is identical on all
// ranks because all factor the same allreduced Gram, but the barriers must still match).
#pragma once
#include <nccl_device.h>

namespace tsqr {

constexpr int AR_CTAS = 148;  // CTAs of the fused kernel (one per SM) = LSA barrier indices
constexpr int AR_NT = 256;

__global__ void __launch_bounds__(AR_NT) k_reduce_allreduce(const double* __restrict__ part, int Sfull, int Sdiag,
                                                            int p, int q, int ldp, int64_t pstride,
                                                            double* __restrict__ out, int ldo, int gram,
                                                            const int* status, ncclDevComm dc, ncclWindow_t win,
                                                            int nranks, int rank, int64_t cap) {
  __shared__ double ws[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool skip = failed(status);  // uniform across CTAs and ranks
  const int64_t pq = (int64_t)p * q;
  const int64_t ngroups = (pq + 31) / 32;
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x);
  const size_t half = (size_t)(bar.epoch & 1) * (size_t)nranks * (size_t)cap;  // window half of this call
  if (!skip) {
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int64_t e = g * 32 + lane;
      const int i = (int)(e % p), j = (int)(e / p);
      const bool live = e < pq && !(gram && i > j);
      const int S = !live ? 0 : ((gram && (i >> 6) == (j >> 6)) ? Sdiag : Sfull);
      const double* src = part + i + (int64_t)j * ldp;
      double s[4] = {0, 0, 0, 0};
      for (int t = warp; t < S; t += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t + 8 * u < S) s[u] += src[(int64_t)(t + 8 * u) * pstride];
      }
      ws[warp][lane] = (s[0] + s[1]) + (s[2] + s[3]);
      __syncthreads();
      if (warp == 0 && live) {
        const double v = ((ws[0][lane] + ws[1][lane]) + (ws[2][lane] + ws[3][lane])) +
                         ((ws[4][lane] + ws[5][lane]) + (ws[6][lane] + ws[7][lane]));
        const size_t off = sizeof(double) * (half + (size_t)rank * (size_t)cap + (size_t)e);
        for (int r = 0; r < nranks; ++r) *reinterpret_cast<double*>(ncclGetLsaPointer(win, off, r)) = v;
      }
      __syncthreads();
    }
  }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  if (!skip && threadIdx.x < 32) {
    const double* slots = reinterpret_cast<const double*>(ncclGetLocalPointer(win, 0)) + half;
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int64_t e = g * 32 + lane;
      const int i = (int)(e % p), j = (int)(e / p);
      if (e < pq && !(gram && i > j)) {
        double v = slots[e];
        for (int r = 1; r < nranks; ++r) v += slots[(size_t)r * (size_t)cap + (size_t)e];
        out[i + (int64_t)j * ldo] = v;
        if (gram && i != j) out[j + (int64_t)i * ldo] = v;
      }
    }
  }
}

}  // namespace tsqr
