// small_kernels.cuh -- the O(b^3) / O(n^2) kernels of the hot path: fixed-order reduction
// of split partials, single-CTA Cholesky + triangular inverse, and R assembly.
#pragma once
#include "common.cuh"

namespace tsqr {

// -----------------------------------------------------------------------------------------
// k_reduce: OUT[i,j] = sum_s PART[s][i,j] in a fixed order (8 interleaved running sums over
// s, then a pairwise combination) -> deterministic.  gram: only i <= j is read and
// OUT[j,i] = OUT[i,j] (bitwise symmetric, R-11); diagonal 64x64 Gram tiles have Sdiag splits,
// the others Sfull.  ldp: leading dimension of a partial.
// -----------------------------------------------------------------------------------------
// One CTA of 8 warps per 32 consecutive elements: warp w sums the partials s = w (mod 8) with
// 4 interleaved running sums, then lane l of warp 0 adds the 8 warp sums pairwise -- a fixed
// order (deterministic) with 8x the memory parallelism of one thread per element (split counts
// reach ~150-300 partials per output).
constexpr int RED_NT = 256;
__global__ void __launch_bounds__(RED_NT) k_reduce(const double* __restrict__ part, int Sfull, int Sdiag, int p,
                                                   int q, int ldp, int64_t pstride, double* __restrict__ out,
                                                   int ldo, int gram, const int* status) {
  if (failed(status)) return;
  __shared__ double ws[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pq = (int64_t)p * q;
  for (int64_t e0 = (int64_t)blockIdx.x * 32; e0 < pq; e0 += (int64_t)gridDim.x * 32) {
    const int64_t e = e0 + lane;
    const int i = (int)(e % p), j = (int)(e / p);
    const bool live = e < pq && !(gram && i > j);
    const int S = !live ? 0 : ((gram && (i >> 6) == (j >> 6)) ? Sdiag : Sfull);  // splits of this tile
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
      out[i + (int64_t)j * ldo] = v;
      if (gram && i != j) out[j + (int64_t)i * ldo] = v;
    }
    __syncthreads();
  }
}

// -----------------------------------------------------------------------------------------
// k_chol_inv: one CTA.  W (b x b, upper triangle read) = U^T U, unpivoted, right-looking
// (Alg. 1 l.2 P:132; R-5): per pivot k, d = S_kk; breakdown iff !(d > 0) or !isfinite(d);
// u_kk = sqrt(d); u_kj = S_kj / u_kk; S_ij -= u_ki u_kj (k < i <= j).
// Then Z = U^{-1} (R-4) row by row from the bottom: Z_ij = (delta_ij - sum_{t=i+1..j}
// U_it Z_tj) / U_ii for all j >= i in parallel (8 threads per column split the sum).
// Work matrices in shared memory when they fit (b <= 64: S and Z; b = 128: S only),
// otherwise in the global scratch `work` (b x b) / the output Z.
// On breakdown: status <- {5, pass, panel, stage, pivot, -, value(double)}.
// -----------------------------------------------------------------------------------------
constexpr int CHOL_NT = 512;
#ifndef TSQR_CHOL_NT_SMALL
#define TSQR_CHOL_NT_SMALL 512
#endif
constexpr int CHOL_NT_SMALL = TSQR_CHOL_NT_SMALL;  // threads of k_chol_inv (b <= 128 in shared memory)

// shared-memory bytes of k_chol_inv for block size b (S and Z with padded leading dimension
// b + 1 so that row- and column-wise accesses are bank-conflict free)
__host__ __device__ constexpr size_t chol_smem_bytes(int b) {
  return b <= 64 ? sizeof(double) * 2 * (size_t)b * (b + 1) : (b <= 128 ? sizeof(double) * (size_t)b * (b + 1) : 0);
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_chol_inv(const double* __restrict__ W, int ldw, int b,
                                                        double* __restrict__ U, int ldu, double* __restrict__ Z,
                                                        int ldz, int* status, int pass, int panel, int stage,
                                                        double* work) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_urow[256];
  if (failed(status)) return;
  const int tid = threadIdx.x;
  const bool s_in_smem = b <= 128;
  const bool z_in_smem = b <= 64;
  const int lds = s_in_smem ? b + 1 : b;
  double* S = s_in_smem ? smem : work;                          // S[i + j*lds]
  double* Zw = z_in_smem ? smem + (size_t)b * (b + 1) : Z;      // Zw[i + j*ldzw]
  const int ldzw = z_in_smem ? b + 1 : ldz;
  for (int e = tid; e < b * b; e += NT) {
    const int i = e % b, j = e / b;
    S[i + j * lds] = (i <= j) ? W[i + (int64_t)j * ldw] : 0.0;
  }
  __syncthreads();
  // right-looking Cholesky (R-5).  Thread -> column jj = tid % 64 (+64 per pass),
  // rows ii0 = tid / 64 (mod 8): no integer division in the trailing update.
  const int jj = tid & 63, ii0 = tid >> 6;
  for (int k = 0; k < b; ++k) {
    const double d = S[k + k * lds];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) {
        status[1] = pass; status[2] = panel; status[3] = stage; status[4] = k;
        *reinterpret_cast<double*>(status + 6) = d;
        __threadfence();
        status[0] = 5;
      }
      return;  // uniform: every thread read the same d
    }
    const double ukk = sqrt(d);
    for (int j = k + tid; j < b; j += NT) s_urow[j] = (j == k) ? ukk : S[k + j * lds] / ukk;
    __syncthreads();
    for (int j0 = 0; j0 < b; j0 += 64) {
      const int j = j0 + jj;
      if (j < b && j >= k) {
        if (ii0 == 0) S[k + j * lds] = s_urow[j];
        const double uj = s_urow[j];
        for (int i = k + 1 + ((ii0 - (k + 1)) & (NT / 64 - 1)); i <= j; i += NT / 64) S[i + j * lds] = fma(-s_urow[i], uj, S[i + j * lds]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += NT) {
    const int i = e % b, j = e / b;
    U[i + (int64_t)j * ldu] = (i <= j) ? S[i + j * lds] : 0.0;
    Zw[i + (int64_t)j * ldzw] = 0.0;
  }
  __syncthreads();
  // Z = U^{-1} (R-4): rows from the bottom, Z_ij = (delta_ij - sum_{t=i+1..j} U_it Z_tj) / U_ii for
  // all j >= i in parallel; column j handled by 8 lanes of one warp (the t-range split 8 ways)
  const int sub = tid & 7, jg = tid >> 3;
  for (int i = b - 1; i >= 0; --i) {
    for (int jb = 0; jb < b; jb += NT / 8) {  // uniform trip count: shuffles stay converged
      const int j = jb + jg;
      const bool act = j < b && j >= i;
      double s = 0.0;
      if (act)
        for (int t = i + 1 + sub; t <= j; t += 8) s = fma(S[i + t * lds], Zw[t + (int64_t)j * ldzw], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      if (sub == 0 && act) Zw[i + (int64_t)j * ldzw] = (((i == j) ? 1.0 : 0.0) - s) / S[i + i * lds];
    }
    __syncthreads();
  }
  if (z_in_smem)
    for (int e = tid; e < b * b; e += NT) {
      const int i = e % b, j = e / b;
      Z[i + (int64_t)j * ldz] = Zw[i + j * ldzw];
    }
}

// -----------------------------------------------------------------------------------------
// k_chol_inv_blocked: the same factorisation for b in {128, 256} as a blocked algorithm on
// 64x64 blocks (one CTA): for each block column J, factor W_JJ (the scalar right-looking
// kernel above, on a 64x64 block in shared memory) and invert it, form the block row
// U_JK = U_JJ^{-T} W_JK, and update the trailing blocks W_KL -= U_JK^T U_JL (the blocked form
// of the same right-looking elimination, R-5).  Then Z = U^{-1} block column by block column:
// Z_JJ = U_JJ^{-1}, Z_IJ = -Z_II (sum_{K=I+1..J} U_IK Z_KJ) (R-4).  W is copied to the
// workspace `work` (b x b, L2-resident) and updated there.
// -----------------------------------------------------------------------------------------
constexpr int CHB = 64;       // block size
constexpr int CHLD = 65;      // padded leading dimension in shared memory
constexpr size_t CHOL_BLK_SMEM = sizeof(double) * 6 * CHB * CHLD;

// C (64x64, ldc) (+)= op(A) * B for 64x64 blocks in shared memory, 512 threads: thread t owns
// row i = t % 64 and columns c = t / 64 + 8v.  transA: A^T (A[t + i*lda]), else A[i + t*lda].
// triA: A upper triangular (t restricted to the non-zero range).  sign: +1 / -1.
template <bool TRANS_A, bool SUB>
__device__ __forceinline__ void blk_mm(const double* A, const double* B, double* C, int tid) {
  const int i = tid & 63, c0 = tid >> 6;
  double acc[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) acc[v] = SUB ? C[i + (c0 + 8 * v) * CHLD] : 0.0;
  for (int t = 0; t < 64; ++t) {
    const double a = TRANS_A ? A[t + i * CHLD] : A[i + t * CHLD];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      if (SUB) acc[v] = fma(-a, B[t + (c0 + 8 * v) * CHLD], acc[v]);
      else acc[v] = fma(a, B[t + (c0 + 8 * v) * CHLD], acc[v]);
    }
  }
  __syncthreads();  // every thread has read A and B (C may alias neither, but callers reuse buffers)
#pragma unroll
  for (int v = 0; v < 8; ++v) C[i + (c0 + 8 * v) * CHLD] = acc[v];
  __syncthreads();
}

__device__ __forceinline__ void blk_load(double* dst, const double* src, int64_t ld, int tid) {
  for (int e = tid; e < CHB * CHB; e += CHOL_NT) dst[(e & 63) + (e >> 6) * CHLD] = src[(e & 63) + (int64_t)(e >> 6) * ld];
  __syncthreads();
}
__device__ __forceinline__ void blk_store(double* dst, int64_t ld, const double* src, int tid) {
  for (int e = tid; e < CHB * CHB; e += CHOL_NT) dst[(e & 63) + (int64_t)(e >> 6) * ld] = src[(e & 63) + (e >> 6) * CHLD];
  __syncthreads();
}

// factor the 64x64 block D (upper part valid) in place into U_JJ and write its inverse to Di;
// returns false (and sets the status) on breakdown
__device__ bool blk_chol_inv(double* D, double* Di, double* urow, int* status, int pass, int panel, int stage,
                             int piv0, int tid) {
  const int jj = tid & 63, ii0 = tid >> 6;
  for (int k = 0; k < CHB; ++k) {
    const double d = D[k + k * CHLD];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) {
        status[1] = pass; status[2] = panel; status[3] = stage; status[4] = piv0 + k;
        *reinterpret_cast<double*>(status + 6) = d;
        __threadfence();
        status[0] = 5;
      }
      return false;
    }
    const double ukk = sqrt(d);
    if (tid >= k && tid < CHB) urow[tid] = (tid == k) ? ukk : D[k + tid * CHLD] / ukk;
    __syncthreads();
    if (jj >= k) {
      if (ii0 == 0) D[k + jj * CHLD] = urow[jj];
      const double uj = urow[jj];
      for (int i = k + 1 + ((ii0 - (k + 1)) & 7); i <= jj; i += 8) D[i + jj * CHLD] = fma(-urow[i], uj, D[i + jj * CHLD]);
    }
    __syncthreads();
  }
  for (int e = tid; e < CHB * CHB; e += CHOL_NT) {
    const int i = e & 63, j = e >> 6;
    if (i > j) D[i + j * CHLD] = 0.0;
    Di[i + j * CHLD] = 0.0;
  }
  __syncthreads();
  const int sub = tid & 7, jg = tid >> 3;  // 64 columns x 8 lanes
  for (int i = CHB - 1; i >= 0; --i) {
    const int j = jg;
    const bool act = j >= i;
    double sacc = 0.0;
    if (act)
      for (int t = i + 1 + sub; t <= j; t += 8) sacc = fma(D[i + t * CHLD], Di[t + j * CHLD], sacc);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 4);
    if (sub == 0 && act) Di[i + j * CHLD] = (((i == j) ? 1.0 : 0.0) - sacc) / D[i + i * CHLD];
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_inv_blocked(const double* __restrict__ W, int ldw, int b,
                                                                double* __restrict__ U, int ldu, double* __restrict__ Z,
                                                                int ldz, int* status, int pass, int panel, int stage,
                                                                double* work) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_urow[CHB];
  if (failed(status)) return;
  const int tid = threadIdx.x;
  const int nb = b / CHB;
  double* D = smem;                 // diagonal block -> U_JJ
  double* Di = smem + CHB * CHLD;   // U_JJ^{-1}
  double* P = smem + 2 * CHB * CHLD;  // up to 3 panel blocks U_JK
  double* T = smem + 5 * CHB * CHLD;  // scratch block
  // work <- upper triangle of W
  for (int64_t e = tid; e < (int64_t)b * b; e += CHOL_NT) {
    const int i = (int)(e % b), j = (int)(e / b);
    work[i + (int64_t)j * b] = (i <= j) ? W[i + (int64_t)j * ldw] : 0.0;
    U[i + (int64_t)j * ldu] = 0.0;
    Z[i + (int64_t)j * ldz] = 0.0;
  }
  __syncthreads();
  for (int J = 0; J < nb; ++J) {
    blk_load(D, work + (int64_t)J * CHB * b + J * CHB, b, tid);
    if (!blk_chol_inv(D, Di, s_urow, status, pass, panel, stage, J * CHB, tid)) return;
    blk_store(U + (int64_t)J * CHB * ldu + J * CHB, ldu, D, tid);
    blk_store(Z + (int64_t)J * CHB * ldz + J * CHB, ldz, Di, tid);
    // block row: U_JK = U_JJ^{-T} W_JK
    for (int K = J + 1; K < nb; ++K) {
      double* PK = P + (K - J - 1) * CHB * CHLD;
      blk_load(T, work + (int64_t)K * CHB * b + J * CHB, b, tid);
      blk_mm<true, false>(Di, T, PK, tid);
      blk_store(U + (int64_t)K * CHB * ldu + J * CHB, ldu, PK, tid);
    }
    // trailing update: W_KL -= U_JK^T U_JL, J < K <= L
    for (int K = J + 1; K < nb; ++K)
      for (int L2 = K; L2 < nb; ++L2) {
        double* wkl = work + (int64_t)L2 * CHB * b + K * CHB;
        blk_load(T, wkl, b, tid);
        blk_mm<true, true>(P + (K - J - 1) * CHB * CHLD, P + (L2 - J - 1) * CHB * CHLD, T, tid);
        blk_store(wkl, b, T, tid);
      }
  }
  // Z = U^{-1}: block column J, rows I = J-1 .. 0: Z_IJ = -Z_II * sum_{K=I+1..J} U_IK Z_KJ
  for (int J = 1; J < nb; ++J)
    for (int I = J - 1; I >= 0; --I) {
      for (int e = tid; e < CHB * CHB; e += CHOL_NT) P[(e & 63) + (e >> 6) * CHLD] = 0.0;  // S accumulator
      __syncthreads();
      for (int K = I + 1; K <= J; ++K) {
        blk_load(D, U + (int64_t)K * CHB * ldu + I * CHB, ldu, tid);    // U_IK
        blk_load(Di, Z + (int64_t)J * CHB * ldz + K * CHB, ldz, tid);   // Z_KJ
        // P += U_IK Z_KJ  (blk_mm with SUB adds -A*B: accumulate the negative, fixed below)
        blk_mm<false, true>(D, Di, P, tid);
      }
      blk_load(D, Z + (int64_t)I * CHB * ldz + I * CHB, ldz, tid);      // Z_II
      blk_mm<false, false>(D, P, T, tid);                              // Z_II * (-S) = Z_IJ
      blk_store(Z + (int64_t)J * CHB * ldz + I * CHB, ldz, T, tid);
    }
}

// -----------------------------------------------------------------------------------------
// Multi-CTA blocked Cholesky + inverse for wide panels (b = 64 nb > 256, the
// strong-scaling panels of 400-4000 columns): the same right-looking blocked algorithm
// as k_chol_inv_blocked (R-5), one launch per step so the independent blocks of a step run
// on separate CTAs:
//   prep:           work <- upper(W); U, Z <- 0
//   for J:  diag:   U_JJ = chol(W_JJ), Z_JJ = U_JJ^{-1}                       (1 CTA)
//           row:    U_JK = Z_JJ^T W_JK, K > J                                (nb-J-1 CTAs)
//           trail:  W_KL -= U_JK^T U_JL, J < K <= L                          ((nb-J-1)(nb-J)/2 CTAs)
//   for d = 1..nb-1: Z_IJ = -Z_II sum_{K=I+1..J} U_IK Z_KJ, J - I = d        (nb-d CTAs; R-4)
// Blocks are staged through shared memory with the 512-thread block primitives above; the
// breakdown (status) is reported with the global pivot index, later kernels return at once.
// -----------------------------------------------------------------------------------------
__global__ void k_chol_prep(const double* __restrict__ W, int ldw, int b, double* __restrict__ work,
                            double* __restrict__ U, int ldu, double* __restrict__ Z, int ldz, const int* status) {
  if (failed(status)) return;
  const int64_t bb = (int64_t)b * b;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < bb; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % b), j = (int)(e / b);
    work[e] = (i <= j) ? W[i + (int64_t)j * ldw] : 0.0;
    U[i + (int64_t)j * ldu] = 0.0;
    Z[i + (int64_t)j * ldz] = 0.0;
  }
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_diag(const double* __restrict__ work, int b, int J,
                                                          double* __restrict__ U, int ldu, double* __restrict__ Z,
                                                          int ldz, int* status, int pass, int panel, int stage) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_urow[CHB];
  if (failed(status)) return;
  const int tid = threadIdx.x;
  double* D = smem;
  double* Di = smem + CHB * CHLD;
  blk_load(D, work + (int64_t)J * CHB * b + J * CHB, b, tid);
  if (!blk_chol_inv(D, Di, s_urow, status, pass, panel, stage, J * CHB, tid)) return;
  blk_store(U + (int64_t)J * CHB * ldu + J * CHB, ldu, D, tid);
  blk_store(Z + (int64_t)J * CHB * ldz + J * CHB, ldz, Di, tid);
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_row(const double* __restrict__ work, int b, int J,
                                                         double* __restrict__ U, int ldu, const double* __restrict__ Z,
                                                         int ldz, const int* status) {
  extern __shared__ __align__(16) double smem[];
  if (failed(status)) return;
  const int tid = threadIdx.x, K = J + 1 + blockIdx.x;
  double* Di = smem;
  double* T = smem + CHB * CHLD;
  double* PK = smem + 2 * CHB * CHLD;
  blk_load(Di, Z + (int64_t)J * CHB * ldz + J * CHB, ldz, tid);
  blk_load(T, work + (int64_t)K * CHB * b + J * CHB, b, tid);
  blk_mm<true, false>(Di, T, PK, tid);
  blk_store(U + (int64_t)K * CHB * ldu + J * CHB, ldu, PK, tid);
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_trail(double* __restrict__ work, int b, int J,
                                                           const double* __restrict__ U, int ldu, const int* status) {
  extern __shared__ __align__(16) double smem[];
  if (failed(status)) return;
  const int tid = threadIdx.x, r = (b / CHB) - J - 1;
  // blockIdx.x -> (K, L), J < K <= L < nb, enumerated column by column of the trailing triangle
  int t = blockIdx.x, L2 = 0;
  while (t >= L2 + 1) { t -= L2 + 1; ++L2; }
  const int K = J + 1 + t, L = J + 1 + L2;
  (void)r;
  double* A = smem;
  double* B = smem + CHB * CHLD;
  double* T = smem + 2 * CHB * CHLD;
  double* wkl = work + (int64_t)L * CHB * b + K * CHB;
  blk_load(A, U + (int64_t)K * CHB * ldu + J * CHB, ldu, tid);
  blk_load(B, U + (int64_t)L * CHB * ldu + J * CHB, ldu, tid);
  blk_load(T, wkl, b, tid);
  blk_mm<true, true>(A, B, T, tid);
  blk_store(wkl, b, T, tid);
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_tri_inv_step(const double* __restrict__ U, int ldu,
                                                             double* __restrict__ Z, int ldz, int d, const int* status) {
  extern __shared__ __align__(16) double smem[];
  if (failed(status)) return;
  const int tid = threadIdx.x, I = blockIdx.x, J = I + d;
  double* D = smem;
  double* Di = smem + CHB * CHLD;
  double* P = smem + 2 * CHB * CHLD;
  double* T = smem + 3 * CHB * CHLD;
  for (int e = tid; e < CHB * CHB; e += CHOL_NT) P[(e & 63) + (e >> 6) * CHLD] = 0.0;
  __syncthreads();
  for (int K = I + 1; K <= J; ++K) {
    blk_load(D, U + (int64_t)K * CHB * ldu + I * CHB, ldu, tid);   // U_IK
    blk_load(Di, Z + (int64_t)J * CHB * ldz + K * CHB, ldz, tid);  // Z_KJ
    blk_mm<false, true>(D, Di, P, tid);                             // P -= U_IK Z_KJ
  }
  blk_load(D, Z + (int64_t)I * CHB * ldz + I * CHB, ldz, tid);     // Z_II
  blk_mm<false, false>(D, P, T, tid);                              // Z_IJ = Z_II (-S)
  blk_store(Z + (int64_t)J * CHB * ldz + I * CHB, ldz, T, tid);
}

// -----------------------------------------------------------------------------------------
// R assembly (Alg. 3 l.3 P:185; Alg. 6 l.5/l.8 P:295/P:298; R-8).  Negligible work.
// -----------------------------------------------------------------------------------------
// C (n x n) = A * B for upper-triangular A, B: C[i,j] = sum_{t=i..j} A[i,t] B[t,j]; zeros below.
__global__ void k_trimul(const double* __restrict__ A, int lda, const double* __restrict__ B, int ldb,
                         double* __restrict__ C, int ldc, int n, const int* status) {
  if (failed(status)) return;
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    double s = 0.0;
    for (int t = i; t <= j; ++t) s = fma(A[i + (int64_t)t * lda], B[t + (int64_t)j * ldb], s);
    C[i + (int64_t)j * ldc] = s;
  }
}

// C (p x q) += A (p x q') * B with B upper triangular (q x q): R_{1:j-1,j} += C U1 (R-8)
__global__ void k_gemm_acc_tri(const double* __restrict__ A, int lda, const double* __restrict__ B, int ldb,
                               double* __restrict__ C, int ldc, int p, int q, const int* status) {
  if (failed(status)) return;
  const int64_t pq = (int64_t)p * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pq; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % p), j = (int)(e / p);
    double s = 0.0;
    for (int t = 0; t <= j; ++t) s = fma(A[i + (int64_t)t * lda], B[t + (int64_t)j * ldb], s);
    C[i + (int64_t)j * ldc] += s;
  }
}

// D <- alpha S (alpha = +-1 in use: exact)
// Shift of the Gram matrix for shifted CholeskyQR (Alg. 4 l.2-3):
// W_ii += s with s = (sqrt(m) u) * ||A||_F^2, where ||A||_F^2 = sum_j W_jj is taken from the
// diagonal of the allreduced Gram (the row sums of the squares of A's entries) in index
// order -- identical on every rank.  sqrt_m_u = sqrt(m_global) * 2^-53 from the host.
__global__ void k_shift(double* W, int ldw, int n, double sqrt_m_u, const int* status) {
  if (failed(status)) return;
  __shared__ double s_shift;
  if (threadIdx.x == 0) {
    double fro2 = 0.0;
    for (int j = 0; j < n; ++j) fro2 += W[j + (int64_t)j * ldw];
    s_shift = sqrt_m_u * fro2;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) W[j + (int64_t)j * ldw] += s_shift;
}

__global__ void k_copy2d(const double* __restrict__ S, int64_t lds, double* __restrict__ D, int64_t ldd, int rows,
                         int cols, double alpha, const int* status) {
  if (failed(status)) return;
  const int64_t nn = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    D[i + j * ldd] = alpha * S[i + j * lds];
  }
}

__global__ void k_zero2d(double* __restrict__ D, int64_t ldd, int rows, int cols) {
  const int64_t nn = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    D[i + j * ldd] = 0.0;
  }
}

// ---- runtime-adaptive repetition (TSQR_MCQR2GS_ADAPTIVE, DESIGN R-23) ----
// status[0] codes: 0 running, 5 breakdown, 7 = "this panel's repetition is skipped": every
// kernel checks failed(status) and returns at once, the fused cross-GPU sum keeps its barrier.
constexpr int STATUS_SKIP = 7;

// After the first CholeskyQR of a panel: E = max(u nu(U1)^2 nu(Z)^2, u nu(R_{1:j,j}) nu(Z)),
// nu(M) = ||M||_F / sqrt(b) (Z = U1^{-1}, R_{1:j-1,j} = Rcol rows 0..c0-1).  E <= tau: mark the
// skip (status[0] = 7, status[9] += 1) and prepare the R-8 bookkeeping to be exact no-ops:
// U2 = I (R_jj = U2 U1 = U1 bitwise) and C = 0 (R_{1:j-1,j} += C U1 adds zeros).  One CTA,
// fixed-order reduction: the decision is bitwise identical on every rank.
__global__ void __launch_bounds__(256) k_adapt_decide(const double* __restrict__ U1, int ldu,
                                                      const double* __restrict__ Z, int ldz,
                                                      const double* __restrict__ Rcol, int ldr, int c0, int b,
                                                      double tau, double* __restrict__ U2, int ldu2,
                                                      double* __restrict__ C, int ldc, int* status) {
  if (failed(status)) return;
  __shared__ double red[3][256];
  __shared__ int skip;
  double su = 0.0, sz = 0.0, sy = 0.0;
  for (int e = threadIdx.x; e < b * b; e += 256) {
    const int i = e % b, j = e / b;
    if (i <= j) {
      const double u = U1[i + (int64_t)j * ldu], z = Z[i + (int64_t)j * ldz];
      su = fma(u, u, su);
      sz = fma(z, z, sz);
    }
  }
  for (int e = threadIdx.x; e < c0 * b; e += 256) {
    const double y = Rcol[(e % c0) + (int64_t)(e / c0) * ldr];
    sy = fma(y, y, sy);
  }
  red[0][threadIdx.x] = su; red[1][threadIdx.x] = sz; red[2][threadIdx.x] = sy;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h)
      for (int v = 0; v < 3; ++v) red[v][threadIdx.x] += red[v][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double u = 1.1102230246251565e-16, bb = (double)b;
    const double nu_u2 = red[0][0] / bb, nu_z2 = red[1][0] / bb, nu_r2 = (red[2][0] + red[0][0]) / bb;
    const double own = u * nu_u2 * nu_z2, across = u * sqrt(nu_r2) * sqrt(nu_z2);
    skip = (own > across ? own : across) <= tau;
    if (skip) { status[9] += 1; status[0] = STATUS_SKIP; }
  }
  __syncthreads();
  if (skip) {
    for (int e = threadIdx.x; e < b * b; e += 256) U2[(e % b) + (int64_t)(e / b) * ldu2] = (e % b == e / b) ? 1.0 : 0.0;
    for (int e = threadIdx.x; e < c0 * b; e += 256) C[(e % c0) + (int64_t)(e / c0) * ldc] = 0.0;
  }
}

// end of a skippable section: a skip mark becomes "running" again (a breakdown stays)
__global__ void k_adapt_resume(int* status) {
  if (threadIdx.x == 0 && status[0] == STATUS_SKIP) status[0] = 0;
}

}  // namespace tsqr
