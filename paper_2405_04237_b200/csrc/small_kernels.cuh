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
__global__ void k_reduce(const double* __restrict__ part, int Sfull, int Sdiag, int p, int q, int ldp,
                         int64_t pstride, double* __restrict__ out, int ldo, int gram, const int* status) {
  if (failed(status)) return;
  const int64_t pq = (int64_t)p * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pq; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % p), j = (int)(e / p);
    if (gram && i > j) continue;
    const int S = (gram && (i >> 6) == (j >> 6)) ? Sdiag : Sfull;  // splits of this element's tile
    const double* src = part + i + (int64_t)j * ldp;
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int t = 0; t < S; t += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t + u < S) s[u] += src[(int64_t)(t + u) * pstride];
    }
    const double v = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    out[i + (int64_t)j * ldo] = v;
    if (gram && i != j) out[j + (int64_t)i * ldo] = v;
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

// shared-memory bytes of k_chol_inv for block size b (S and Z with padded leading dimension
// b + 1 so that row- and column-wise accesses are bank-conflict free)
__host__ __device__ constexpr size_t chol_smem_bytes(int b) {
  return b <= 64 ? sizeof(double) * 2 * (size_t)b * (b + 1) : (b <= 128 ? sizeof(double) * (size_t)b * (b + 1) : 0);
}

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_inv(const double* __restrict__ W, int ldw, int b,
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
  for (int e = tid; e < b * b; e += CHOL_NT) {
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
    for (int j = k + tid; j < b; j += CHOL_NT) s_urow[j] = (j == k) ? ukk : S[k + j * lds] / ukk;
    __syncthreads();
    for (int j0 = 0; j0 < b; j0 += 64) {
      const int j = j0 + jj;
      if (j < b && j >= k) {
        if (ii0 == 0) S[k + j * lds] = s_urow[j];
        const double uj = s_urow[j];
        for (int i = k + 1 + ((ii0 - (k + 1)) & 7); i <= j; i += 8) S[i + j * lds] = fma(-s_urow[i], uj, S[i + j * lds]);
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += CHOL_NT) {
    const int i = e % b, j = e / b;
    U[i + (int64_t)j * ldu] = (i <= j) ? S[i + j * lds] : 0.0;
    Zw[i + (int64_t)j * ldzw] = 0.0;
  }
  __syncthreads();
  // Z = U^{-1} (R-4): rows from the bottom, Z_ij = (delta_ij - sum_{t=i+1..j} U_it Z_tj) / U_ii for
  // all j >= i in parallel; column j handled by 8 lanes of one warp (the t-range split 8 ways)
  const int sub = tid & 7, jg = tid >> 3;
  for (int i = b - 1; i >= 0; --i) {
    for (int jb = 0; jb < b; jb += CHOL_NT / 8) {  // uniform trip count: shuffles stay converged
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
    for (int e = tid; e < b * b; e += CHOL_NT) {
      const int i = e % b, j = e / b;
      Z[i + (int64_t)j * ldz] = Zw[i + j * ldzw];
    }
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

__global__ void k_copy2d(const double* __restrict__ S, int64_t lds, double* __restrict__ D, int64_t ldd, int rows,
                         int cols, const int* status) {
  if (failed(status)) return;
  const int64_t nn = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    D[i + j * ldd] = S[i + j * lds];
  }
}

__global__ void k_zero2d(double* __restrict__ D, int64_t ldd, int rows, int cols) {
  const int64_t nn = (int64_t)rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    D[i + j * ldd] = 0.0;
  }
}

}  // namespace tsqr
