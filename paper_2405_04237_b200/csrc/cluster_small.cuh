// cluster_small.cuh -- the whole factorisation of a SMALL problem in one kernel launch
// (BASELINE configs[0]: 4096 x 64, b = 16; SURVEY §8(a) a1-a12 on one GPU).
//
// At this size the streaming path is latency-bound: ~70 small kernels (Gram, reduce,
// Cholesky, TRMM, projection, update, R assembly) and the launch / drain gap between them
// dominate, not FLOPs or bytes (2 MiB of A).  Here one thread-block CLUSTER of CS CTAs
// (16, non-portable, or 8) keeps the whole m x n matrix in distributed shared memory: CTA r
// holds rows [r*mr, (r+1)*mr) (zero-padded to mr) of every column, column-major with a
// padded leading dimension ldx == 4 (mod 16) (conflict-free DMMA fragment loads).  A is read
// from HBM once and Q written once; every step of the paper's algorithms runs in place:
//   * Gram / projection (Alg. 2 l.2, Alg. 7 l.7, Alg. 8 l.3, l.7): each CTA forms its local
//     L^T R with DMMA.8x8x4 (warps split output tiles and, for few tiles, row ranges, summed in
//     a fixed order), then the cluster "allreduce" (the P = 1 case of the paper's Allreduce,
//     P:154) is a reduce-scatter + all-gather over DSMEM: CTA r sums elements
//     [r*c, (r+1)*c) of all CS partials in RANK ORDER and stores the sums into every CTA's
//     destination -- deterministic, bitwise identical in every CTA;
//   * Cholesky of the b x b Gram (R-5) redundantly in every CTA (one warp, lane j owns
//     columns j, j+32): no broadcast is needed, and a breakdown is seen by every CTA at the
//     same pivot (same Gram bits) and reported once in the status word;
//   * Q = A U^{-1} (Alg. 2 l.5) as a row-wise forward substitution (the trsm form of P:122;
//     one thread per row, x_j <- x_j / u_jj via the reciprocal, then x_l -= x_j u_jl);
//   * updates A -= Q Y (Alg. 7 l.9, Alg. 8 l.5, l.7) with DMMA on 8 x 8 tiles in place;
//   * R assembly (R-8) by CTA 0 into global R.
// Cluster barriers: two per reduction (partials complete; sums distributed), none elsewhere.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"

namespace tsqr {

namespace cgx = cooperative_groups;

constexpr int CL_NT = 256;  // threads per CTA
constexpr int CL_NW = CL_NT / 32;

struct ClusterArgs {
  double* A;       // m x n, column-major (Q on exit)
  int64_t lda;
  double* R;       // n x n
  int ldr;
  double* R1;      // n x n global scratch (CQR2GS pass 1 / sCQR3)
  double* R2;      // n x n global scratch (CQR2GS pass 2)
  int* status;     // status word (breakdown record, as k_chol_inv)
  int64_t m;       // rows
  int n;
  int algo;        // tsqr_algo
  int mr;          // rows per CTA (multiple of 32)
  int ldx;         // shared leading dimension (mr + 4)
  int pq;          // capacity of the reduction buffers (doubles)
  double shift_scale;  // sqrt(m_global) * u (sCQR, Alg. 4 l.2)
};

// Phase profiling (development builds only: nvcc -DTSQR_CL_PROF): thread 0 of CTA 0 adds
// clock64 deltas per phase and prints them at the end of the kernel.
#ifdef TSQR_CL_PROF
#include <cstdio>
struct ClProf {
  long long last = 0, acc[10] = {0};
  __device__ void mark(int ph) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      const long long t = clock64();
      if (last) acc[ph] += t - last;
      last = t;
    }
  }
};
#define CLP(ph) prof.mark(ph)
#else
struct ClProf {
  __device__ void mark(int) {}
};
#define CLP(ph)
#endif

__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Shared memory per CTA (doubles).  `red` is the destination of every cluster sum: the
// projection blocks Y (B x N_j, ld B) / C (jB x B, ld jB), which are dead once their update and
// R bookkeeping are done, and the Gram W (B x B), which the Cholesky factors IN PLACE into U.
// Ua keeps the first CQR's U1 while the second CQR runs (Alg. 3, Alg. 8 l.6-8); Ub keeps the
// shifted CQR's factor through sCQR3's CQR2 (Alg. 5) and exists only for that algorithm.
template <int B>
struct ClusterSmem {
  double* X;      // ldx x n
  double* part;   // pq: this CTA's local partial of the current reduction
  double* red;    // pq: reduced block (Y, C, or W -> U in place)
  double* Ua;     // B x B (ld B)
  double* Ub;     // B x B (sCQR3 only)
  double* dinv;   // B: reciprocals of the current factor's diagonal (+ B: Cholesky row broadcast)
  double* tmp;    // 2 x 256 (B == 16 only): row-range partials of the 16 x 16 Gram
  int* flag;      // [0]: breakdown seen
};

// ---- local contraction: part (p x q, ld p) = X[:, l0:l0+p]^T X[:, r0:r0+q] over this CTA's rows.
// 8 x 8 output tiles (DMMA.8x8x4: A fragment = L^T rows, B fragment = R columns, both read
// straight from the column-major X).  A warp owns tiles t = g, g + G, ...; up to 4 of them are
// accumulated together (independent DMMA chains), each as two chains over even / odd
// 4-row k-steps, combined in a fixed order at the end.  Exactly the warp's tiles are issued
// (no predicated-off DMMA: it would still occupy the FP64 pipe).
template <int NTL>
__device__ __forceinline__ void atb_tiles(const double* __restrict__ X, int ldx, int rlo, int rows, int l0, int r0,
                                          int tp, int t0, int G, double* __restrict__ out, int p) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  int oa[NTL], ob[NTL];
#pragma unroll
  for (int u = 0; u < NTL; ++u) {
    const int t = t0 + u * G, ti = t % tp, tj = t / tp;
    oa[u] = (l0 + ti * 8 + gid) * ldx + tig + rlo;
    ob[u] = (r0 + tj * 8 + gid) * ldx + tig + rlo;
  }
  double c[NTL][4];
#pragma unroll
  for (int u = 0; u < NTL; ++u) c[u][0] = c[u][1] = c[u][2] = c[u][3] = 0.0;
  for (int k0 = 0; k0 < rows; k0 += 8) {
#pragma unroll
    for (int u = 0; u < NTL; ++u) {
      dmma(c[u][0], c[u][1], X[oa[u] + k0], X[ob[u] + k0]);
      dmma(c[u][2], c[u][3], X[oa[u] + k0 + 4], X[ob[u] + k0 + 4]);
    }
  }
#pragma unroll
  for (int u = 0; u < NTL; ++u) {
    const int t = t0 + u * G, ti = t % tp, tj = t / tp;
    const int i = ti * 8 + gid, j = tj * 8 + 2 * tig;
    out[i + j * p] = c[u][0] + c[u][2];
    out[i + (j + 1) * p] = c[u][1] + c[u][3];
  }
}

template <int B>
__device__ void cl_atb_local(const ClusterSmem<B>& s, int ldx, int mr, int l0, int p, int r0, int q) {
  const int warp = threadIdx.x >> 5;
  const int tp = p >> 3, T8 = tp * (q >> 3);
  const int G = T8 >= CL_NW ? CL_NW : T8;  // tile groups (T8 is a multiple of 4)
  const int RS = CL_NW / G;                // row ranges per tile group (1 or 2)
  const int g = warp % G, rp = warp / G;
  const int rows = mr / RS, rlo = rp * rows;  // rows: a multiple of 16
  double* out = RS == 1 ? s.part : s.tmp + rp * (p * q);
  int nt = (T8 - g + G - 1) / G;  // this warp's tiles
  for (int t0 = g; nt > 0; t0 += 4 * G, nt -= 4) {
    switch (nt < 4 ? nt : 4) {
      case 1: atb_tiles<1>(s.X, ldx, rlo, rows, l0, r0, tp, t0, G, out, p); break;
      case 2: atb_tiles<2>(s.X, ldx, rlo, rows, l0, r0, tp, t0, G, out, p); break;
      case 3: atb_tiles<3>(s.X, ldx, rlo, rows, l0, r0, tp, t0, G, out, p); break;
      default: atb_tiles<4>(s.X, ldx, rlo, rows, l0, r0, tp, t0, G, out, p); break;
    }
  }
  if (RS > 1) {
    __syncthreads();
    for (int e = threadIdx.x; e < p * q; e += CL_NT) s.part[e] = s.tmp[e] + s.tmp[p * q + e];
  }
}

// ---- cluster sum: dst (count doubles, same offset in every CTA) = sum over CTAs of part.
// Reduce-scatter + all-gather over DSMEM: CTA `me` owns elements [me*chunk, (me+1)*chunk),
// loads them from all CS partials at once (independent remote loads in flight), adds them in
// rank order and stores the sum into every CTA's dst.
template <int CS>
__device__ __forceinline__ void cl_reduce_cs(cgx::cluster_group& cl, double* part, double* dst, int count) {
  const int me = (int)cl.block_rank();
  const int chunk = (count + CS - 1) / CS;
  const int lo = me * chunk, hi = min(count, lo + chunk);
  for (int e = lo + (int)threadIdx.x; e < hi; e += CL_NT) {
    double v[CS];
#pragma unroll
    for (int r = 0; r < CS; ++r) v[r] = cl.map_shared_rank(part, r)[e];
    double sum = v[0];
#pragma unroll
    for (int r = 1; r < CS; ++r) sum += v[r];  // rank order
#pragma unroll
    for (int r = 0; r < CS; ++r) cl.map_shared_rank(dst, r)[e] = sum;
  }
}

__device__ void cl_reduce(cgx::cluster_group& cl, double* part, double* dst, int count) {
  cl_sync();  // every CTA's partial is complete
  if (cl.num_blocks() == 16) cl_reduce_cs<16>(cl, part, dst, count);
  else cl_reduce_cs<8>(cl, part, dst, count);
  cl_sync();  // every CTA holds the sums; the partial buffers may be rewritten
}

__device__ __forceinline__ void cl_breakdown(int* status, int pass, int panel, int stage, int k, double d) {
  status[1] = pass; status[2] = panel; status[3] = stage; status[4] = k;
  *reinterpret_cast<double*>(status + 6) = d;
  __threadfence();
  status[0] = 5;
}

// B <= 32: one warp, lane j holds column j of W / U in registers; row k of U is broadcast
// through shared memory (measured 4.7k cycles for b = 16 vs 13k with per-element shuffles,
// tools/microbench/chol_variants.cu).  Per pivot one rsqrt on the critical path (B200 latencies:
// DFMA 23, rsqrt ~40, sqrt ~65, division ~46 cycles): r = rsqrt(d), u_kk = d r (within an ulp
// of sqrt(d)), the row is scaled by r, then the rank-1 trailing update.  No early exit: the loop
// unrolls fully so x stays in registers; the first failed pivot is reported after the loop.
template <int B>
__device__ bool cl_chol_reg(const ClusterSmem<B>& s, int* status, int pass, int panel, int stage, bool rank0) {
  double* Uo = s.red;
  double* row = s.dinv + B;  // B doubles of broadcast row (allocated after dinv)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double x[B];
#pragma unroll
    for (int i = 0; i < B; ++i) x[i] = (lane < B && i <= lane) ? Uo[i + lane * B] : 0.0;
    int bad = -1;
    double dbad = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (lane == k) row[k] = x[k];
      __syncwarp();
      const double d = row[k];
      if (bad < 0 && (!(d > 0.0) || !isfinite(d))) { bad = k; dbad = d; }
      const double r = rsqrt(d), ukk = d * r;
      const double ukj = lane == k ? ukk : x[k] * r;
      if (lane >= k) x[k] = ukj;
      if (lane == k) s.dinv[k] = r;
      if (lane > k && lane < B) row[lane] = ukj;
      __syncwarp();
#pragma unroll
      for (int i = k + 1; i < B; ++i)
        if (lane >= i) x[i] = fma(-row[i], ukj, x[i]);
      __syncwarp();
    }
    if (bad >= 0 && rank0 && lane == 0) cl_breakdown(status, pass, panel, stage, bad, dbad);
    if (lane < B)
#pragma unroll
      for (int i = 0; i < B; ++i) Uo[i + lane * B] = i <= lane ? x[i] : 0.0;
    if (lane == 0) s.flag[0] = bad < 0 ? 0 : 1;
  }
  __syncthreads();
  return s.flag[0] == 0;
}

template <int B>
__device__ bool cl_chol(const ClusterSmem<B>& s, int* status, int pass, int panel, int stage, bool rank0) {
  if constexpr (B <= 32) return cl_chol_reg<B>(s, status, pass, panel, stage, rank0);
  double* Uo = s.red;
  for (int e = threadIdx.x; e < B * B; e += CL_NT)
    if (e % B > e / B) Uo[e] = 0.0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    bool ok = true;
    for (int k = 0; k < B; ++k) {
      const double d = Uo[k + k * B];
      if (!(d > 0.0) || !isfinite(d)) {
        if (rank0 && lane == 0) cl_breakdown(status, pass, panel, stage, k, d);
        ok = false;
        break;
      }
      const double ukk = sqrt(d), r = rsqrt(d);
      __syncwarp();
#pragma unroll
      for (int h = 0; h < (B + 31) / 32; ++h) {
        const int j = lane + 32 * h;
        if (j < B && j > k) Uo[k + j * B] *= r;
      }
      if (lane == 0) { Uo[k + k * B] = ukk; s.dinv[k] = r; }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < (B + 31) / 32; ++h) {
        const int j = lane + 32 * h;
        if (j < B && j > k) {
          const double ukj = Uo[k + j * B];
          for (int i = k + 1; i <= j; ++i) Uo[i + j * B] = fma(-Uo[k + i * B], ukj, Uo[i + j * B]);
        }
      }
      __syncwarp();
    }
    if (lane == 0) s.flag[0] = ok ? 0 : 1;
  }
  __syncthreads();
  return s.flag[0] == 0;
}

// ---- X[:, c0:c0+B] <- X[:, c0:c0+B] U^{-1} (row-wise forward substitution, the trsm of P:122)
template <int B>
__device__ void cl_trsm(const ClusterSmem<B>& s, int ldx, int mr, int c0, const double* U) {
  for (int i = threadIdx.x; i < mr; i += CL_NT) {
    double x[B];
    double* xr = s.X + i + (int64_t)c0 * ldx;
#pragma unroll
    for (int j = 0; j < B; ++j) x[j] = xr[(int64_t)j * ldx];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      x[j] *= s.dinv[j];
#pragma unroll
      for (int l = j + 1; l < B; ++l) x[l] = fma(-x[j], U[j + l * B], x[l]);
    }
#pragma unroll
    for (int j = 0; j < B; ++j) xr[(int64_t)j * ldx] = x[j];
  }
  __syncthreads();
}

// ---- X[:, r0:r0+q] -= X[:, l0:l0+p] S   (S = s.red, p x q, ld p), DMMA on 8 x 8 tiles in place;
// a warp advances NTL of its tiles together (independent accumulator chains).
template <int NTL>
__device__ __forceinline__ void upd_tiles(double* __restrict__ X, int ldx, const double* __restrict__ S, int tr,
                                          int t0, int r0, int l0, int p) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  double* xo[NTL];
  const double* xa[NTL];
  const double* sb[NTL];
  double c[NTL][2];
#pragma unroll
  for (int u = 0; u < NTL; ++u) {
    const int t = t0 + u * CL_NW, ri = t % tr, cj = t / tr;
    xo[u] = X + ri * 8 + gid + (int64_t)(r0 + cj * 8 + 2 * tig) * ldx;
    xa[u] = X + ri * 8 + gid + (int64_t)(l0 + tig) * ldx;
    sb[u] = S + tig + (cj * 8 + gid) * p;
    c[u][0] = xo[u][0];
    c[u][1] = xo[u][ldx];
  }
  for (int k0 = 0; k0 < p; k0 += 4)
#pragma unroll
    for (int u = 0; u < NTL; ++u) dmma(c[u][0], c[u][1], xa[u][(int64_t)k0 * ldx], -sb[u][k0]);
#pragma unroll
  for (int u = 0; u < NTL; ++u) {
    xo[u][0] = c[u][0];
    xo[u][ldx] = c[u][1];
  }
}

template <int B>
__device__ void cl_update(const ClusterSmem<B>& s, int ldx, int mr, int r0, int q, int l0, int p) {
  const int warp = threadIdx.x >> 5;
  const int tr = mr >> 3, T = tr * (q >> 3);
  int nt = (T - warp + CL_NW - 1) / CL_NW;
  int t0 = warp;
  for (; nt >= 4; nt -= 4, t0 += 4 * CL_NW) upd_tiles<4>(s.X, ldx, s.red, tr, t0, r0, l0, p);
  for (; nt > 0; --nt, t0 += CL_NW) upd_tiles<1>(s.X, ldx, s.red, tr, t0, r0, l0, p);
  __syncthreads();
}

// ---- R assembly helpers (CTA 0 only, global R): D[i,j] (+)= sum_{t} A[i,t] Bm[t,j], upper Bm
// trimul: D (w x w) = Ua Ub, both upper triangular (ld lda_/ldb_), lower part written as 0
__device__ void cl_trimul(const double* Ua, int lda_, const double* Ub, int ldb_, double* D, int ldd, int w) {
  for (int e = threadIdx.x; e < w * w; e += CL_NT) {
    const int i = e % w, j = e / w;
    double v = 0.0;
    for (int t = i; t <= j; ++t) v = fma(Ua[i + (int64_t)t * lda_], Ub[t + (int64_t)j * ldb_], v);
    D[i + (int64_t)j * ldd] = i <= j ? v : 0.0;
  }
}
// D (p x w) += C (p x w, ld ldc) U (w x w upper, ld w)
__device__ void cl_gemm_acc_tri(const double* C, int ldc, const double* U, int w, double* D, int ldd, int p) {
  for (int e = threadIdx.x; e < p * w; e += CL_NT) {
    const int i = e % p, j = e / p;
    double v = 0.0;
    for (int t = 0; t <= j; ++t) v = fma(C[i + t * ldc], U[t + j * w], v);
    D[i + (int64_t)j * ldd] += v;
  }
}
__device__ void cl_copy(const double* S, int lds, double* D, int ldd, int rows, int cols) {
  for (int e = threadIdx.x; e < rows * cols; e += CL_NT) {
    const int i = e % rows, j = e / rows;
    D[i + (int64_t)j * ldd] = S[i + j * lds];
  }
}

template <int B>
struct ClusterRun {
  const ClusterArgs& a;
  ClusterSmem<B> s;
  cgx::cluster_group cl;
  bool rank0;
  ClProf prof;

  // Gram of X[:, c0:c0+B], cluster sum -> W (s.red); optional sCQR shift; Cholesky -> U in
  // s.red; X_c <- X_c U^{-1}.  keep: copy U to `keep` (ld B) as well.
  // B = 16 (cfg1) inlines the CholeskyQR at every call site (measured 0.125 vs 0.149 ms/step
  // outlined); wider B are outlined: fully inlined, the unrolled trsm / Cholesky bodies of every
  // call site made the library take ~14 minutes to compile.
  __device__ bool cqr(int c0, int pass, int panel, int stage, double* keep = nullptr, bool shift = false) {
    if constexpr (B == 16) return cqr_body(c0, pass, panel, stage, keep, shift);
    else return cqr_outlined(c0, pass, panel, stage, keep, shift);
  }
  __device__ __noinline__ bool cqr_outlined(int c0, int pass, int panel, int stage, double* keep, bool shift) {
    return cqr_body(c0, pass, panel, stage, keep, shift);
  }
  __device__ __forceinline__ bool cqr_body(int c0, int pass, int panel, int stage, double* keep, bool shift) {
    cl_atb_local<B>(s, a.ldx, a.mr, c0, B, c0, B);
    CLP(1);
    cl_reduce(cl, s.part, s.red, B * B);
    CLP(2);
    if (shift) {  // Alg. 4 l.2-3: W += s I, s = sqrt(m) u ||A||_F^2, ||A||_F^2 = trace(W)
      double tr = 0.0;
      for (int j = 0; j < B; ++j) tr += s.red[j + j * B];
      const double sh = a.shift_scale * tr;
      __syncthreads();
      if (threadIdx.x < B) s.red[threadIdx.x * (B + 1)] += sh;
      __syncthreads();
    }
    if (!cl_chol<B>(s, a.status, pass, panel, stage, rank0)) return false;
    CLP(3);
    if (keep)
      for (int e = threadIdx.x; e < B * B; e += CL_NT) keep[e] = s.red[e];
    cl_trsm<B>(s, a.ldx, a.mr, c0, s.red);  // ends with __syncthreads
    CLP(4);
    return true;
  }
  // red (p x q, ld p) = cluster sum of X[:, l0:+p]^T X[:, r0:+q]
  __device__ void proj(int l0, int p, int r0, int q) {
    CLP(7);
    cl_atb_local<B>(s, a.ldx, a.mr, l0, p, r0, q);
    CLP(5);
    cl_reduce(cl, s.part, s.red, p * q);
    CLP(2);
  }

  // one CQRGS pass (Alg. 7) with its R into Rp (global, ld ldrp)
  __device__ bool cqrgs_pass(double* Rp, int ldrp, int pass) {
    const int n = a.n, k = n / B;
    for (int j = 0; j < k; ++j) {
      if (!cqr(j * B, pass, j + 1, 1)) return false;                         // l.2-6
      if (rank0) cl_copy(s.red, B, Rp + j * B + (int64_t)j * B * ldrp, ldrp, B, B);
      const int nt = n - (j + 1) * B;
      if (nt > 0) {
        proj(j * B, B, (j + 1) * B, nt);                                      // l.7-8
        if (rank0) cl_copy(s.red, B, Rp + j * B + (int64_t)(j + 1) * B * ldrp, ldrp, B, nt);  // l.10
        cl_update<B>(s, a.ldx, a.mr, (j + 1) * B, nt, j * B, B);              // l.9
      }
    }
    return true;
  }

  __device__ bool run() {
    const int n = a.n, k = n / B;
    double* R = a.R;
    const int ldr = a.ldr;
    switch (a.algo) {
      case 3:  // TSQR_CQR (Alg. 2), B == n
        if (!cqr(0, 1, 1, 1)) return false;
        if (rank0) cl_copy(s.red, B, R, ldr, B, B);
        return true;
      case 0:  // TSQR_CQR2 (Alg. 3), B == n: R = U2 U1
        if (!cqr(0, 1, 1, 1, s.Ua) || !cqr(0, 1, 1, 2)) return false;
        if (rank0) cl_trimul(s.red, B, s.Ua, B, R, ldr, B);
        return true;
      case 4:  // TSQR_CQRGS (Alg. 7)
        return cqrgs_pass(R, ldr, 1);
      case 1:  // TSQR_CQR2GS: two CQRGS passes, R = R2 R1
        if (k == 1) {  // b == n: CholeskyQR2
          if (!cqr(0, 1, 1, 1, s.Ua) || !cqr(0, 1, 1, 2)) return false;
          if (rank0) cl_trimul(s.red, B, s.Ua, B, R, ldr, B);
          return true;
        }
        if (!cqrgs_pass(a.R1, n, 1) || !cqrgs_pass(a.R2, n, 2)) return false;
        __syncthreads();
        if (rank0) cl_trimul(a.R2, n, a.R1, n, R, ldr, n);
        return true;
      case 2: {  // TSQR_MCQR2GS (Alg. 8)
        if (!cqr(0, 1, 1, 1, s.Ua) || !cqr(0, 1, 1, 2)) return false;        // l.1
        if (rank0) cl_trimul(s.red, B, s.Ua, B, R, ldr, B);
        for (int j = 1; j < k; ++j) {
          const int jb = j * B, Nj = n - jb;
          proj(jb - B, B, jb, Nj);                                            // l.3: Y
          if (rank0) cl_copy(s.red, B, R + (jb - B) + (int64_t)jb * ldr, ldr, B, Nj);  // R_{j-1,j:k} = Y
          CLP(7);
          cl_update<B>(s, a.ldx, a.mr, jb, Nj, jb - B, B);                    // l.4-5
          CLP(6);
          if (!cqr(jb, 1, j + 1, 1, s.Ua)) return false;                      // l.6: U1 -> Ua
          proj(0, jb, jb, B);                                                 // l.7: C
          if (rank0) cl_gemm_acc_tri(s.red, jb, s.Ua, B, R + (int64_t)jb * ldr, ldr, jb);  // R_{1:j-1,j} += C U1 (R-8)
          CLP(7);
          cl_update<B>(s, a.ldx, a.mr, jb, B, 0, jb);
          CLP(6);
          if (!cqr(jb, 1, j + 1, 2)) return false;                            // l.8: U2 in red
          if (rank0) cl_trimul(s.red, B, s.Ua, B, R + jb + (int64_t)jb * ldr, ldr, B);  // R_jj = U2 U1
        }
        return true;
      }
      case 6:  // TSQR_SCQR (Alg. 4), B == n
        if (!cqr(0, 1, 1, 1, nullptr, true)) return false;
        if (rank0) cl_copy(s.red, B, R, ldr, B, B);
        return true;
      case 5:  // TSQR_SCQR3 (Alg. 5): sCQR (-> Ub), then CQR2 (U1 -> Ua, U2); R = (U2 U1) Ub
        if (!cqr(0, 1, 1, 1, s.Ub, true) || !cqr(0, 1, 1, 2, s.Ua) || !cqr(0, 1, 1, 3)) return false;
        if (rank0) {
          cl_trimul(s.red, B, s.Ua, B, a.R2, n, B);
          __syncthreads();
          cl_trimul(a.R2, n, s.Ub, B, R, ldr, B);
        }
        return true;
    }
    return false;
  }
};

template <int B>
__global__ void __launch_bounds__(CL_NT, 1) k_cluster_factor(ClusterArgs a) {
  extern __shared__ __align__(16) double csm[];
  cgx::cluster_group cl = cgx::this_cluster();
  const int me = (int)cl.block_rank();
  ClusterRun<B> run{a, {}, cl, me == 0};
  run.prof.mark(9);
  ClusterSmem<B>& s = run.s;
  double* p = csm;
  s.X = p; p += (size_t)a.ldx * a.n;
  s.part = p; p += a.pq;
  s.red = p; p += a.pq;
  s.Ua = p; p += B * B;
  s.Ub = p; if (a.algo == 5) p += B * B;
  s.dinv = p; p += B <= 32 ? 2 * B : B;  // dinv[B] (+ the register Cholesky's broadcast row[B])
  s.tmp = p; if (B == 16) p += 512;
  s.flag = reinterpret_cast<int*>(p);
  // load this CTA's block rows: one bulk (TMA) copy per column when the rows are 16-byte aligned
  // (one thread issues them, an mbarrier counts the bytes), else 8-byte cp.async; rows beyond m
  // are zero padding
  __shared__ __align__(8) uint64_t lbar;
  const int64_t row0 = (int64_t)me * a.mr;
  const int64_t left = a.m - row0;
  const int rows = left <= 0 ? 0 : (left < a.mr ? (int)left : a.mr);
  const bool bulk = rows > 0 && rows % 2 == 0 && a.lda % 2 == 0 && ((reinterpret_cast<uintptr_t>(a.A) & 15u) == 0);
  for (int c = 0; c < a.n; ++c)
    for (int i = rows + threadIdx.x; i < a.mr; i += CL_NT) s.X[i + (int64_t)c * a.ldx] = 0.0;
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&lbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      mbar_arrive_expect_tx(&lbar, (uint32_t)(sizeof(double) * rows * a.n));
      for (int c = 0; c < a.n; ++c)
        bulk_g2s(s.X + (int64_t)c * a.ldx, a.A + row0 + (int64_t)c * a.lda, (uint32_t)(sizeof(double) * rows), &lbar);
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    mbar_wait(&lbar, 0);
  } else {
    for (int c = 0; c < a.n; ++c) {
      const double* src = a.A + row0 + (int64_t)c * a.lda;
      double* dst = s.X + (int64_t)c * a.ldx;
      for (int i = threadIdx.x; i < rows; i += CL_NT) cp_async8(dst + i, src + i, 8);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }
  if (me == 0 && threadIdx.x < 16) a.status[threadIdx.x] = 0;  // this factorisation's status word
  if (me == 0) {  // R (and the CQR2GS / sCQR3 scratch) start at zero: the lower triangles stay zero
    for (int e = threadIdx.x; e < a.n * a.n; e += CL_NT) {
      const int i = e % a.n, j = e / a.n;
      a.R[i + (int64_t)j * a.ldr] = 0.0;
      a.R1[e] = 0.0;
      a.R2[e] = 0.0;
    }
  }
  __syncthreads();
  run.prof.mark(0);
  run.run();
  __syncthreads();
  run.prof.mark(7);
  // store Q (also after a breakdown: the status word tells the caller): bulk copies from shared
  // memory (after a proxy fence orders every thread's generic writes of X before them)
  if (bulk) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c = 0; c < a.n; ++c)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(a.A + row0 + (int64_t)c * a.lda),
                     "r"(smem_u32(s.X + (int64_t)c * a.ldx)), "r"((uint32_t)(sizeof(double) * rows))
                     : "memory");
      bulk_commit();
      bulk_wait0();
    }
  } else {
    for (int i = threadIdx.x; i < rows; i += CL_NT) {
      double* dst = a.A + row0 + i;
      const double* src = s.X + i;
#pragma unroll 8
      for (int c = 0; c < a.n; ++c) dst[(int64_t)c * a.lda] = src[(int64_t)c * a.ldx];
    }
  }
  cl_sync();  // no CTA exits while another may still address its shared memory
  run.prof.mark(8);
#ifdef TSQR_CL_PROF
  if (threadIdx.x == 0 && me == 0)
    printf("CLPROF load %lld gram %lld reduce %lld chol %lld trsm %lld proj %lld update %lld r0 %lld store %lld\n",
           run.prof.acc[0], run.prof.acc[1], run.prof.acc[2], run.prof.acc[3], run.prof.acc[4], run.prof.acc[5],
           run.prof.acc[6], run.prof.acc[7], run.prof.acc[8]);
#endif
}

// shared-memory bytes of k_cluster_factor<B> (layout of ClusterSmem)
inline size_t cluster_smem_bytes(int B, int ldx, int n, int pq, int algo) {
  return sizeof(double) * ((size_t)ldx * n + 2 * (size_t)pq + (size_t)B * B * (algo == 5 ? 2 : 1) + (B <= 32 ? 2 * B : B) +
                           (B == 16 ? 512 : 0)) + 16;
}

}  // namespace tsqr
