// kernels.cuh -- sm_100a FP64 kernels for the CholeskyQR2 / CQR2GS / mCQR2GS hot path of
// arXiv 2405.04237.  Every contraction runs on the FP64 tensor pipe through
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; the B200 has no tcgen05 kind for f64), with
// operand tiles staged in padded shared memory by cp.async (LDGSTS).
//
// Layout: every matrix is FP64 column-major, element (r, c) at X[r + c*ld], 64-bit offsets.
// Row tiles of TR rows are the unit of streaming; a staged tile is stored column by column
// with leading dimension LDT = TR + 4 doubles (== 4 mod 16), which makes every DMMA
// fragment load below bank-conflict free (2 wavefronts per 32 doubles).
//
// DMMA m8n8k4 fragments (lane = 4*gid + tig):  A (8x4, row): a = A[gid][tig]
//                                              B (4x8, col): b = B[tig][gid]
//                                              C (8x8):      c0,c1 = C[gid][2*tig + {0,1}]
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tsqr {

constexpr int NT = 256;  // threads per CTA (8 warps) for the streaming kernels
constexpr int NWARPS = NT / 32;

// ---------------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Stage a (TR rows) x (NCOLS columns) tile of column-major G (leading dimension ld) starting at
// (row0, col0) into shared memory sm[c*LDT + r].  Rows >= m and columns >= colmax are
// zero-filled (cp.async with a short source size), so ragged tails contribute nothing.
// V16: 16-byte copies (requires ld even and G 16-byte aligned), else 8-byte copies.
template <int TR, int LDT, bool V16, int NCOLS = 64>
__device__ __forceinline__ void stage_tile(double* sm, const double* __restrict__ G, int64_t ld,
                                           int64_t row0, int64_t m, int col0, int colmax) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 2
  for (int c = warp; c < NCOLS; c += NWARPS) {
    const int gc = col0 + c;
    const bool cv = gc < colmax;
    const double* src = G + (int64_t)(cv ? gc : 0) * ld;
    if (V16) {
#pragma unroll
      for (int rp = lane; rp < TR / 2; rp += 32) {
        const int64_t r = row0 + 2 * rp;
        int64_t rem = cv ? (m - r) : 0;
        int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
        cp_async16(sm + c * LDT + 2 * rp, bytes ? (const void*)(src + r) : (const void*)G, bytes);
      }
    } else {
#pragma unroll
      for (int rr = lane; rr < TR; rr += 32) {
        const int64_t r = row0 + rr;
        int bytes = (cv && r < m) ? 8 : 0;
        cp_async8(sm + c * LDT + rr, bytes ? (const void*)(src + r) : (const void*)G, bytes);
      }
    }
  }
}

__device__ __forceinline__ bool failed(const int* status) {
  return status != nullptr && *((volatile const int*)status) != 0;
}

// ---------------------------------------------------------------------------------------
// k_atb: split-row partial products  PART[s] (p x q, ld p) = sum over rows of split s of
// L^T Rm  (Gram W = X^T X when gram != 0; projections Y = Q^T A and C = Q^T V otherwise).
// grid.x enumerates 64x64 output tiles (upper tiles only for a Gram), grid.y = S splits.
// Diagonal Gram tiles use the "DIAG" schedule: every warp owns 1/8 of the rows of a staged
// tile and all 36 upper 8x8 blocks (A and B fragments of X^T X coincide, so one fragment
// load feeds up to 8 DMMAs).  Other tiles use "FULL": 2 k-halves x (2x2 warp tiles of
// 32x32).  Partial results of the warps are combined in a fixed order -> deterministic.
// ---------------------------------------------------------------------------------------
constexpr int ATB_TR = 64;
constexpr int ATB_LDT = ATB_TR + 4;
constexpr int ATB_STAGES = 3;
constexpr int ATB_TILE_DBL = 64 * ATB_LDT;
constexpr size_t ATB_SMEM = sizeof(double) * (size_t)ATB_STAGES * 2 * ATB_TILE_DBL;

struct AtbArgs {
  const double* L;
  int64_t ldl;
  const double* R;
  int64_t ldr;
  int64_t m;
  int p, q;
  int gram;           // 1: L == R, upper tiles only, lower part of diagonal tiles not written
  int ntp, ntq;       // output tiles along p and q
  int64_t tiles_per_split;  // row tiles per split
  double* part;       // [S][p*q]
  const int* status;
};

template <bool V16>
__global__ void __launch_bounds__(NT, 1) k_atb(AtbArgs a) {
  extern __shared__ __align__(16) double smem[];
  if (failed(a.status)) return;
  // decode the output tile
  int ti, tj;
  {
    int bx = blockIdx.x;
    if (a.gram) {
      int t = 0;
      ti = 0; tj = 0;
      for (int j = 0; j < a.ntq; ++j)
        for (int i = 0; i <= j; ++i) {
          if (t == bx) { ti = i; tj = j; }
          ++t;
        }
    } else {
      ti = bx % a.ntp;
      tj = bx / a.ntp;
    }
  }
  const bool diag = a.gram && ti == tj;
  const int s = blockIdx.y;
  const int64_t ntr = (a.m + ATB_TR - 1) / ATB_TR;
  const int64_t t0 = (int64_t)s * a.tiles_per_split;
  int64_t t1 = t0 + a.tiles_per_split;
  if (t1 > ntr) t1 = ntr;
  const int nt = (int)(t1 > t0 ? t1 - t0 : 0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int pc0 = ti * 64, qc0 = tj * 64;
  double* bufL = smem;                                   // [STAGES][TILE]
  double* bufR = smem + ATB_STAGES * ATB_TILE_DBL;       // [STAGES][TILE]

  auto issue = [&](int it) {
    if (it < nt) {
      const int st = it % ATB_STAGES;
      const int64_t row0 = (t0 + it) * ATB_TR;
      stage_tile<ATB_TR, ATB_LDT, V16>(bufL + st * ATB_TILE_DBL, a.L, a.ldl, row0, a.m, pc0, a.p);
      if (!diag) stage_tile<ATB_TR, ATB_LDT, V16>(bufR + st * ATB_TILE_DBL, a.R, a.ldr, row0, a.m, qc0, a.q);
    }
    cp_async_commit();
  };

  // accumulators: DIAG uses acc[0..71] (36 upper blocks), FULL uses acc[0..31] (4x4 blocks)
  double acc[72];
#pragma unroll
  for (int i = 0; i < 72; ++i) acc[i] = 0.0;

#pragma unroll
  for (int it = 0; it < ATB_STAGES - 1; ++it) issue(it);

  for (int it = 0; it < nt; ++it) {
    cp_async_wait<ATB_STAGES - 2>();
    __syncthreads();
    issue(it + ATB_STAGES - 1);
    const double* sL = bufL + (it % ATB_STAGES) * ATB_TILE_DBL;
    if (diag) {
      // rows [warp*8, warp*8+8) of the tile = 2 k-steps
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int k0 = warp * 8 + ks * 4 + tig;
        double f[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) f[c] = sL[(c * 8 + gid) * ATB_LDT + k0];
        int t = 0;
#pragma unroll
        for (int bj = 0; bj < 8; ++bj)
#pragma unroll
          for (int bi = 0; bi <= bj; ++bi) {
            dmma(acc[2 * t], acc[2 * t + 1], f[bi], f[bj]);
            ++t;
          }
      }
    } else {
      const double* sR = bufR + (it % ATB_STAGES) * ATB_TILE_DBL;
      const int h = warp >> 2, wi = (warp >> 1) & 1, wj = warp & 1;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const int k0 = h * 32 + ks * 4 + tig;
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) fa[i] = sL[(wi * 32 + i * 8 + gid) * ATB_LDT + k0];
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[j] = sR[(wj * 32 + j * 8 + gid) * ATB_LDT + k0];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[2 * (i * 4 + j)], acc[2 * (i * 4 + j) + 1], fa[i], fb[j]);
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // combine the warps' partials in a fixed order, write the 64x64 tile of PART[s]
  double* red = smem;  // reuse the staging buffers
  double* outp = a.part + (int64_t)s * a.p * a.q;
  if (diag) {
    // red[w][t*64 + lane*2 + {0,1}] for the 36 upper blocks t of warp w (147 KB)
#pragma unroll
    for (int t = 0; t < 36; ++t) {
      red[warp * 2304 + t * 64 + lane * 2] = acc[2 * t];
      red[warp * 2304 + t * 64 + lane * 2 + 1] = acc[2 * t + 1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2304; e += NT) {
      const double v = ((red[e] + red[2304 + e]) + (red[2 * 2304 + e] + red[3 * 2304 + e])) +
                       ((red[4 * 2304 + e] + red[5 * 2304 + e]) + (red[6 * 2304 + e] + red[7 * 2304 + e]));
      int t = e >> 6;
      const int ln = (e & 63) >> 1, hi = e & 1;
      int bj = 0;
      while (t > bj) { t -= bj + 1; ++bj; }
      const int bi = t;
      const int r = bi * 8 + (ln >> 2), c = bj * 8 + 2 * (ln & 3) + hi;
      const int gr = pc0 + r, gc = qc0 + c;
      if (gr < a.p && gc < a.q && r <= c) outp[gr + (int64_t)gc * a.p] = v;
    }
  } else {
    const int h = warp >> 2, wi = (warp >> 1) & 1, wj = warp & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = wi * 32 + i * 8 + gid, c = wj * 32 + j * 8 + 2 * tig;
        red[h * 4096 + c * 64 + r] = acc[2 * (i * 4 + j)];
        red[h * 4096 + (c + 1) * 64 + r] = acc[2 * (i * 4 + j) + 1];
      }
    __syncthreads();
    for (int e = threadIdx.x; e < 4096; e += NT) {
      const int r = e & 63, c = e >> 6;
      const double v = red[e] + red[4096 + e];
      const int gr = pc0 + r, gc = qc0 + c;
      if (gr < a.p && gc < a.q && (!a.gram || gr <= gc)) outp[gr + (int64_t)gc * a.p] = v;
    }
  }
}

// ---------------------------------------------------------------------------------------
// k_reduce: OUT[i,j] = sum_s PART[s][i,j] in a fixed order (8 interleaved running sums,
// then a pairwise combination).  gram: only i <= j is read; OUT[j,i] = OUT[i,j] (bitwise
// symmetric, R-11).
// ---------------------------------------------------------------------------------------
__global__ void k_reduce(const double* __restrict__ part, int S, int p, int q, double* __restrict__ out,
                         int ldo, int gram, const int* status) {
  if (failed(status)) return;
  const int64_t pq = (int64_t)p * q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < pq; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % p), j = (int)(e / p);
    if (gram && i > j) continue;
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int t = 0;
    for (; t + 8 <= S; t += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) s[u] += part[(int64_t)(t + u) * pq + e];
    }
    for (int u = 0; t + u < S; ++u) s[u] += part[(int64_t)(t + u) * pq + e];
    const double v = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    out[i + (int64_t)j * ldo] = v;
    if (gram && i != j) out[j + (int64_t)i * ldo] = v;
  }
}

// ---------------------------------------------------------------------------------------
// k_trmm: X (m x b) <- X * Z in place, Z upper triangular (b x b): the panel
// orthogonalisation Q = A R^{-1} with the explicit inverse (R-4).  Row tiles are
// independent.  Warp w owns a set of row blocks and a balanced set of column-block
// pairs (cb, NB-1-cb) so the triangular work is even across warps.
// B (= b) is a template parameter: 16, 32, 64 (Z staged in smem) or 128, 256 (Z read
// from global / L2).
// ---------------------------------------------------------------------------------------
template <int B>
struct TrmmCfg {
  static constexpr int NB = B / 8;                                  // 8-col blocks
  static constexpr int PAIRS = NB / 2;                              // balanced pairs
  static constexpr int PAIRS_PER_WARP = PAIRS >= NWARPS ? PAIRS / NWARPS : 1;
  static constexpr int ROW_GROUPS = PAIRS >= NWARPS ? 1 : NWARPS / PAIRS;
  static constexpr int TR = (B <= 64) ? 64 : 32;
  static constexpr int RB = TR / 8 / ROW_GROUPS;                    // 8-row blocks per warp
  static constexpr int LDT = TR + 4;
  static constexpr bool ZSMEM = (B <= 64);
  static constexpr int LDZ = B + 4;                                 // smem Z leading dim
  static constexpr int STAGES = (B <= 64) ? 3 : 2;
  static constexpr int TILE_DBL = B * LDT;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)STAGES * TILE_DBL + (ZSMEM ? (size_t)B * LDZ : 0));
};

template <int B, bool V16>
__global__ void __launch_bounds__(NT, 1) k_trmm(double* __restrict__ X, int64_t ldx, int64_t m,
                                                const double* __restrict__ Z, int ldz, const int* status) {
  using C = TrmmCfg<B>;
  extern __shared__ __align__(16) double smem[];
  if (failed(status)) return;
  double* sZ = smem + C::STAGES * C::TILE_DBL;
  if (C::ZSMEM) {
    // sZ[col*LDZ + k] = Z[k, col]
    for (int e = threadIdx.x; e < B * B; e += NT) {
      const int k = e % B, col = e / B;
      sZ[col * C::LDZ + k] = Z[k + (int64_t)col * ldz];
    }
  }
  const int64_t ntr = (m + C::TR - 1) / C::TR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int rg = warp % C::ROW_GROUPS;            // row group
  const int pw = warp / C::ROW_GROUPS;            // pair group
  constexpr int CBW = 2 * C::PAIRS_PER_WARP;      // column blocks per warp
  int cbs[CBW];
#pragma unroll
  for (int u = 0; u < C::PAIRS_PER_WARP; ++u) {
    const int pr = pw * C::PAIRS_PER_WARP + u;
    cbs[2 * u] = pr;
    cbs[2 * u + 1] = C::NB - 1 - pr;
  }
  int maxcb = 0;
#pragma unroll
  for (int u = 0; u < CBW; ++u) maxcb = cbs[u] > maxcb ? cbs[u] : maxcb;

  // row tiles handled by this CTA: blockIdx.x, +gridDim.x, ...
  const int64_t first = blockIdx.x;
  const int64_t stride = gridDim.x;
  const int nmine = (int)(first < ntr ? (ntr - 1 - first) / stride + 1 : 0);

  auto issue = [&](int it) {
    if (it < nmine) {
      const int st = it % C::STAGES;
      const int64_t row0 = (first + (int64_t)it * stride) * C::TR;
      for (int c0 = 0; c0 < B; c0 += 64)
        stage_tile<C::TR, C::LDT, V16, (B < 64 ? B : 64)>(smem + st * C::TILE_DBL + c0 * C::LDT, X, ldx, row0, m, c0, B);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int it = 0; it < C::STAGES - 1; ++it) issue(it);

  for (int it = 0; it < nmine; ++it) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    issue(it + C::STAGES - 1);
    const double* sX = smem + (it % C::STAGES) * C::TILE_DBL;
    const int64_t row0 = (first + (int64_t)it * stride) * C::TR;
    double acc[C::RB][CBW][2];
#pragma unroll
    for (int i = 0; i < C::RB; ++i)
#pragma unroll
      for (int u = 0; u < CBW; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;
    const int kend = (maxcb + 1) * 8;
    for (int k0 = 0; k0 < kend; k0 += 4) {
      double fa[C::RB];
#pragma unroll
      for (int i = 0; i < C::RB; ++i) fa[i] = sX[(k0 + tig) * C::LDT + (rg * C::RB + i) * 8 + gid];
#pragma unroll
      for (int u = 0; u < CBW; ++u) {
        if (k0 < (cbs[u] + 1) * 8) {
          const int col = cbs[u] * 8 + gid;
          const double fb = C::ZSMEM ? sZ[col * C::LDZ + k0 + tig] : __ldg(Z + (k0 + tig) + (int64_t)col * ldz);
#pragma unroll
          for (int i = 0; i < C::RB; ++i) dmma(acc[i][u][0], acc[i][u][1], fa[i], fb);
        }
      }
    }
    // write X_new directly to global (each lane: 2 columns x 1 row per block)
#pragma unroll
    for (int i = 0; i < C::RB; ++i) {
      const int64_t r = row0 + (rg * C::RB + i) * 8 + gid;
      if (r < m) {
#pragma unroll
        for (int u = 0; u < CBW; ++u) {
          const int c = cbs[u] * 8 + 2 * tig;
          X[r + (int64_t)c * ldx] = acc[i][u][0];
          X[r + (int64_t)(c + 1) * ldx] = acc[i][u][1];
        }
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------
// k_update: X (m x q) -= L (m x p) * S (p x q), in place, row-tile local.
// Per row tile (64 rows) and per 64-column chunk of X: accumulators start from X (loaded
// straight into C fragments), then loop over 64-wide k-chunks of L / S staged in shared
// memory by cp.async (3 stages).  Warp tile 32 rows x 16 cols (2 x 4 warp grid).
// When p <= 64 the L tile is staged once per row tile and reused for every X chunk.
// ---------------------------------------------------------------------------------------
constexpr int UPD_TR = 64;
constexpr int UPD_LDT = UPD_TR + 4;
constexpr int UPD_STAGES = 3;
constexpr int UPD_LTILE = 64 * UPD_LDT;   // L chunk: 64 k-columns x 64 rows
constexpr int UPD_STILE = 64 * UPD_LDT;   // S chunk: 64 x-columns x 64 k
constexpr size_t UPD_SMEM = sizeof(double) * (size_t)UPD_STAGES * (UPD_LTILE + UPD_STILE);

struct UpdArgs {
  double* X;
  int64_t ldx;
  const double* L;
  int64_t ldl;
  const double* S;
  int64_t lds;
  int64_t m;
  int p, q;
  const int* status;
};

template <bool V16>
__global__ void __launch_bounds__(NT, 1) k_update(UpdArgs a) {
  extern __shared__ __align__(16) double smem[];
  if (failed(a.status)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 2;      // 0..1 : rows [wr*32, +32)
  const int wc = warp & 3;       // 0..3 : cols [wc*16, +16)
  const int64_t ntr = (a.m + UPD_TR - 1) / UPD_TR;
  const int nxc = (a.q + 63) / 64, nkc = (a.p + 63) / 64;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int nmine = (int)(first < ntr ? (ntr - 1 - first) / stride + 1 : 0);
  const int steps = nmine * nxc * nkc;
  const bool lonce = (nkc == 1);
  double* bufL = smem;
  double* bufS = smem + UPD_STAGES * UPD_LTILE;

  // steps (row tile tl, x chunk xc, k chunk kc); S chunks live in a ring indexed by step, L
  // chunks in a ring indexed by step, or -- when p <= 64 and the L tile is staged once per
  // row tile -- by row tile (at most STAGES tiles are in flight, so slots never collide).
  auto decode = [&](int st, int& tl, int64_t& row0, int& xc, int& kc) {
    tl = st / (nxc * nkc);
    const int rem = st % (nxc * nkc);
    xc = rem / nkc;
    kc = rem % nkc;
    row0 = (first + (int64_t)tl * stride) * UPD_TR;
  };
  auto issue = [&](int st) {
    if (st < steps) {
      int64_t row0; int tl, xc, kc;
      decode(st, tl, row0, xc, kc);
      const int sb = st % UPD_STAGES;
      if (!lonce || xc == 0)
        stage_tile<UPD_TR, UPD_LDT, V16>(bufL + (lonce ? tl % UPD_STAGES : sb) * UPD_LTILE, a.L, a.ldl, row0,
                                         a.m, kc * 64, a.p);
      // S chunk: columns xc*64.. of S (q direction), rows kc*64.. (k direction); S is p x q col-major
      stage_tile<64, UPD_LDT, V16>(bufS + sb * UPD_STILE, a.S, a.lds, (int64_t)kc * 64, a.p, xc * 64, a.q);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int st = 0; st < UPD_STAGES - 1; ++st) issue(st);

  double acc[4][2][2];
  for (int st = 0; st < steps; ++st) {
    int64_t row0; int tl, xc, kc;
    decode(st, tl, row0, xc, kc);
    if (kc == 0) {
      // accumulators <- X chunk
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t r = row0 + wr * 32 + i * 8 + gid;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int c = xc * 64 + wc * 16 + j * 8 + 2 * tig;
          const bool ok = r < a.m;
          acc[i][j][0] = (ok && c < a.q) ? a.X[r + (int64_t)c * a.ldx] : 0.0;
          acc[i][j][1] = (ok && c + 1 < a.q) ? a.X[r + (int64_t)(c + 1) * a.ldx] : 0.0;
        }
      }
    }
    cp_async_wait<UPD_STAGES - 2>();
    __syncthreads();
    issue(st + UPD_STAGES - 1);
    const int sb = st % UPD_STAGES;
    const double* sL = bufL + (lonce ? tl % UPD_STAGES : sb) * UPD_LTILE;
    const double* sS = bufS + sb * UPD_STILE;
    const int kmax = min(64, a.p - kc * 64);
#pragma unroll 4
    for (int k0 = 0; k0 < kmax; k0 += 4) {
      double fa[4], fb[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = -sL[(k0 + tig) * UPD_LDT + wr * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 2; ++j) fb[j] = sS[(wc * 16 + j * 8 + gid) * UPD_LDT + k0 + tig];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    if (kc == nkc - 1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t r = row0 + wr * 32 + i * 8 + gid;
        if (r < a.m) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = xc * 64 + wc * 16 + j * 8 + 2 * tig;
            if (c < a.q) a.X[r + (int64_t)c * a.ldx] = acc[i][j][0];
            if (c + 1 < a.q) a.X[r + (int64_t)(c + 1) * a.ldx] = acc[i][j][1];
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------
// k_chol_inv: single CTA.  W (b x b, upper triangle read) = U^T U, unpivoted, right-looking
// (R-5), then Z = U^{-1} by back substitution of U Z = I column by column (R-4).
// Breakdown iff a pivot d is not > 0 or not finite: status <- {5, pass, panel, stage,
// pivot, -, value(double)}; U and Z are then left undefined.
// Work matrix in shared memory for b <= 128, else in the global scratch `work`.
// ---------------------------------------------------------------------------------------
constexpr int CHOL_NT = 512;

__global__ void __launch_bounds__(CHOL_NT, 1) k_chol_inv(const double* __restrict__ W, int ldw, int b,
                                                        double* __restrict__ U, int ldu, double* __restrict__ Z,
                                                        int ldz, int* status, int pass, int panel, int stage,
                                                        double* work, int use_smem) {
  extern __shared__ __align__(16) double smem[];
  __shared__ int s_fail;
  if (failed(status)) return;
  double* S = use_smem ? smem : work;  // S[i + j*b], upper triangle used
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += CHOL_NT) {
    const int i = e % b, j = e / b;
    S[e] = (i <= j) ? W[i + (int64_t)j * ldw] : 0.0;
  }
  if (tid == 0) s_fail = 0;
  __syncthreads();
  for (int k = 0; k < b; ++k) {
    if (tid == 0) {
      const double d = S[k + k * b];
      if (!(d > 0.0) || !isfinite(d)) {
        s_fail = 1;
        status[1] = pass; status[2] = panel; status[3] = stage; status[4] = k;
        *reinterpret_cast<double*>(status + 6) = d;
        __threadfence();
        status[0] = 5;
      } else {
        S[k + k * b] = sqrt(d);
      }
    }
    __syncthreads();
    if (s_fail) return;
    const double ukk = S[k + k * b];
    for (int j = k + 1 + tid; j < b; j += CHOL_NT) S[k + j * b] = S[k + j * b] / ukk;
    __syncthreads();
    // trailing update S[i][j] -= U[k][i] U[k][j], k < i <= j
    const int nrem = b - k - 1;
    const int npairs = nrem * nrem;
    for (int e = tid; e < npairs; e += CHOL_NT) {
      const int i = k + 1 + e % nrem, j = k + 1 + e / nrem;
      if (i <= j) S[i + j * b] = fma(-S[k + i * b], S[k + j * b], S[i + j * b]);
    }
    __syncthreads();
  }
  // U out (exact zeros below the diagonal)
  for (int e = tid; e < b * b; e += CHOL_NT) {
    const int i = e % b, j = e / b;
    U[i + (int64_t)j * ldu] = (i <= j) ? S[e] : 0.0;
  }
  // Z = U^{-1}: column j solves U z = e_j; one warp per column, lanes split the dot products
  const int warp = tid >> 5, lane = tid & 31;
  for (int j = warp; j < b; j += CHOL_NT / 32) {
    double* zc = Z + (int64_t)j * ldz;
    for (int i = lane; i < b; i += 32)
      if (i > j) zc[i] = 0.0;
    for (int i = j; i >= 0; --i) {
      double s = 0.0;
      for (int t = i + 1 + lane; t <= j; t += 32) s = fma(S[i + t * b], zc[t], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) zc[i] = (((i == j) ? 1.0 : 0.0) - s) / S[i + i * b];
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------------------
// Small R-assembly kernels (n <= 4096; negligible work).
// ---------------------------------------------------------------------------------------
// C (n x n) = A * B for upper-triangular A, B: C[i,j] = sum_{t=i..j} A[i,t] B[t,j]; zeros below.
__global__ void k_trimul(const double* __restrict__ A, int lda, const double* __restrict__ B, int ldb,
                         double* __restrict__ C, int ldc, int n, const int* status) {
  if (failed(status)) return;
  const int64_t nn = (int64_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    double s = 0.0;
    for (int t = i; t <= j; ++t) s = fma(A[i + (int64_t)t * lda], B[t + (int64_t)j * ldb], s);
    C[i + (int64_t)j * ldc] = s;  // i > j: empty sum -> exact zero
  }
}

// C (p x q) += A (p x r) * B (r x q), B upper triangular (r == q): R_{1:j-1,j} += C U1 (R-8)
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

// D (rows x cols, ldd) = S (rows x cols, lds)
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
