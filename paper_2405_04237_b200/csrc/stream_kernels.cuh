// stream_kernels.cuh -- the O(m) streaming kernels of the hot path:
// split-row projections / Gram (k_proj), in-place trailing and re-orthogonalisation
// updates (k_update) and in-place panel orthogonalisation (k_trmm).
//
// All three are persistent, warp-specialised CTAs: one producer warp streams tiles of the
// tall operands into a ring of shared-memory stages with 2-D TMA tensor copies -- ONE
// cp.async.bulk.tensor per 64-column tile, box = (TR + 4) rows x 64 columns, so the tile
// lands column by column with the padded leading dimension LDT = TR + 4 == 4 (mod 16) that
// makes every DMMA fragment load bank-conflict free; the 4 extra rows are never read, rows
// past m and columns past the operand are zero-filled by the TMA unit.  Each stage has a
// "full" mbarrier (arrive.expect_tx + complete_tx) and an "empty" mbarrier released by the
// eight consumer warps, which run DMMA.8x8x4 contractions.  No CTA-wide barrier sits on the
// streaming path.  Odd leading dimensions (no 16-byte TMA strides) fall back to a cp.async
// producer with the same pipeline.
#pragma once
#include "common.cuh"

namespace tsqr {

constexpr int TR = 64;                // rows per streamed tile
constexpr int LDT = TR + 4;           // padded leading dimension (== 4 mod 16) = TMA box rows
constexpr int TILE = 64 * LDT;        // doubles in one 64-column tile
constexpr uint32_t TILE_BYTES = TILE * 8;

// smem base rounded up to `al` bytes (TMA destinations; 1024 for 128-byte swizzled boxes);
// callers request +al bytes.  Pointer arithmetic on the __shared__ array keeps the address
// space, so accesses stay LDS/STS.
__device__ __forceinline__ double* aligned_smem(double* p, uint32_t al = 128) {
  return p + (((al - (smem_u32(p) & (al - 1))) & (al - 1)) >> 3);
}

// =========================================================================================
// k_proj: PART[s] (p x q, ld p) = sum over the rows of split s of L^T Rm.
//   gram = 1: L == Rm, upper 64x64 output tiles only; diagonal tiles use the DIAG schedule
//   (diag_half: the A and B fragments of X^T X coincide, 8 fragment loads feed 18 DMMAs).
//   Other tiles: FULL schedule, 2 k-halves x 2x2 warp tiles of 32x32.
// grid = (#output tiles, S splits); the warps' partials are combined in a fixed order.
// (Alg. 2 l.2 P:152, Alg. 7 l.2/l.7 P:344/Alg. 8 l.3/l.7 P:464/P:468)
// =========================================================================================
constexpr int PROJ_NS = 3;
constexpr size_t PROJ_SMEM = sizeof(double) * (size_t)PROJ_NS * 2 * TILE + 2 * PROJ_NS * sizeof(uint64_t) + 128;

struct ProjArgs {
  CUtensorMap mapL;  // L: rows m, cols p   (TMA path)
  CUtensorMap mapR;  // Rm: rows m, cols q
  const double* L;
  int64_t ldl;
  const double* R;
  int64_t ldr;
  int64_t m;
  int p, q;
  int gram;
  int ntp, ntq;
  int64_t tiles_per_split;       // full tiles
  int S_full, S_diag;            // row splits of full / diagonal (Gram) tiles
  int64_t tiles_per_split_diag;
  double* part;  // [S][p*q]
  const int* status;
};

// DIAG schedule of a diagonal Gram tile: warp group H (= warp / 4) owns the upper 8x8 blocks
// t in [18H, 18H+18) (column-major block order), warp wq = warp % 4 owns rows [16wq, 16wq+16)
// of every staged tile (4 k-steps): 36 accumulators per lane, 8 fragment loads per 18 DMMAs.
template <int H>
__device__ __forceinline__ void diag_half(const double* sL, int wq, int gid, int tig, double (&acc)[36]) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k0 = wq * 16 + ks * 4 + tig;
    double f[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) f[c] = sL[(c * 8 + gid) * LDT + k0];
    int t = 0;
#pragma unroll
    for (int bj = 0; bj < 8; ++bj)
#pragma unroll
      for (int bi = 0; bi <= bj; ++bi) {
        if (t >= 18 * H && t < 18 * H + 18) dmma(acc[2 * (t - 18 * H)], acc[2 * (t - 18 * H) + 1], f[bi], f[bj]);
        ++t;
      }
  }
}

template <bool TMA>
__global__ void __launch_bounds__(NTHR, 1) k_proj(const __grid_constant__ ProjArgs a) {
  extern __shared__ __align__(128) double smem_raw[];
  if (failed(a.status)) return;
  double* smem = aligned_smem(smem_raw);
  double* bufL = smem;
  double* bufR = smem + PROJ_NS * TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * PROJ_NS * TILE);
  uint64_t* empty = full + PROJ_NS;

  int ti, tj;
  if (a.gram) {
    int bx = blockIdx.x, j = 0;
    while (bx > j) { bx -= j + 1; ++j; }
    ti = bx; tj = j;
  } else {
    ti = blockIdx.x % a.ntp;
    tj = blockIdx.x / a.ntp;
  }
  const bool diag = a.gram && ti == tj;
  const int s = blockIdx.y;
  if (s >= (diag ? a.S_diag : a.S_full)) return;  // this tile type has fewer splits
  const int64_t tps = diag ? a.tiles_per_split_diag : a.tiles_per_split;
  const int64_t ntr = (a.m + TR - 1) / TR;
  const int64_t t0 = (int64_t)s * tps;
  const int64_t t1 = min(ntr, t0 + tps);
  const int nt = (int)(t1 > t0 ? t1 - t0 : 0);
  const int pc0 = ti * 64, qc0 = tj * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PROJ_NS; ++i) {
      mbar_init(&full[i], TMA ? 1 : 32);
      mbar_init(&empty[i], NCW);
    }
    if (TMA) {
      tma_prefetch_map(&a.mapL);
      if (!diag) tma_prefetch_map(&a.mapR);
    }
  }
  __syncthreads();

  if (warp == PRODUCER) {
    for (int it = 0; it < nt; ++it) {
      const int st = it % PROJ_NS, use = it / PROJ_NS;
      if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
      const int64_t row0 = (t0 + it) * TR;
      if (TMA) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], diag ? TILE_BYTES : 2 * TILE_BYTES);
          tma_load_2d(bufL + st * TILE, &a.mapL, (int)row0, pc0, &full[st]);
          if (!diag) tma_load_2d(bufR + st * TILE, &a.mapR, (int)row0, qc0, &full[st]);
        }
      } else {
        produce_tile<TR, LDT, false, 64>(bufL + st * TILE, a.L, a.ldl, row0, a.m, pc0, a.p, lane);
        if (!diag) produce_tile<TR, LDT, false, 64>(bufR + st * TILE, a.R, a.ldr, row0, a.m, qc0, a.q, lane);
        cp_async_arrive(&full[st]);
      }
    }
    return;
  }

  const int gid = lane >> 2, tig = lane & 3;
  double acc[36];
#pragma unroll
  for (int i = 0; i < 36; ++i) acc[i] = 0.0;

  for (int it = 0; it < nt; ++it) {
    const int st = it % PROJ_NS;
    mbar_wait(&full[st], (it / PROJ_NS) & 1);
    const double* sL = bufL + st * TILE;
    if (diag) {
      if (warp < 4) diag_half<0>(sL, warp & 3, gid, tig, acc);
      else diag_half<1>(sL, warp & 3, gid, tig, acc);
    } else {
      const double* sR = bufR + st * TILE;
      const int h = warp >> 2, wi = (warp >> 1) & 1, wj = warp & 1;
#pragma unroll 2
      for (int ks = 0; ks < 8; ++ks) {
        const int k0 = h * 32 + ks * 4 + tig;
        double fa[4], fb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) fa[i] = sL[(wi * 32 + i * 8 + gid) * LDT + k0];
#pragma unroll
        for (int j = 0; j < 4; ++j) fb[j] = sR[(wj * 32 + j * 8 + gid) * LDT + k0];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[2 * (i * 4 + j)], acc[2 * (i * 4 + j) + 1], fa[i], fb[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

  // every staged tile has been consumed -> the ring can be reused for the warp partials
  consumer_sync();
  double* red = smem;
  double* outp = a.part + (int64_t)s * a.p * a.q;
  if (diag) {
#pragma unroll
    for (int u = 0; u < 18; ++u) {
      red[warp * 1152 + u * 64 + lane * 2] = acc[2 * u];
      red[warp * 1152 + u * 64 + lane * 2 + 1] = acc[2 * u + 1];
    }
    consumer_sync();
    for (int e = threadIdx.x; e < 2304; e += NCW * 32) {
      const int t = e >> 6, H = t / 18, u = t - 18 * H, off = u * 64 + (e & 63);
      const double* base = red + H * 4 * 1152 + off;
      const double v = (base[0] + base[1152]) + (base[2 * 1152] + base[3 * 1152]);
      int bi, bj;
      upper_block(t, bi, bj);
      const int ln = (e & 63) >> 1, hi = e & 1;
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
    consumer_sync();
    for (int e = threadIdx.x; e < 4096; e += NCW * 32) {
      const int r = e & 63, c = e >> 6;
      const double v = red[e] + red[4096 + e];
      const int gr = pc0 + r, gc = qc0 + c;
      if (gr < a.p && gc < a.q && (!a.gram || gr <= gc)) outp[gr + (int64_t)gc * a.p] = v;
    }
  }
}

// =========================================================================================
// k_update (fallback for operands without 16-byte TMA strides): X (m x q) -= L (m x p) S,
// in place (Alg. 7 l.9 P:351; Alg. 8 l.4 P:465 and l.7 P:468).  Work units (row tile, 64-
// column chunk xc, 64-wide k-chunk kc); one cp.async producer warp stages X, L and S tiles
// into 2-slot rings; 8 consumer warps with 32x16 warp tiles whose accumulators start from -X.
// The production path is k_update_pp below.
// =========================================================================================
constexpr size_t UPD_SMEM = sizeof(double) * (size_t)6 * TILE + 12 * sizeof(uint64_t) + 1024;
constexpr int XSLOT = 64 * 64;  // k_update_pp: dense 64x64 X tile in four 16-row swizzled boxes

// double index of element (column c, row r) of a swizzled X slot: box r/16 is [64 cols][16 rows],
// the 16-byte chunk (r%16)/2 of column c is XORed with c%8 (CU_TENSOR_MAP_SWIZZLE_128B)
__device__ __forceinline__ int xs_idx(int c, int r) {
  return (r >> 4) * 1024 + c * 16 + (((((r & 15) >> 1) ^ (c & 7))) << 1) + (r & 1);
}

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

__global__ void __launch_bounds__(NTHR, 1) k_update(const __grid_constant__ UpdArgs a) {
  extern __shared__ __align__(128) double smem_raw[];
  if (failed(a.status)) return;
  double* smem = aligned_smem(smem_raw, 128);
  double* ringL = smem;             // 2 slots
  double* ringS = smem + 2 * TILE;  // 2 slots
  double* ringX = smem + 4 * TILE;  // 2 slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE);
  uint64_t *fullL = bars, *emptyL = bars + 2, *fullS = bars + 4, *emptyS = bars + 6, *fullX = bars + 8,
           *emptyX = bars + 10;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntr = (a.m + TR - 1) / TR;
  const int nxc = (a.q + 63) / 64, nkc = (a.p + 63) / 64;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int nmine = (int)(first < ntr ? (ntr - 1 - first) / stride + 1 : 0);
  const int units = nmine * nxc * nkc;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fullL[i], 32); mbar_init(&emptyL[i], NCW);
      mbar_init(&fullS[i], 32); mbar_init(&emptyS[i], NCW);
      mbar_init(&fullX[i], 32); mbar_init(&emptyX[i], NCW);
    }
  }
  __syncthreads();
  // every unit stages its L and S chunks; X once per (tile, xc) (unit kc == 0)
  if (warp == PRODUCER) {
    for (int u = 0; u < units; ++u) {
      const int tl = u / (nxc * nkc), rem = u % (nxc * nkc), xc = rem / nkc, kc = rem % nkc;
      const int64_t row0 = (first + (int64_t)tl * stride) * TR;
      const int vX = u / nkc;
      if (kc == 0) {
        const int sl = vX & 1, use = vX >> 1;
        if (use > 0) mbar_wait(&emptyX[sl], (use - 1) & 1);
        produce_tile<TR, LDT, false, 64>(ringX + sl * TILE, a.X, a.ldx, row0, a.m, xc * 64, a.q, lane);
        cp_async_arrive(&fullX[sl]);
      }
      {
        const int sl = u & 1, use = u >> 1;
        if (use > 0) mbar_wait(&emptyL[sl], (use - 1) & 1);
        produce_tile<TR, LDT, false, 64>(ringL + sl * TILE, a.L, a.ldl, row0, a.m, kc * 64, a.p, lane);
        cp_async_arrive(&fullL[sl]);
        if (use > 0) mbar_wait(&emptyS[sl], (use - 1) & 1);
        produce_tile<64, LDT, false, 64>(ringS + sl * TILE, a.S, a.lds, (int64_t)kc * 64, a.p, xc * 64, a.q, lane);
        cp_async_arrive(&fullS[sl]);
      }
    }
    return;
  }
  const int gid = lane >> 2, tig = lane & 3, wr = warp >> 2, wc = warp & 3;
  double acc[4][2][2];
  for (int u = 0; u < units; ++u) {
    const int tl = u / (nxc * nkc), rem = u % (nxc * nkc), xc = rem / nkc, kc = rem % nkc;
    const int64_t row0 = (first + (int64_t)tl * stride) * TR;
    const int vX = u / nkc;
    if (kc == 0) {  // accumulators <- -X
      const int sl = vX & 1;
      mbar_wait(&fullX[sl], (vX >> 1) & 1);
      const double* sX = ringX + sl * TILE;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int r = wr * 32 + i * 8 + gid, col = wc * 16 + j * 8 + 2 * tig;
          acc[i][j][0] = -sX[col * LDT + r];
          acc[i][j][1] = -sX[(col + 1) * LDT + r];
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyX[sl]);
    }
    const int sl = u & 1;
    mbar_wait(&fullL[sl], (u >> 1) & 1);
    mbar_wait(&fullS[sl], (u >> 1) & 1);
    const double* sL = ringL + sl * TILE;
    const double* sS = ringS + sl * TILE;
    // k beyond p is zero-filled in both L and S: the full 64-wide chunk is exact
#pragma unroll 4
    for (int k0 = 0; k0 < 64; k0 += 4) {
      double fa[4], fb[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = sL[(k0 + tig) * LDT + wr * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 2; ++j) fb[j] = sS[(wc * 16 + j * 8 + gid) * LDT + k0 + tig];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[i], fb[j]);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&emptyL[sl]);
      mbar_arrive(&emptyS[sl]);
    }
    if (kc == nkc - 1) {  // X <- -acc
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t r = row0 + wr * 32 + i * 8 + gid;
        if (r < a.m) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = xc * 64 + wc * 16 + j * 8 + 2 * tig;
            if (col < a.q) a.X[r + (int64_t)col * a.ldx] = -acc[i][j][0];
            if (col + 1 < a.q) a.X[r + (int64_t)(col + 1) * a.ldx] = -acc[i][j][1];
          }
        }
      }
    }
  }
}

// =========================================================================================
// k_update_pp: update X -= L S (TMA operands; Alg. 7 l.9 P:351, Alg. 8 l.4 P:465 and l.7
// P:468) by two independent consumer warp groups.  Each group owns alternate 64-row tiles and
// walks all 64-column chunks of its tile with its own producer warp and 2-slot ring of 32-wide
// k halves (L half: [32 cols][68 rows], S half: [64 cols][36 k], both conflict-free for the
// m8n8k4 fragments).  Epilogue (UPP_RED, default): -acc goes into a 128B-swizzled slot and
// per-warp TMA REDUCE-ADD boxes (cp.reduce.async.bulk.tensor .add, FLOAT64) add it into X in
// the L2 -- X is never loaded into the SM, and the X - acc subtraction costs no DADD (DADDs
// queue on the FP64/DMMA pipe behind the other group's DMMAs); the L2's add is the same IEEE
// operation, so results are bitwise those of the load / subtract / store epilogue
// (UPP_RED = 0: TMA load of X into the slot, X - acc in place, TMA stores), ~2% slower at cfg3.
// With GW = 8 warps per group (32x16 warp tiles) every SMSP hosts two warps of each group, so
// while one group runs its epilogue the other still has two warps per SMSP issuing DMMAs --
// one warp per SMSP cannot keep the DMMA pipe full on shared-memory operands (measured ~30 of
// 37 TF; strict alternation of two 4-warp groups ran at exactly that rate).  Registers are
// moved from the producer warpgroup to the consumers with setmaxnreg.
// =========================================================================================
constexpr int UPP_GW = 8;                                  // warps per consumer group
constexpr int UPP_NJ = 16 / UPP_GW;                        // 8-column blocks per warp tile
constexpr int UPP_NTHR = (2 * UPP_GW + 4) * 32;            // + one producer warpgroup
constexpr int UPP_REG_CONS = UPP_GW == 8 ? 104 : 232;      // setmaxnreg budgets
constexpr int UPP_REG_PROD = 40;
#ifndef TSQR_UPP_RED
#define TSQR_UPP_RED 1
#endif
constexpr bool UPP_RED = TSQR_UPP_RED;  // epilogue: -acc through the slot + TMA reduce-add into X
#ifndef TSQR_UPP_KQ
#define TSQR_UPP_KQ 32
#endif
constexpr int UPP_KQ = TSQR_UPP_KQ;        // k per ring slot (32: halves; 16: quarters)
constexpr int UPP_NSL = 64 / UPP_KQ;       // ring slots (one 64-deep k chunk in flight)
constexpr int UPP_LSL = UPP_KQ * LDT;      // L slot (doubles)
constexpr int UPP_LDS = UPP_KQ + 4;        // S slot leading dimension (== 4 mod 16)
constexpr int UPP_SSL = 64 * UPP_LDS;      // S slot (doubles)
constexpr uint32_t UPP_TX = (UPP_LSL + UPP_SSL) * 8;
constexpr int UPP_GROUP = XSLOT + UPP_NSL * UPP_LSL + UPP_NSL * UPP_SSL;  // doubles per group
constexpr int UPP_NBAR = 2 * UPP_NSL + 2;  // full/empty per slot + fullX/emptyX
constexpr size_t UPP_SMEM = sizeof(double) * 2 * (size_t)UPP_GROUP + 2 * UPP_NBAR * sizeof(uint64_t) + 1024;

struct UppArgs {
  CUtensorMap mapX;   // X: box (16 rows, 64 cols), 128-byte swizzle (loads)
  CUtensorMap mapXs;  // X: box (16 rows, 8*UPP_NJ cols), 128-byte swizzle (stores)
  CUtensorMap mapL;   // L: box (68 rows, UPP_KQ cols)
  CUtensorMap mapS;   // S: box (UPP_KQ + 4 rows, 64 cols)
  int64_t m;
  int p, q;
  const int* status;
};

// optional per-phase cycle counters (build with -DTSQR_UPP_PROF; tools only): waits for the X
// slot / k halves, DMMA phases, epilogue, TMA-store read wait -- printed for two CTAs
#ifdef TSQR_UPP_PROF
#define UPP_PROF_DECL long long pf_[5] = {0, 0, 0, 0, 0}, pf_t_ = 0; const long long pf_s_ = clock64();
#define UPP_PROF_T0 pf_t_ = clock64();
#define UPP_PROF_ADD(i) { const long long n_ = clock64(); pf_[i] += n_ - pf_t_; pf_t_ = n_; }
#define UPP_PROF_PRINT                                                                                  \
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77) && (wg == 0 || wg == 5))                      \
    printf("upp cta %d grp %d wg %d: waitX %lld waitLS %lld mma %lld epi %lld wread %lld total %lld\n", \
           blockIdx.x, grp, wg, pf_[0], pf_[1], pf_[2], pf_[3], pf_[4], clock64() - pf_s_);
#else
#define UPP_PROF_DECL
#define UPP_PROF_T0
#define UPP_PROF_ADD(i)
#define UPP_PROF_PRINT
#endif

__global__ void __launch_bounds__(UPP_NTHR, 1) k_update_pp(const __grid_constant__ UppArgs a) {
  extern __shared__ __align__(128) double smem_raw[];
  if (failed(a.status)) return;
  double* smem = aligned_smem(smem_raw, 1024);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * UPP_GROUP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp >= 2 * UPP_GW;
  const int grp = producer ? (warp - 2 * UPP_GW) & 1 : warp / UPP_GW;
  double* sX = smem + grp * UPP_GROUP;  // 1024-byte aligned (swizzled slot)
  double* ringL = sX + XSLOT;
  double* ringS = ringL + UPP_NSL * UPP_LSL;
  uint64_t* fullLS = bars + grp * UPP_NBAR;
  uint64_t* emptyLS = fullLS + UPP_NSL;
  uint64_t* fullX = fullLS + 2 * UPP_NSL;
  uint64_t* emptyX = fullX + 1;

  const int64_t ntr = (a.m + TR - 1) / TR;
  const int nxc = (a.q + 63) / 64, nkh = (a.p + UPP_KQ - 1) / UPP_KQ;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int nmine = (int)(first < ntr ? (ntr - 1 - first) / stride + 1 : 0);
  const int ntl = nmine > grp ? (nmine - 1 - grp) / 2 + 1 : 0;  // this group's row tiles
  const int nch = ntl * nxc;

  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      uint64_t* b = bars + g * UPP_NBAR;
      for (int s = 0; s < UPP_NSL; ++s) {
        mbar_init(&b[s], 1);                  // fullLS
        mbar_init(&b[UPP_NSL + s], UPP_GW);   // emptyLS
      }
      mbar_init(&b[2 * UPP_NSL], 1); mbar_init(&b[2 * UPP_NSL + 1], UPP_GW);  // fullX, emptyX
    }
    tma_prefetch_map(&a.mapX);
    tma_prefetch_map(&a.mapXs);
    tma_prefetch_map(&a.mapL);
    tma_prefetch_map(&a.mapS);
  }
  __syncthreads();

  if (producer) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(UPP_REG_PROD) : "memory");
    if (warp >= 2 * UPP_GW + 2 || lane != 0) return;
    int vLS = 0;
    for (int ch = 0; ch < nch; ++ch) {
      const int tl = grp + 2 * (ch / nxc), xc = ch % nxc;
      const int64_t row0 = (first + (int64_t)tl * stride) * TR;
      for (int h = 0; h < nkh; ++h, ++vLS) {
        const int sl = vLS % UPP_NSL, use = vLS / UPP_NSL;
        if (use > 0) mbar_wait(&emptyLS[sl], (use - 1) & 1);
        mbar_arrive_expect_tx(&fullLS[sl], UPP_TX);
        tma_load_2d(ringL + sl * UPP_LSL, &a.mapL, (int)row0, h * UPP_KQ, &fullLS[sl]);
        tma_load_2d(ringS + sl * UPP_SSL, &a.mapS, h * UPP_KQ, xc * 64, &fullLS[sl]);
      }
      if (UPP_RED) continue;  // X is never loaded: the L2 adds -acc into it
      if (ch > 0) mbar_wait(emptyX, (ch - 1) & 1);
      mbar_arrive_expect_tx(fullX, XSLOT * 8);
      for (int t = 0; t < 4; ++t) tma_load_2d(sX + t * 1024, &a.mapX, (int)(row0 + 16 * t), xc * 64, fullX);
    }
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(UPP_REG_CONS) : "memory");
  const int wg = warp % UPP_GW, wr = wg / (UPP_GW / 2), wc = wg % (UPP_GW / 2);
  const int gid = lane >> 2, tig = lane & 3;
  const int c0 = wc * 8 * UPP_NJ;  // first column of this warp's tile within the chunk
  UPP_PROF_DECL
  int vLS = 0;
  for (int ch = 0; ch < nch; ++ch) {
    const int tl = grp + 2 * (ch / nxc), xc = ch % nxc;
    const int64_t row0 = (first + (int64_t)tl * stride) * TR;
    double acc[4][UPP_NJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < UPP_NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int h = 0; h < nkh; ++h, ++vLS) {
      const int sl = vLS % UPP_NSL;
      UPP_PROF_T0
      mbar_wait(&fullLS[sl], (vLS / UPP_NSL) & 1);
      UPP_PROF_ADD(1)
      const double* sL = ringL + sl * UPP_LSL + tig * LDT + wr * 32 + gid;
      const double* sS = ringS + sl * UPP_SSL + (c0 + gid) * UPP_LDS + tig;
      // fragments double-buffered in registers: step s+1 is loaded while step s issues
      double fa[2][4], fb[2][UPP_NJ];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[0][i] = sL[i * 8];
#pragma unroll
      for (int j = 0; j < UPP_NJ; ++j) fb[0][j] = sS[j * 8 * UPP_LDS];
#pragma unroll
      for (int s = 0; s < UPP_KQ / 4; ++s) {
        const int cb = s & 1, nb = cb ^ 1;
        if (s + 1 < UPP_KQ / 4) {
#pragma unroll
          for (int i = 0; i < 4; ++i) fa[nb][i] = sL[(s + 1) * 4 * LDT + i * 8];
#pragma unroll
          for (int j = 0; j < UPP_NJ; ++j) fb[nb][j] = sS[j * 8 * UPP_LDS + (s + 1) * 4];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < UPP_NJ; ++j) dmma(acc[i][j][0], acc[i][j][1], fa[cb][i], fb[cb][j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyLS[sl]);
      UPP_PROF_ADD(2)
    }
    // epilogue: X <- X - acc in the slot (all loads before any store: a store may alias a
    // later load for the compiler, and interleaving them serialises the load->add->store
    // chains), then TMA stores of 16 rows x 8*NJ columns per warp
    if (UPP_RED) {  // slot <- -acc (sign flips on the integer pipe)
      // the previous chunk's reduce-add boxes must have read this warp's region: waited for
      // here, a whole chunk of DMMAs after they were issued, instead of right after issuing
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < UPP_NJ; ++j) {
          const int r = wr * 32 + i * 8 + gid, col = c0 + j * 8 + 2 * tig;
          sX[xs_idx(col, r)] = __longlong_as_double(__double_as_longlong(acc[i][j][0]) ^ (long long)0x8000000000000000ULL);
          sX[xs_idx(col + 1, r)] = __longlong_as_double(__double_as_longlong(acc[i][j][1]) ^ (long long)0x8000000000000000ULL);
        }
    } else {
      UPP_PROF_T0
      mbar_wait(fullX, ch & 1);
      UPP_PROF_ADD(0)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < UPP_NJ; ++j) {
          const int r = wr * 32 + i * 8 + gid, col = c0 + j * 8 + 2 * tig;
          acc[i][j][0] = sX[xs_idx(col, r)] - acc[i][j][0];
          acc[i][j][1] = sX[xs_idx(col + 1, r)] - acc[i][j][1];
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < UPP_NJ; ++j) {
          const int r = wr * 32 + i * 8 + gid, col = c0 + j * 8 + 2 * tig;
          sX[xs_idx(col, r)] = acc[i][j][0];
          sX[xs_idx(col + 1, r)] = acc[i][j][1];
        }
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int box = 2 * wr + t;
        if (UPP_RED)
          tma_reduce_add_2d(&a.mapXs, (int)(row0 + 16 * box), xc * 64 + c0, sX + box * 1024 + c0 * 16);
        else
          tma_store_2d(&a.mapXs, (int)(row0 + 16 * box), xc * 64 + c0, sX + box * 1024 + c0 * 16);
      }
      bulk_commit();
    }
    UPP_PROF_ADD(3)
    if (!UPP_RED) {
      if (lane == 0) bulk_wait_read0();  // the TMA stores have read the slot
      __syncwarp();
      UPP_PROF_ADD(4)
      if (lane == 0) mbar_arrive(emptyX);
    }
  }
  UPP_PROF_PRINT
  if (lane == 0) bulk_wait0();
}

// =========================================================================================
// k_trmm: X (m x B) <- X * Z in place, Z upper triangular (B x B): panel orthogonalisation
// Q = A R^{-1} with the explicit inverse (Alg. 1 l.3 P:133; R-4).  Row tiles are streamed
// through a 3-stage ring; warp w owns a row group and balanced column-block pairs
// (cb, NB-1-cb) so the triangular work is even.  Z is in shared memory for B <= 64, read
// through L1/L2 otherwise (b >= 128 panels use the blocked 64-wide TRMM + update path).
// =========================================================================================
template <int B>
struct TrmmCfg {
  static constexpr int NB = B / 8;
  static constexpr int PAIRS = NB / 2;
  static constexpr int PAIRS_PER_WARP = PAIRS >= NCW ? PAIRS / NCW : 1;
  static constexpr int ROW_GROUPS = PAIRS >= NCW ? 1 : NCW / PAIRS;
  static constexpr int TRR = (B <= 128) ? 64 : 32;
  static constexpr int LD = TRR + 4;
  static constexpr int RB = TRR / 8 / ROW_GROUPS;
  // U^{-1} in shared memory: square (B <= 64, ld B + 4) or packed by 8-column block (B = 128:
  // block cb keeps rows 0..8cb+7 with ld == 4 mod 16, conflict-free B fragments); B = 256
  // reads it through L1 / L2
  static constexpr bool ZSMEM = (B <= 128);
  static constexpr bool ZPACK = (B == 128);
  static constexpr int LDZ = B + 4;
  __host__ __device__ static constexpr int zld(int cb) { return (8 * (cb + 1)) % 16 == 0 ? 8 * (cb + 1) + 4 : 8 * (cb + 1) + 12; }
  __host__ __device__ static constexpr int zoff(int cb) { return cb == 0 ? 0 : zoff(cb - 1) + 8 * zld(cb - 1); }
  static constexpr int ZDBL = ZPACK ? zoff(NB) : (ZSMEM ? B * LDZ : 0);
  static constexpr int NS = (B == 128) ? 2 : 3;  // ring stages
  static constexpr int BOXC = B < 64 ? B : 64;  // columns per TMA box
  static constexpr int TILE_DBL = B * LD;
  // TMA-store epilogue (B = 32, 64): 2 output slots of 64 rows x B columns, 128B-swizzled
  // 16-row boxes; each warp's 8-column blocks are stored by box (16 rows x 8 columns)
  static constexpr bool OUT_TMA = (B == 32 || B == 64);
  static constexpr int OUT_DBL = OUT_TMA ? B * 64 : 0;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)2 * OUT_DBL + (size_t)NS * TILE_DBL + (size_t)ZDBL) +
                                 2 * NS * sizeof(uint64_t) + 1024;
};

struct TrmmArgs {
  CUtensorMap mapX;   // X: rows m, cols B, box (LD rows, BOXC cols)
  CUtensorMap mapXs;  // X: rows m, cols B, box (16 rows, 8 cols), 128B swizzle (stores)
  double* X;
  int64_t ldx;
  int64_t m;
  const double* Z;
  int ldz;
  const int* status;
};

template <int B, bool TMA>
__global__ void __launch_bounds__(NTHR, 1) k_trmm(const __grid_constant__ TrmmArgs a) {
  using C = TrmmCfg<B>;
  extern __shared__ __align__(128) double smem_raw[];
  if (failed(a.status)) return;
  double* smem = aligned_smem(smem_raw, 1024);
  double* outs = smem;                        // 2 swizzled output slots (TMA path, B = 32, 64)
  double* ring = smem + 2 * C::OUT_DBL;
  double* sZ = ring + C::NS * C::TILE_DBL;
  uint64_t* full = reinterpret_cast<uint64_t*>(sZ + C::ZDBL);
  uint64_t* empty = full + C::NS;
  double* X = a.X;
  const int64_t ldx = a.ldx, m = a.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntr = (m + C::TRR - 1) / C::TRR;
  const int64_t first = blockIdx.x, stride = gridDim.x;
  const int nmine = (int)(first < ntr ? (ntr - 1 - first) / stride + 1 : 0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(&full[i], TMA ? 1 : 32);
      mbar_init(&empty[i], NCW);
    }
    if (TMA) {
      tma_prefetch_map(&a.mapX);
      if (C::OUT_TMA) tma_prefetch_map(&a.mapXs);
    }
  }
  __syncthreads();

  if (warp == PRODUCER) {
    for (int it = 0; it < nmine; ++it) {
      const int st = it % C::NS, use = it / C::NS;
      if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
      const int64_t row0 = (first + (int64_t)it * stride) * C::TRR;
      if (TMA) {
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[st], (uint32_t)(C::TILE_DBL * 8));
          for (int c0 = 0; c0 < B; c0 += 64)
            tma_load_2d(ring + st * C::TILE_DBL + c0 * C::LD, &a.mapX, (int)row0, c0, &full[st]);
        }
      } else {
        for (int c0 = 0; c0 < B; c0 += 64)
          produce_tile<C::TRR, C::LD, false, C::BOXC>(ring + st * C::TILE_DBL + c0 * C::LD, X, ldx, row0, m, c0, B,
                                                      lane);
        cp_async_arrive(&full[st]);
      }
    }
    return;
  }

  if (C::ZPACK) {
    for (int e = threadIdx.x; e < B * B; e += NCW * 32) {
      const int k = e % B, col = e / B, cb = col >> 3;
      if (k < 8 * (cb + 1)) sZ[C::zoff(cb) + (col & 7) * C::zld(cb) + k] = a.Z[k + (int64_t)col * a.ldz];
    }
    consumer_sync();
  } else if (C::ZSMEM) {
    for (int e = threadIdx.x; e < B * B; e += NCW * 32) {
      const int k = e % B, col = e / B;
      sZ[col * C::LDZ + k] = a.Z[k + (int64_t)col * a.ldz];
    }
    consumer_sync();
  }
  const int gid = lane >> 2, tig = lane & 3;
  const int rg = warp % C::ROW_GROUPS, pw = warp / C::ROW_GROUPS;
  constexpr int CBW = 2 * C::PAIRS_PER_WARP;
  int cbs[CBW];
#pragma unroll
  for (int u = 0; u < C::PAIRS_PER_WARP; ++u) {
    const int pr = pw * C::PAIRS_PER_WARP + u;
    cbs[2 * u] = pr;
    cbs[2 * u + 1] = C::NB - 1 - pr;
  }
  // the same blocks sorted by their k-bound (ascending): pr_0 < pr_1 < ... < NB-1-pr_1 < NB-1-pr_0
  int cs[CBW];
#pragma unroll
  for (int u = 0; u < C::PAIRS_PER_WARP; ++u) {
    cs[u] = cbs[2 * u];
    cs[CBW - 1 - u] = cbs[2 * u + 1];
  }

  for (int it = 0; it < nmine; ++it) {
    const int st = it % C::NS;
    mbar_wait(&full[st], (it / C::NS) & 1);
    double* sX = ring + st * C::TILE_DBL;
    const int64_t row0 = (first + (int64_t)it * stride) * C::TRR;
    double acc[C::RB][CBW][2];
#pragma unroll
    for (int i = 0; i < C::RB; ++i)
#pragma unroll
      for (int u = 0; u < CBW; ++u) acc[i][u][0] = acc[i][u][1] = 0.0;
    // triangular k-loop in phases: in phase ph only the column blocks whose k-range is not yet
    // exhausted are active (sorted by bound, compile-time active set) -- no predicated DMMAs,
    // which would still occupy the tensor pipe
    int k0 = 0;
#pragma unroll
    for (int ph = 0; ph < CBW; ++ph) {
      const int kend = (cs[ph] + 1) * 8;
      for (; k0 < kend; k0 += 4) {
        double fa[C::RB];
#pragma unroll
        for (int i = 0; i < C::RB; ++i) fa[i] = sX[(k0 + tig) * C::LD + (rg * C::RB + i) * 8 + gid];
#pragma unroll
        for (int u = ph; u < CBW; ++u) {
          const int col = cs[u] * 8 + gid;
          const double fb = C::ZPACK   ? sZ[C::zoff(cs[u]) + gid * C::zld(cs[u]) + k0 + tig]
                            : C::ZSMEM ? sZ[col * C::LDZ + k0 + tig]
                                       : __ldg(a.Z + (k0 + tig) + (int64_t)col * a.ldz);
#pragma unroll
          for (int i = 0; i < C::RB; ++i) dmma(acc[i][u][0], acc[i][u][1], fa[i], fb);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (TMA && C::OUT_TMA) {
      // X_new -> swizzled output slot -> TMA box stores (rows past m are clipped)
      double* so = outs + (it & 1) * C::OUT_DBL;
      if (it >= 2) {
        if (lane == 0) bulk_wait_read1();  // this slot's stores from tile it-2 have been read
        __syncwarp();
      }
#pragma unroll
      for (int i = 0; i < C::RB; ++i) {
        const int r = (rg * C::RB + i) * 8 + gid;
#pragma unroll
        for (int u = 0; u < CBW; ++u) {
          const int c = cs[u] * 8 + 2 * tig;
          so[(r >> 4) * (B * 16) + c * 16 + ((((r & 15) >> 1) ^ (c & 7)) << 1) + (r & 1)] = acc[i][u][0];
          so[(r >> 4) * (B * 16) + (c + 1) * 16 + ((((r & 15) >> 1) ^ ((c + 1) & 7)) << 1) + (r & 1)] =
              acc[i][u][1];
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int rb = 0; rb < C::RB / 2; ++rb) {
          const int box = (rg * C::RB) / 2 + rb;
#pragma unroll
          for (int u = 0; u < CBW; ++u)
            tma_store_2d(&a.mapXs, (int)(row0 + 16 * box), cs[u] * 8, so + box * (B * 16) + cs[u] * 8 * 16);
        }
        bulk_commit();
      }
    } else {
#pragma unroll
      for (int i = 0; i < C::RB; ++i) {
        const int64_t r = row0 + (rg * C::RB + i) * 8 + gid;
        if (r < m) {
#pragma unroll
          for (int u = 0; u < CBW; ++u) {
            const int c = cs[u] * 8 + 2 * tig;
            X[r + (int64_t)c * ldx] = acc[i][u][0];
            X[r + (int64_t)(c + 1) * ldx] = acc[i][u][1];
          }
        }
      }
    }
  }
  if (TMA && C::OUT_TMA && lane == 0) bulk_wait0();
}

}  // namespace tsqr
