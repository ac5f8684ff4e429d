// tsqr.cu -- host orchestrator and C ABI of libtsqr (include/tsqr.h).
//
// The panel loops of the paper's algorithms (Alg. 2, 3, 7, 8 of arXiv 2405.04237) are
// enqueued on one CUDA stream: every O(m) step is one of the sm_100a kernels in
// kernels.cuh, every cross-GPU sum is one in-stream ncclAllReduce(ncclFloat64, ncclSum) of
// a small replicated block (b x b Gram, b x N projection, (j-1)b x b re-orthogonalisation
// block), and Cholesky / R assembly run redundantly on every rank.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "tsqr.h"

using namespace tsqr;

namespace {

thread_local char g_err[512] = "";

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define CUDA_TRY(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      set_err("%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return TSQR_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

#define NCCL_TRY(x)                                                                      \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess) {                                                             \
      set_err("%s failed: %s (%s:%d)", #x, ncclGetErrorString(r_), __FILE__, __LINE__); \
      return TSQR_ERR_NCCL;                                                              \
    }                                                                                    \
  } while (0)

#define TRY(x)                          \
  do {                                  \
    tsqr_status s_ = (x);               \
    if (s_ != TSQR_OK) return s_;       \
  } while (0)

// SM count of the current device (148 on B200), queried once per process: the split-row
// partition below is a function of (m, p, q, SM count) only, so it is identical on every rank
// of a homogeneous node.
int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      n = v;
    else
      n = 148;
  }
  return n;
}
constexpr size_t kAlign = 256;

size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// panel widths: 16, 32, or any multiple of 64 up to 4096 (b > 256: the wide panels of the paper's
// strong-scaling workload, with the multi-CTA blocked Cholesky; DESIGN R-24)
bool valid_b(int b) { return b == 16 || b == 32 || (b % 64 == 0 && b >= 64 && b <= 4096); }

// ---- split-row policy of k_atb (a function of the problem only -> deterministic) ----
struct AtbShape {
  int ntp, ntq, tiles, S;  // S: splits of full tiles
  int64_t tps;             // row tiles per split (full tiles)
  int Sd;                  // splits of diagonal Gram tiles
  int64_t tpsd;
  int Smax() const { return S > Sd ? S : Sd; }
};

// splits of `total` row tiles into about `want` parts of equal size (>= 4 row tiles each)
void split_rows(int64_t ntr, double want, int& S, int64_t& tps) {
  int64_t s = (int64_t)(want + 1e-9);
  const int64_t maxS = std::max<int64_t>(1, ntr / 4);
  s = std::max<int64_t>(1, std::min<int64_t>(s, maxS));
  tps = std::max<int64_t>(1, (ntr + s - 1) / s);
  S = (int)std::max<int64_t>(1, (ntr + tps - 1) / tps);
  if (ntr == 0) S = 1;
}

// Diagonal Gram tiles cost 576 DMMA per 64-row tile, full tiles 1024: give each tile type
// its own number of row splits so every CTA carries the same work.  The split count is then
// raised (up to 4x) to the value whose CTA count fills whole waves of 148 SMs best (one CTA
// per SM), e.g. 112 projection tiles -> 5 splits (560 CTAs, 95% of 4 waves) instead of 1.
AtbShape atb_shape(int64_t m, int p, int q, bool gram) {
  AtbShape s;
  s.ntp = (p + 63) / 64;
  s.ntq = (q + 63) / 64;
  const int nd = gram ? s.ntq : 0;                                  // diagonal tiles
  const int nf = gram ? s.ntq * (s.ntq - 1) / 2 : s.ntp * s.ntq;    // full tiles
  s.tiles = nd + nf;
  const int64_t ntr = (m + TR - 1) / TR;
  const double wd = 576.0 / 1024.0;
  const int kSMs = sm_count();
  double unit = (double)kSMs / (nd * wd + nf);                      // splits per full tile
  if (unit < 4.0) {
    // few splits: choose the multiplier with the best wave efficiency (weighted CTA work)
    double best_eff = 0.0, best_u = std::max(1.0, unit);
    for (int f = 1; f <= 16; ++f) {
      const double u = std::max(1.0, unit) * f / 4.0;
      if (u < 1.0) continue;
      const double work = nf * std::floor(u) + nd * std::max(1.0, std::floor(u * wd)) * wd;
      const double ctas = nf * std::floor(u) + nd * std::max(1.0, std::floor(u * wd));
      const double waves = std::ceil(ctas / kSMs);
      const double eff = work / (waves * kSMs);
      if (eff > best_eff + 1e-3) { best_eff = eff; best_u = u; }
    }
    unit = best_u;
  }
  split_rows(ntr, nf ? std::max(1.0, unit) : 1.0, s.S, s.tps);
  split_rows(ntr, nd ? std::max(1.0, unit * wd) : 1.0, s.Sd, s.tpsd);
  return s;
}

size_t atb_part_doubles(int64_t m, int p, int q, bool gram) {
  AtbShape s = atb_shape(m, p, q, gram);
  return (size_t)s.Smax() * (size_t)p * (size_t)q;
}

int grid_1d(int64_t n, int nt = 256) {
  int64_t g = (n + nt - 1) / nt;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 4 * sm_count()));
}

// ---- TMA tensor maps (cuTensorMapEncodeTiled fetched through the runtime: no -lcuda) ----
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

tsqr_status tma_encoder() {
  if (g_encode) return TSQR_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) {
    set_err("cuTensorMapEncodeTiled unavailable");
    return TSQR_ERR_CUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return TSQR_OK;
}

// column-major FP64 matrix (rows x cols, leading dimension ld) as a 2-D tensor map with a
// (box_rows x box_cols) box; out-of-bounds elements read as zero
tsqr_status make_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int box_cols, bool swizzle128 = false) {
  TRY(tma_encoder());
  cuuint64_t dims[2] = {(cuuint64_t)std::max<int64_t>(rows, 1), (cuuint64_t)std::max<int64_t>(cols, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_err("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld", (int)r, (long long)rows,
            (long long)cols, (long long)ld);
    return TSQR_ERR_CUDA;
  }
  return TSQR_OK;
}

// TMA needs a 16-byte aligned base, 16-byte multiple strides and at least one row
bool tma_ok(const void* ptr, int64_t ld, int64_t rows) {
  return rows > 0 && ((reinterpret_cast<uintptr_t>(ptr) & 15u) == 0) && (ld % 2 == 0);
}

// ---- optional per-kernel-class event timing ----
struct Timer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Rec { int cls; size_t e0, e1; double flops, bytes; };
  std::vector<Rec> recs;
  // accumulated totals per class (filled by harvest)
  double ms[TSQR_KCLASS_COUNT] = {0}, fl[TSQR_KCLASS_COUNT] = {0}, by[TSQR_KCLASS_COUNT] = {0};
  int64_t cnt[TSQR_KCLASS_COUNT] = {0};

  size_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return (size_t)-1;
      pool.push_back(e);
    }
    return used++;
  }
  size_t begin(cudaStream_t st) {
    if (!on) return (size_t)-1;
    size_t e = ev();
    // External: during stream capture this becomes a timestamped event-record node of the graph
    if (e != (size_t)-1) cudaEventRecordWithFlags(pool[e], st, capturing ? cudaEventRecordExternal : 0u);
    return e;
  }
  void end(cudaStream_t st, size_t e0, int cls, double flops, double bytes) {
    if (!on || e0 == (size_t)-1) return;
    size_t e1 = ev();
    if (e1 == (size_t)-1) return;
    cudaEventRecordWithFlags(pool[e1], st, capturing ? cudaEventRecordExternal : 0u);
    recs.push_back({cls, e0, e1, flops, bytes});
  }
  // fold recorded events into the totals (events must be complete)
  // graph mode: `recs` were recorded while capturing a CUDA graph and are re-recorded by every
  // replay; `pending` counts replays whose events have not been folded in yet
  bool graph_recs = false;
  bool capturing = false;  // events are being recorded into a CUDA graph capture
  int pending = 0;
  void harvest() {
    if (graph_recs && pending == 0) return;
    for (const Rec& r : recs) {
      float t = 0.f;
      cudaEventElapsedTime(&t, pool[r.e0], pool[r.e1]);
      ms[r.cls] += t; fl[r.cls] += r.flops; by[r.cls] += r.bytes; cnt[r.cls] += 1;
    }
    pending = 0;
    if (!graph_recs) {
      recs.clear();
      used = 0;
    }
  }
  void drop_recs() { recs.clear(); used = 0; graph_recs = false; pending = 0; }
  void reset() {
    if (!graph_recs) { recs.clear(); used = 0; }
    pending = 0;
    for (int c = 0; c < TSQR_KCLASS_COUNT; ++c) { ms[c] = fl[c] = by[c] = 0; cnt[c] = 0; }
  }
  ~Timer() { for (auto e : pool) cudaEventDestroy(e); }
};

// ---- kernel launchers (single GPU, enqueue only) ----

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

struct Launcher {
  cudaStream_t st = nullptr;
  int64_t launches = 0;
  const int* status = nullptr;
  Timer* timer = nullptr;

  size_t tbegin() { return timer ? timer->begin(st) : (size_t)-1; }
  void tend(size_t e0, int cls, double flops, double bytes) { if (timer) timer->end(st, e0, cls, flops, bytes); }

  tsqr_status reduce(const double* part, int S, int p, int q, int ldp, int64_t pstride, double* out, int ldo,
                     bool gram, int Sdiag = -1) {
    const int64_t groups = ((int64_t)p * q + 31) / 32;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, 8 * sm_count()));
    k_reduce<<<grid, RED_NT, 0, st>>>(part, S, Sdiag < 0 ? S : Sdiag, p, q, ldp, pstride, out, ldo, gram ? 1 : 0,
                                      status);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    return TSQR_OK;
  }

  // cross-GPU sum fused into the reduction (fused_allreduce.cuh); ar_on with 2-4 ranks (or forced)
  bool ar_on = false;
  ncclDevComm ar_dc{};
  ncclWindow_t ar_win = nullptr;
  int ar_nranks = 1, ar_rank = 0;
  int64_t ar_cap = 0;  // doubles per rank slot of the window (b * n: the largest summed block)
  // Blocks above this many doubles take k_reduce + ncclAllReduce even on the fused plane: the
  // fused kernel's element-wise peer stores suit the <= 224 KiB blocks of the weak-scaling
  // configurations, NCCL's bandwidth algorithms the 100+ MB blocks of the wide panels (NEXT-f3).
  // A function of the block shape only -> the same choice on every rank.
  int64_t ar_fuse_max = int64_t(1) << 20;
  bool fuse(int64_t count) const { return ar_on && count <= ar_fuse_max; }

  // OUT (p x q, ldo) = L^T R summed over all m rows (split-row partials + fixed-order reduce);
  // with `global` and the fused path on: summed over every rank as well (one kernel)
  tsqr_status atb(const double* L, int64_t ldl, const double* R, int64_t ldr, int64_t m, int p, int q, bool gram,
                  double* part, double* out, int ldo, bool global = false) {
    AtbShape sh = atb_shape(m, p, q, gram);
    ProjArgs a;
    std::memset(&a, 0, sizeof(a));
    a.L = L; a.ldl = ldl; a.R = R; a.ldr = ldr; a.m = m; a.p = p; a.q = q; a.gram = gram ? 1 : 0;
    a.ntp = sh.ntp; a.ntq = sh.ntq; a.tiles_per_split = sh.tps; a.part = part; a.status = status;
    a.S_full = sh.S; a.S_diag = sh.Sd; a.tiles_per_split_diag = sh.tpsd;
    dim3 grid(sh.tiles, sh.Smax());
    const bool tma = tma_ok(L, ldl, m) && tma_ok(R, ldr, m);
    if (tma) {
      TRY(make_map(&a.mapL, L, m, p, ldl, LDT, 64));
      TRY(make_map(&a.mapR, R, m, q, ldr, LDT, 64));
    }
    const size_t t0 = tbegin();
    if (tma) {
      CUDA_TRY(set_smem(k_proj<true>, PROJ_SMEM));
      k_proj<true><<<grid, NTHR, PROJ_SMEM, st>>>(a);
    } else {
      CUDA_TRY(set_smem(k_proj<false>, PROJ_SMEM));
      k_proj<false><<<grid, NTHR, PROJ_SMEM, st>>>(a);
    }
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    if (global && fuse((int64_t)p * q)) {
      if (gram) tend(t0, TSQR_KCLASS_GRAM, (double)m * p * p, 8.0 * m * p);
      else tend(t0, TSQR_KCLASS_PROJ, 2.0 * m * p * q, 8.0 * m * (p + q));
      const size_t t1 = tbegin();
      k_reduce_allreduce<<<AR_CTAS, AR_NT, 0, st>>>(part, sh.S, sh.Sd, p, q, p, (int64_t)p * q, out, ldo,
                                                    gram ? 1 : 0, status, ar_dc, ar_win, ar_nranks, ar_rank, ar_cap);
      CUDA_TRY(cudaGetLastError());
      launches += 1;
      tend(t1, TSQR_KCLASS_ALLREDUCE, 0.0, 8.0 * p * q);
      return TSQR_OK;
    }
    TRY(reduce(part, sh.S, p, q, p, (int64_t)p * q, out, ldo, gram, sh.Sd));
    if (gram) tend(t0, TSQR_KCLASS_GRAM, (double)m * p * p, 8.0 * m * p);
    else tend(t0, TSQR_KCLASS_PROJ, 2.0 * m * p * q, 8.0 * m * (p + q));
    return TSQR_OK;
  }

  // X <- X Z (in place)
  template <int B>
  tsqr_status trmm_b(double* X, int64_t ldx, int64_t m, const double* Z, int ldz) {
    using C = TrmmCfg<B>;
    const int grid = sm_count();
    TrmmArgs a;
    std::memset(&a, 0, sizeof(a));
    a.X = X; a.ldx = ldx; a.m = m; a.Z = Z; a.ldz = ldz; a.status = status;
    const bool tma = tma_ok(X, ldx, m);
    if (tma) {
      TRY(make_map(&a.mapX, X, m, B, ldx, C::LD, C::BOXC));
      if (C::OUT_TMA) TRY(make_map(&a.mapXs, X, m, B, ldx, 16, 8, true));
    }
    const size_t t0 = tbegin();
    if (tma) {
      CUDA_TRY(set_smem(k_trmm<B, true>, C::SMEM));
      k_trmm<B, true><<<grid, NTHR, C::SMEM, st>>>(a);
    } else {
      CUDA_TRY(set_smem(k_trmm<B, false>, C::SMEM));
      k_trmm<B, false><<<grid, NTHR, C::SMEM, st>>>(a);
    }
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_TRMM, (double)m * B * B, 16.0 * m * B);
    return TSQR_OK;
  }

  tsqr_status trmm(double* X, int64_t ldx, int64_t m, int b, const double* Z, int ldz) {
    switch (b) {
      case 16: return trmm_b<16>(X, ldx, m, Z, ldz);
      case 32: return trmm_b<32>(X, ldx, m, Z, ldz);
      case 64: return trmm_b<64>(X, ldx, m, Z, ldz);
      case 128: return trmm_b<128>(X, ldx, m, Z, ldz);
      case 256: return trmm_b<256>(X, ldx, m, Z, ldz);
      default: set_err("trmm: unsupported b=%d", b); return TSQR_ERR_UNSUPPORTED;
    }
  }

  // X <- X Z for b = 64 c (c >= 2) by 64-column blocks, last block first (so every block
  // still reads the old columns to its left):  X_J <- X_J Z_JJ  (64-wide TRMM), then
  // X_J -= X_{0:J} (-Z_{0:J,J})  (update kernel, Zn = -Z staged in `zwork`, b x b).
  // Same flops as the direct kernel, but on the two kernels that run near the DMMA roof
  // instead of the B = 128/256 TRMM whose Z no longer fits shared memory at full width.
  tsqr_status trmm_blocked(double* X, int64_t ldx, int64_t m, int b, const double* Z, int ldz, double* zwork) {
    TRY(copy2d(Z, ldz, zwork, b, b, b, -1.0));
    for (int J = b / 64 - 1; J >= 0; --J) {
      double* XJ = X + (int64_t)J * 64 * ldx;
      TRY(trmm_b<64>(XJ, ldx, m, Z + (int64_t)J * 64 + (int64_t)J * 64 * ldz, ldz));
      if (J > 0) TRY(update(XJ, ldx, X, ldx, zwork + (int64_t)J * 64 * b, b, m, 64 * J, 64));
    }
    return TSQR_OK;
  }

  // X (m x q) -= L (m x p) S (p x q)
  tsqr_status update(double* X, int64_t ldx, const double* L, int64_t ldl, const double* S, int64_t lds, int64_t m,
                     int p, int q) {
    const int grid = sm_count();
    const bool tma = tma_ok(X, ldx, m) && tma_ok(L, ldl, m) && tma_ok(S, lds, p);
    const size_t t0 = tbegin();
    if (tma) {
      UppArgs a;
      std::memset(&a, 0, sizeof(a));
      a.m = m; a.p = p; a.q = q; a.status = status;
      TRY(make_map(&a.mapX, X, m, q, ldx, 16, 64, true));
      TRY(make_map(&a.mapXs, X, m, q, ldx, 16, 8 * UPP_NJ, true));
      TRY(make_map(&a.mapL, L, m, p, ldl, LDT, UPP_KQ));
      TRY(make_map(&a.mapS, S, p, q, lds, UPP_LDS, 64));
      CUDA_TRY(set_smem(k_update_pp, UPP_SMEM));
      k_update_pp<<<grid, UPP_NTHR, UPP_SMEM, st>>>(a);
    } else {
      UpdArgs a;
      std::memset(&a, 0, sizeof(a));
      a.X = X; a.ldx = ldx; a.L = L; a.ldl = ldl; a.S = S; a.lds = lds; a.m = m; a.p = p; a.q = q;
      a.status = status;
      CUDA_TRY(set_smem(k_update, UPD_SMEM));
      k_update<<<grid, NTHR, UPD_SMEM, st>>>(a);
    }
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_UPDATE, 2.0 * m * p * q, 8.0 * m * (p + 2.0 * q));
    return TSQR_OK;
  }

  // Z = U^{-1} on the 64-block range [lo, hi) by recursive halving (the diagonal blocks Z_II come
  // from k_chol_diag): inv([A B; 0 C]) = [A^-1, -A^-1 B C^-1; 0, C^-1] (R-4), the two products of
  // every split on the DMMA update kernel: T = 0; T -= Z_AA U_AC; T = -T; Z_AC -= T Z_CC.
  // (A chain of block back-substitutions would serialise ~nb^2/2 block products; the halving
  // needs log2(nb) dependent levels of large GEMMs.)  T uses `work` (b x b, ld b).
  tsqr_status tri_inv_rec(const double* U, int ldu, double* Z, int ldz, int b, int lo, int hi, double* work) {
    if (hi - lo < 2) return TSQR_OK;
    const int mid = lo + (hi - lo) / 2;
    TRY(tri_inv_rec(U, ldu, Z, ldz, b, lo, mid, work));
    TRY(tri_inv_rec(U, ldu, Z, ldz, b, mid, hi, work));
    const int a0 = lo * CHB, c0 = mid * CHB, sa = (mid - lo) * CHB, sc = (hi - mid) * CHB;
    double* T = work;
    k_zero2d<<<grid_1d((int64_t)sa * sc), 256, 0, st>>>(T, b, sa, sc);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    TRY(update(T, b, Z + a0 + (int64_t)a0 * ldz, ldz, U + a0 + (int64_t)c0 * ldu, ldu, sa, sa, sc));
    TRY(copy2d(T, b, T, b, sa, sc, -1.0));
    return update(Z + a0 + (int64_t)c0 * ldz, ldz, T, b, Z + c0 + (int64_t)c0 * ldz, ldz, sa, sc, sc);
  }

  tsqr_status chol_inv(const double* W, int ldw, int b, double* U, int ldu, double* Z, int ldz, int* status_rw,
                       int pass, int panel, int stage, double* work) {
    const size_t t0 = tbegin();
    if (b > 256 && b % 64 == 0 && work) {  // wide panels: multi-CTA blocked variant, one launch per step
      const int nb = b / CHB;
      CUDA_TRY(set_smem(k_chol_diag, CHOL_BLK_SMEM));
      CUDA_TRY(set_smem(k_chol_row, CHOL_BLK_SMEM));
      CUDA_TRY(set_smem(k_chol_trail, CHOL_BLK_SMEM));
      CUDA_TRY(set_smem(k_tri_inv_step, CHOL_BLK_SMEM));
      k_chol_prep<<<grid_1d((int64_t)b * b), 256, 0, st>>>(W, ldw, b, work, U, ldu, Z, ldz, status_rw);
      launches += 1;
      for (int J = 0; J < nb; ++J) {
        k_chol_diag<<<1, CHOL_NT, CHOL_BLK_SMEM, st>>>(work, b, J, U, ldu, Z, ldz, status_rw, pass, panel, stage);
        const int r = nb - J - 1;
        if (r > 0) {
          k_chol_row<<<r, CHOL_NT, CHOL_BLK_SMEM, st>>>(work, b, J, U, ldu, Z, ldz, status_rw);
          k_chol_trail<<<r * (r + 1) / 2, CHOL_NT, CHOL_BLK_SMEM, st>>>(work, b, J, U, ldu, status_rw);
        }
        launches += r > 0 ? 3 : 1;
      }
      CUDA_TRY(cudaGetLastError());
      Timer* tm = timer;
      timer = nullptr;  // the inverse's update launches are part of this Cholesky's timed range
      const tsqr_status si = tri_inv_rec(U, ldu, Z, ldz, b, 0, nb, work);
      timer = tm;
      TRY(si);

      tend(t0, TSQR_KCLASS_CHOL, 2.0 * b * b * b / 3.0, 16.0 * b * b);
      return TSQR_OK;
    }
    if (b >= 128 && b % 64 == 0 && work) {  // blocked variant (64x64 blocks, W staged in `work`)
      CUDA_TRY(set_smem(k_chol_inv_blocked, CHOL_BLK_SMEM));
      k_chol_inv_blocked<<<1, CHOL_NT, CHOL_BLK_SMEM, st>>>(W, ldw, b, U, ldu, Z, ldz, status_rw, pass, panel, stage,
                                                            work);
    } else {
      const size_t smem = chol_smem_bytes(b);
      CUDA_TRY(set_smem(k_chol_inv<CHOL_NT_SMALL>, smem > 0 ? smem : 1));
      k_chol_inv<CHOL_NT_SMALL><<<1, CHOL_NT_SMALL, smem, st>>>(W, ldw, b, U, ldu, Z, ldz, status_rw, pass, panel, stage,
                                                               work);
    }
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_CHOL, 2.0 * b * b * b / 3.0, 16.0 * b * b);
    return TSQR_OK;
  }

  tsqr_status shift(double* W, int ldw, int n, double sqrt_m_u) {
    const size_t t0 = tbegin();
    k_shift<<<1, 256, 0, st>>>(W, ldw, n, sqrt_m_u, status);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_SMALL, 0.0, 0.0);
    return TSQR_OK;
  }

  // Cm (n x n) = A B for upper-triangular A, B.  n >= 512 (wide panels, NEXT-f3): a dense DMMA
  // product through the update kernel -- Cm = 0, A <- -A IN PLACE (every caller passes a factor
  // that is dead afterwards: U2, R2), Cm -= (-A) B -- instead of one thread per entry (the
  // triangular zeros stay exact zeros: their products are exact).
  tsqr_status trimul(double* A, int lda, const double* B, int ldb, double* Cm, int ldc, int n) {
    if (n >= 512) {
      k_zero2d<<<grid_1d((int64_t)n * n), 256, 0, st>>>(Cm, ldc, n, n);
      CUDA_TRY(cudaGetLastError());
      launches += 1;
      TRY(copy2d(A, lda, A, lda, n, n, -1.0));
      return update(Cm, ldc, A, lda, B, ldb, n, n, n);
    }
    const size_t t0 = tbegin();
    k_trimul<<<grid_1d((int64_t)n * n), 256, 0, st>>>(A, lda, B, ldb, Cm, ldc, n, status);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_SMALL, 0.0, 0.0);
    return TSQR_OK;
  }

  tsqr_status adapt_decide(const double* U1, const double* Z, const double* Rcol, int ldr, int c0, int b, double tau,
                           double* U2, double* C) {
    const size_t t0 = tbegin();
    k_adapt_decide<<<1, 256, 0, st>>>(U1, b, Z, b, Rcol, ldr, c0, b, tau, U2, b, C, c0 > 0 ? c0 : 1,
                                      const_cast<int*>(status));
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_SMALL, 0.0, 0.0);
    return TSQR_OK;
  }
  tsqr_status adapt_resume() {
    k_adapt_resume<<<1, 32, 0, st>>>(const_cast<int*>(status));
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    return TSQR_OK;
  }

  // Cm (p x q) += A (p x q) B (q x q upper).  q >= 512: A <- -A IN PLACE (the dead C block),
  // then the update kernel Cm -= (-A) B.
  tsqr_status gemm_acc_tri(double* A, int lda, const double* B, int ldb, double* Cm, int ldc, int p, int q) {
    if (q >= 512) {
      TRY(copy2d(A, lda, A, lda, p, q, -1.0));
      return update(Cm, ldc, A, lda, B, ldb, p, q, q);
    }
    const size_t t0 = tbegin();
    k_gemm_acc_tri<<<grid_1d((int64_t)p * q), 256, 0, st>>>(A, lda, B, ldb, Cm, ldc, p, q, status);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_SMALL, 0.0, 0.0);
    return TSQR_OK;
  }

  tsqr_status copy2d(const double* S, int64_t lds, double* D, int64_t ldd, int rows, int cols, double alpha = 1.0) {
    const size_t t0 = tbegin();
    k_copy2d<<<grid_1d((int64_t)rows * cols), 256, 0, st>>>(S, lds, D, ldd, rows, cols, alpha, status);
    CUDA_TRY(cudaGetLastError());
    launches += 1;
    tend(t0, TSQR_KCLASS_SMALL, 0.0, 0.0);
    return TSQR_OK;
  }
};

}  // namespace

// =========================================================================================
// Plan
// =========================================================================================
struct tsqr_plan_s {
  int64_t m = 0;        // local rows
  int64_t m_global = 0; // rows over all ranks (the sCQR shift, Alg. 4 l.2)
  int n = 0, b = 0, k = 0;
  tsqr_algo algo = TSQR_CQR2;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t stream = nullptr;
  // workspace carve-up
  int* status = nullptr;     // int32[16]
  double* part = nullptr;    // split-row partials
  double* W = nullptr;       // Gram block (b x b)
  double* Y = nullptr;       // projection block (b x n) / (n x b)
  double* C = nullptr;       // re-orthogonalisation block C ((j-1)b x b) of mCQR2GS l.7
  double* U1 = nullptr;      // b x b
  double* U2 = nullptr;      // b x b
  double* Z = nullptr;       // b x b inverse
  double* R1 = nullptr;      // n x n (CQR2GS pass 1 / CQR2 temporaries)
  double* R2 = nullptr;      // n x n
  double* cwork = nullptr;   // b x b Cholesky scratch (blocked variant, b >= 128)
  Launcher L;
  Timer timer;
  int64_t allreduces = 0;
  tsqr_status sticky = TSQR_OK;
  // CUDA graph of the whole factorisation, replayed while (A, lda, R, ldr, timing) match
  bool use_graph = true;
  cudaStream_t gstream = nullptr;  // non-blocking stream the graph is captured on / replayed on
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t exec = nullptr;
  double* gA = nullptr;
  double* gR = nullptr;
  int64_t glda = 0;
  int32_t gldr = 0;
  bool gtiming = false;
  // fused reduce + cross-GPU sum: symmetric NCCL window (one p x q slot per rank) + device comm
  void* ar_buf = nullptr;
  ncclWindow_t ar_win = nullptr;
  bool ar_dc_ok = false;
  ncclDevComm ar_dc{};
  // tsqr_factor_host: per-panel "Q_j is final" events (recorded inside the graph as external
  // event nodes while capturing) so the device->host copy of Q_j overlaps the later panels
  bool panel_events = false, gpanel = false;
  double adapt_tau = 8.8817841970012523e-16;  // 2^-50: TSQR_MCQR2GS_ADAPTIVE skip threshold (R-23)
  // NEXT-f1 look-ahead (mCQR2GS): panel j's CholeskyQR chain (Alg. 8 l.6-8) on a second stream
  // while the rest of the trailing update (l.4) runs on the main one
  bool lookahead = false;
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev_fork, ev_join;
  // single-launch cluster path for small problems (cluster_small.cuh)
  bool cluster = false;
  int cl_cs = 0;          // CTAs per cluster (16 or 8)
  ClusterArgs cl_args{};  // fixed part (A, lda, R, ldr filled per call)
  size_t cl_smem = 0;
  std::vector<cudaEvent_t> ev_panel;
  cudaStream_t d2h = nullptr;
  cudaEvent_t ev_d2h = nullptr, ev_fact = nullptr;
  ~tsqr_plan_s() {
    // tsqr_factor is asynchronous: a graph replay (or the host copies of tsqr_factor_host) may
    // still be running and touching the peer window -- drain every stream the plan enqueued on
    // before releasing the window, the device communicator and the graph
    if (gstream) cudaStreamSynchronize(gstream);
    if (d2h) cudaStreamSynchronize(d2h);
    cudaStreamSynchronize(stream);
    if (comm && ar_dc_ok) ncclDevCommDestroy(comm, &ar_dc);
    if (comm && ar_win) ncclCommWindowDeregister(comm, ar_win);
    if (ar_buf) ncclMemFree(ar_buf);
    for (cudaEvent_t e : ev_panel) cudaEventDestroy(e);
    if (ev_d2h) cudaEventDestroy(ev_d2h);
    if (ev_fact) cudaEventDestroy(ev_fact);
    if (d2h) cudaStreamDestroy(d2h);
    if (exec) cudaGraphExecDestroy(exec);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
    if (gstream) cudaStreamDestroy(gstream);
    if (side) cudaStreamSynchronize(side);
    for (cudaEvent_t e : ev_fork) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_join) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
  }
};

namespace {

struct Carve {
  size_t off = 0;
  char* base = nullptr;
  template <typename T>
  T* take(size_t count) {
    size_t at = align_up(off);
    off = at + count * sizeof(T);
    return base ? reinterpret_cast<T*>(base + at) : nullptr;
  }
};

// Largest split-row partial buffer over every projection / Gram the algorithm issues.
size_t max_part_doubles(int64_t m, int n, int b, tsqr_algo algo) {
  size_t mx = atb_part_doubles(m, b, b, true);
  const int k = n / b;
  if (algo == TSQR_CQR2GS || algo == TSQR_CQRGS) {
    for (int j = 0; j + 1 < k; ++j) mx = std::max(mx, atb_part_doubles(m, b, n - (j + 1) * b, false));
  } else if (algo == TSQR_MCQR2GS || algo == TSQR_MCQR2GS_ADAPTIVE) {
    for (int j = 1; j < k; ++j) {
      mx = std::max(mx, atb_part_doubles(m, b, n - j * b, false));
      mx = std::max(mx, atb_part_doubles(m, j * b, b, false));
    }
  }
  return mx;
}

size_t carve(Carve& c, tsqr_plan_s* p, int64_t m, int n, int b, tsqr_algo algo) {
  int* status = c.take<int>(16);
  double* part = c.take<double>(max_part_doubles(m, n, b, algo));
  double* W = c.take<double>((size_t)b * b);
  double* Y = c.take<double>((size_t)b * n);
  double* Cb = c.take<double>((size_t)b * n);  // mCQR2GS l.7 block C (look-ahead: Y stays live meanwhile)
  double* U1 = c.take<double>((size_t)b * b);
  double* U2 = c.take<double>((size_t)b * b);
  double* Z = c.take<double>((size_t)b * b);
  double* R1 = c.take<double>((size_t)n * n);
  double* R2 = c.take<double>((size_t)n * n);
  double* cw = c.take<double>((size_t)b * b);
  if (p) {
    p->status = status; p->part = part; p->W = W; p->Y = Y; p->C = Cb; p->U1 = U1; p->U2 = U2; p->Z = Z;
    p->R1 = R1; p->R2 = R2; p->cwork = cw;
  }
  return align_up(c.off);
}

tsqr_status check_shape(int64_t m_local, int n, int b, tsqr_algo algo) {
  if (m_local < 0 || n < 1 || n > 16384) { set_err("bad m_local/n"); return TSQR_ERR_INVALID_ARG; }
  // TMA tensor coordinates are 32-bit row indices
  if (m_local >= (int64_t(1) << 31)) { set_err("m_local >= 2^31 rows per rank unsupported"); return TSQR_ERR_UNSUPPORTED; }
  if (algo < TSQR_CQR2 || algo > TSQR_MCQR2GS_ADAPTIVE) { set_err("bad algo"); return TSQR_ERR_INVALID_ARG; }
  if (!valid_b(b)) { set_err("panel_b=%d not 16, 32 or a multiple of 64 up to 4096", b); return TSQR_ERR_UNSUPPORTED; }
  if (n % b != 0) { set_err("ragged panels (n %% b != 0) unsupported"); return TSQR_ERR_UNSUPPORTED; }
  if ((algo == TSQR_CQR2 || algo == TSQR_CQR || algo == TSQR_SCQR3 || algo == TSQR_SCQR) && b != n) {
    set_err("CQR/CQR2/sCQR/sCQR3 need b == n");
    return TSQR_ERR_INVALID_ARG;
  }
  return TSQR_OK;
}

// ---- algorithm building blocks (plan-level, include the allreduce) ----
tsqr_status allreduce(tsqr_plan_s* P, double* buf, size_t count) {
  if (P->comm) {  // a 1-rank communicator runs the collective too (it is a copy): the 'nccl' plane under test
    const size_t t0 = P->L.tbegin();
    NCCL_TRY(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, P->comm, P->L.st));
    P->L.tend(t0, TSQR_KCLASS_ALLREDUCE, 0.0, 8.0 * count);
    P->allreduces++;
  } else {
    P->allreduces++;  // counted: one Allreduce of the distributed algorithm (a no-op at P = 1)
  }
  return TSQR_OK;
}

// panel j's columns of Q are final (no later step writes them): signal tsqr_factor_host
tsqr_status panel_done(tsqr_plan_s* P, int j) {
  if (!P->panel_events || j >= (int)P->ev_panel.size()) return TSQR_OK;
  CUDA_TRY(cudaEventRecordWithFlags(P->ev_panel[j], P->L.st, P->timer.capturing ? cudaEventRecordExternal : 0u));
  return TSQR_OK;
}

// W <- allreduce(X^T X), X = m x w slab (standalone split-row Gram)
tsqr_status gram(tsqr_plan_s* P, const double* X, int64_t ldx, int w) {
  TRY(P->L.atb(X, ldx, X, ldx, P->m, w, w, true, P->part, P->W, w, true));
  if (P->L.fuse((int64_t)w * w)) { P->allreduces++; return TSQR_OK; }
  return allreduce(P, P->W, (size_t)w * w);
}

// Cholesky + inverse of the (already allreduced) Gram W, then X <- X U^{-1}.
// (Every Gram is a standalone split-row kernel.  Fusing the next Gram into the TRMM / update
// epilogues saves one read of the panel, but on B200 the fused epilogue Gram ran at about half
// the DMMA efficiency of the standalone kernel and stalled the update's main loop: measured
// at cfg3, fused 149.7 ms/step vs standalone 146.3 ms/step on the same GPU.)
tsqr_status chol_trmm(tsqr_plan_s* P, double* X, int64_t ldx, int w, double* Uout, int ldu, int pass, int panel,
                      int stage) {
  TRY(P->L.chol_inv(P->W, w, w, Uout, ldu, P->Z, w, P->status, pass, panel, stage, P->cwork));
  if (w >= 128 && w % 64 == 0) return P->L.trmm_blocked(X, ldx, P->m, w, P->Z, w, P->cwork);
  return P->L.trmm(X, ldx, P->m, w, P->Z, w);
}

// CholeskyQR of the m x w slab X in place (Alg. 2): U -> Uout (ldu), X <- X U^{-1}
tsqr_status cqr(tsqr_plan_s* P, double* X, int64_t ldx, int w, double* Uout, int ldu, int pass, int panel, int stage) {
  TRY(gram(P, X, ldx, w));
  return chol_trmm(P, X, ldx, w, Uout, ldu, pass, panel, stage);
}

// OUT (p x q, ld p) <- allreduce(L^T Rm)
tsqr_status proj(tsqr_plan_s* P, const double* Lm, int64_t ldl, int p, const double* Rm, int64_t ldr, int q, double* out) {
  TRY(P->L.atb(Lm, ldl, Rm, ldr, P->m, p, q, false, P->part, out, p, true));
  if (P->L.fuse((int64_t)p * q)) { P->allreduces++; return TSQR_OK; }
  return allreduce(P, out, (size_t)p * q);
}

// X (m x q) -= L S (row-local: no communication)
tsqr_status update(tsqr_plan_s* P, double* X, int64_t ldx, const double* Lm, int64_t ldl, const double* S, int lds,
                   int p, int q) {
  return P->L.update(X, ldx, Lm, ldl, S, lds, P->m, p, q);
}

// CQR2 of the first b columns (Alg. 3; Alg. 8 l.1): U1, U2 -> R_11 = U2 U1
// TSQR_MCQR2GS_ADAPTIVE: after the first CholeskyQR of a panel, decide on the device whether the
// repetition is skipped (k_adapt_decide; R-23).  The skipped kernels still launch and return at
// once (status[0] == 7) -- the graph and the allreduce sequence are the same on every call and
// every rank.
bool adaptive(const tsqr_plan_s* P) { return P->algo == TSQR_MCQR2GS_ADAPTIVE; }

tsqr_status cqr2_block(tsqr_plan_s* P, double* A, int64_t lda, int w, double* R, int ldr) {
  TRY(gram(P, A, lda, w));
  TRY(chol_trmm(P, A, lda, w, P->U1, w, 1, 1, 1));
  if (adaptive(P)) TRY(P->L.adapt_decide(P->U1, P->Z, R, ldr, 0, w, P->adapt_tau, P->U2, P->Y));
  TRY(gram(P, A, lda, w));
  TRY(chol_trmm(P, A, lda, w, P->U2, w, 1, 1, 2));
  if (adaptive(P)) TRY(P->L.adapt_resume());
  return P->L.trimul(P->U2, w, P->U1, w, R, ldr, w);
}

// one CQRGS pass (Alg. 7) writing its R into Rp (ld ldr)
tsqr_status cqrgs_pass(tsqr_plan_s* P, double* A, int64_t lda, double* Rp, int ldr, int pass) {
  const int n = P->n, b = P->b, k = P->k;
  for (int j = 0; j < k; ++j) {
    double* Aj = A + (int64_t)j * b * lda;
    TRY(gram(P, Aj, lda, b));                                                  // l.2-3
    // l.4-6: R_jj = U (the Cholesky writes straight into R's diagonal block)
    TRY(chol_trmm(P, Aj, lda, b, Rp + (int64_t)j * b + (int64_t)j * b * ldr, ldr, pass, j + 1, 1));
    if (pass == 2) TRY(panel_done(P, j));
    const int nt = n - (j + 1) * b;
    if (nt > 0) {
      double* At = A + (int64_t)(j + 1) * b * lda;
      TRY(proj(P, Aj, lda, b, At, lda, nt, P->Y));                            // l.7-8
      TRY(update(P, At, lda, Aj, lda, P->Y, b, b, nt));                       // l.9
      TRY(P->L.copy2d(P->Y, b, Rp + (int64_t)j * b + (int64_t)(j + 1) * b * ldr, ldr, b, nt));  // l.10
    }
  }
  return TSQR_OK;
}

tsqr_status run_mcqr2gs(tsqr_plan_s* P, double* A, int64_t lda, double* R, int ldr) {
  const int n = P->n, b = P->b, k = P->k;
  TRY(cqr2_block(P, A, lda, b, R, ldr));                                      // l.1
  TRY(panel_done(P, 0));
  cudaStream_t main_st = P->L.st;
  for (int j = 1; j < k; ++j) {
    double* Ap = A + (int64_t)(j - 1) * b * lda;  // Q_{j-1}
    double* Aj = A + (int64_t)j * b * lda;
    const int Nj = n - j * b;
    // l.3-5: Y = Q_{j-1}^T A_{:,j:k}; A_{:,j:k} -= Q_{j-1} Y; R_{j-1,j:k} = Y
    TRY(proj(P, Ap, lda, b, Aj, lda, Nj, P->Y));
    TRY(P->L.copy2d(P->Y, b, R + (int64_t)(j - 1) * b + (int64_t)j * b * ldr, ldr, b, Nj));
    const bool fork = P->lookahead && Nj > b;
    if (fork) {
      // look-ahead: update panel j's own columns first, then run its CholeskyQR chain
      // (l.6-8) on the side stream while the main stream updates columns j+1..k.  The same
      // kernels on the same operands (every output column's arithmetic is independent of the
      // launch's column range), so the result is bitwise that of the serial schedule.
      TRY(update(P, Aj, lda, Ap, lda, P->Y, b, b, b));
      CUDA_TRY(cudaEventRecord(P->ev_fork[j], main_st));
      CUDA_TRY(cudaStreamWaitEvent(P->side, P->ev_fork[j], 0));
      P->L.st = main_st;
      TRY(update(P, Aj + (int64_t)b * lda, lda, Ap, lda, P->Y + (int64_t)b * b, b, b, Nj - b));
      P->L.st = P->side;
    } else {
      TRY(update(P, Aj, lda, Ap, lda, P->Y, b, b, Nj));
    }
    // l.6: first CQR, panel -> V1, keep U1
    TRY(gram(P, Aj, lda, b));
    TRY(chol_trmm(P, Aj, lda, b, P->U1, b, 1, j + 1, 1));
    const int jb = j * b;
    if (adaptive(P)) TRY(P->L.adapt_decide(P->U1, P->Z, R + (int64_t)jb * ldr, ldr, jb, b, P->adapt_tau, P->U2, P->C));
    // l.7: C = Q_{1:j-1}^T V1 ((j-1)b x b); V1 -= Q_{1:j-1} C
    TRY(proj(P, A, lda, jb, Aj, lda, b, P->C));
    TRY(update(P, Aj, lda, A, lda, P->C, jb, jb, b));
    // l.8: second CQR -> Q_j, U2
    TRY(gram(P, Aj, lda, b));
    TRY(chol_trmm(P, Aj, lda, b, P->U2, b, 1, j + 1, 2));
    if (adaptive(P)) TRY(P->L.adapt_resume());
    TRY(panel_done(P, j));
    // R_jj = U2 U1; R_{1:j-1,j} += C U1  (R-8)
    TRY(P->L.trimul(P->U2, b, P->U1, b, R + (int64_t)jb + (int64_t)jb * ldr, ldr, b));
    TRY(P->L.gemm_acc_tri(P->C, jb, P->U1, b, R + (int64_t)jb * ldr, ldr, jb, b));
    if (fork) {  // join: step j+1 projects against Q_j (side) and the updated columns (main)
      CUDA_TRY(cudaEventRecord(P->ev_join[j], P->side));
      CUDA_TRY(cudaStreamWaitEvent(main_st, P->ev_join[j], 0));
      P->L.st = main_st;
    }
  }
  return TSQR_OK;
}

// Shifted CholeskyQR3 (Alg. 5) of the whole m x n matrix (b == n):
//   [Q1, R1] = sCQR(A)  -- Gram, shift W += s I (Alg. 4 l.2-3), Cholesky, Q1 = A R1^{-1}
//   [Q, R2] = CQR2(Q1)  -- two CholeskyQR passes, R2 = U2 U1
//   R = R2 R1
// Breakdown stages: 1 = the shifted CQR, 2 and 3 = the CQRs of CQR2 (as in the oracle).
constexpr double kUnitRoundoff = 1.1102230246251565e-16;  // 2^-53 (FP64, round to nearest)

tsqr_status scqr(tsqr_plan_s* P, double* A, int64_t lda, double* Uout, int ldu) {
  const int n = P->n;
  TRY(gram(P, A, lda, n));
  TRY(P->L.shift(P->W, n, n, std::sqrt((double)P->m_global) * kUnitRoundoff));
  return chol_trmm(P, A, lda, n, Uout, ldu, 1, 1, 1);
}

tsqr_status run_scqr3(tsqr_plan_s* P, double* A, int64_t lda, double* R, int ldr) {
  const int n = P->n;
  TRY(scqr(P, A, lda, P->R1, n));                       // l.1
  TRY(gram(P, A, lda, n));                              // l.2: CQR2(Q1)
  TRY(chol_trmm(P, A, lda, n, P->U1, n, 1, 1, 2));
  TRY(gram(P, A, lda, n));
  TRY(chol_trmm(P, A, lda, n, P->U2, n, 1, 1, 3));
  TRY(P->L.trimul(P->U2, n, P->U1, n, P->R2, n, n));   //     R2 = U2 U1
  return P->L.trimul(P->R2, n, P->R1, n, R, ldr, n);    // l.3: R = R2 R1
}

// Fused reduce + cross-GPU sum (fused_allreduce.cuh): a symmetric window of 2 halves x nranks
// slots of the largest allreduced block (b x n doubles) and an NCCL device communicator with
// AR_CTAS LSA barriers.  Collective (all ranks call it from tsqr_create in the same order).
// Each rank's wish (TSQR_NCCL_ALLREDUCE=1 disables it; more than 4 ranks need
// TSQR_FUSED_ALLREDUCE=1) and its local allocation are folded into ONE min-allreduce before any
// other collective, so ranks whose environments differ still all take the same path.  A
// 1-rank communicator uses the fused kernel only with TSQR_FUSED_ALLREDUCE=1 (a test knob: it
// puts k_reduce_allreduce under a single-GPU test).  The plan falls back to ncclAllReduce when
// any rank cannot, or when the ranks are not all load/store reachable.
tsqr_status setup_fused_allreduce(tsqr_plan_s* p) {
  const char* env = std::getenv("TSQR_NCCL_ALLREDUCE");
  const char* force = std::getenv("TSQR_FUSED_ALLREDUCE");
  const bool forced = force && std::atoi(force) != 0;
  // validated on 2 and 4 B200s of one box; larger rank counts keep ncclAllReduce unless forced
  const bool want = !(env && std::atoi(env) != 0) && (p->nranks > 1 ? (p->nranks <= 4 || forced) : forced);
  const size_t count = (size_t)p->b * (size_t)p->n;  // cap: Gram b*b, Y b*(n-b), C (n-b)*b <= b*n
  size_t bytes = sizeof(double) * count * (size_t)p->nranks * 2;  // two halves (call parity)
  bytes = (bytes + 4095) / 4096 * 4096;
  int32_t ok = (want && ncclMemAlloc(&p->ar_buf, bytes) == ncclSuccess) ? 1 : 0;
  {
    int32_t* d = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(int32_t), p->stream));
    CUDA_TRY(cudaMemcpyAsync(d, &ok, sizeof(int32_t), cudaMemcpyHostToDevice, p->stream));
    NCCL_TRY(ncclAllReduce(d, d, 1, ncclInt32, ncclMin, p->comm, p->stream));
    CUDA_TRY(cudaMemcpyAsync(&ok, d, sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    CUDA_TRY(cudaFreeAsync(d, p->stream));
  }
  if (!ok) {  // fall back to ncclAllReduce on every rank
    if (p->ar_buf) ncclMemFree(p->ar_buf);
    p->ar_buf = nullptr;
    return TSQR_OK;
  }
  NCCL_TRY(ncclCommWindowRegister(p->comm, p->ar_buf, bytes, &p->ar_win, NCCL_WIN_COLL_SYMMETRIC));
  ncclDevCommRequirements_t req = {};
  req.lsaBarrierCount = AR_CTAS;
  NCCL_TRY(ncclDevCommCreate(p->comm, &req, &p->ar_dc));
  p->ar_dc_ok = true;
  if (p->ar_dc.lsaSize != p->nranks) return TSQR_OK;  // not every rank is peer-addressable
  p->L.ar_on = true;
  p->L.ar_dc = p->ar_dc;
  p->L.ar_win = p->ar_win;
  p->L.ar_nranks = p->nranks;
  p->L.ar_rank = p->rank;
  p->L.ar_cap = (int64_t)count;
  if (const char* fm = std::getenv("TSQR_FUSE_MAX")) p->L.ar_fuse_max = std::atoll(fm);  // A/B knob (same on all ranks)
  return TSQR_OK;
}

// ---- single-launch cluster path (cluster_small.cuh) ----
template <int B>
cudaError_t cluster_config(size_t smem, int cs, int* active) {
  cudaError_t e = cudaFuncSetAttribute(k_cluster_factor<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(k_cluster_factor<B>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(CL_NT); cfg.dynamicSmemBytes = smem;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(active, k_cluster_factor<B>, &cfg);
}

// Decide at tsqr_create whether the plan runs the one-launch cluster kernel: one rank (no
// communicator), b in {16, 32, 64}, and this rank's m x n block (zero-padded to CS equal row
// blocks) plus the reduction buffers fit in the shared memory of CS CTAs.
void setup_cluster_path(tsqr_plan_s* p) {
  const char* env = std::getenv("TSQR_CLUSTER_PATH");
  if ((env && std::atoi(env) == 0) || p->comm || p->m < 1 || !(p->b == 16 || p->b == 32 || p->b == 64) ||
      p->algo == TSQR_MCQR2GS_ADAPTIVE)
    return;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return;
  }
  const int pq = p->b * std::max(p->b, p->n - p->b);
  for (int cs : {16, 8}) {
    const int64_t mr = ((p->m + cs - 1) / cs + 31) / 32 * 32;
    const int ldx = (int)mr + 4;
    const size_t smem = cluster_smem_bytes(p->b, ldx, p->n, pq, (int)p->algo);
    if (smem > (size_t)optin) continue;
    int active = 0;
    cudaError_t e = p->b == 16 ? cluster_config<16>(smem, cs, &active)
                  : p->b == 32 ? cluster_config<32>(smem, cs, &active)
                               : cluster_config<64>(smem, cs, &active);
    if (e != cudaSuccess || active < 1) { (void)cudaGetLastError(); continue; }
    ClusterArgs& a = p->cl_args;
    a.R1 = p->R1; a.R2 = p->R2; a.status = p->status; a.m = p->m; a.n = p->n; a.algo = (int)p->algo;
    a.mr = (int)mr; a.ldx = ldx; a.pq = pq;
    a.shift_scale = std::sqrt((double)p->m_global) * 1.1102230246251565e-16;  // sqrt(m) u (Alg. 4 l.2)
    p->cl_cs = cs; p->cl_smem = smem; p->cluster = true;
    return;
  }
}

int64_t reductions_of(tsqr_algo algo, int k) {
  switch (algo) {
    case TSQR_CQR: case TSQR_SCQR: return 1;
    case TSQR_CQR2: return 2;
    case TSQR_SCQR3: return 3;
    case TSQR_CQRGS: return 2 * k - 1;
    default: return k == 1 ? 2 : 4 * k - 2;  // CQR2GS, mCQR2GS (k = 1: CholeskyQR2)
  }
}

tsqr_status launch_cluster(tsqr_plan_s* P, double* A, int64_t lda, double* R, int ldr) {
  ClusterArgs a = P->cl_args;
  a.A = A; a.lda = lda; a.R = R; a.ldr = ldr;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->cl_cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(P->cl_cs); cfg.blockDim = dim3(CL_NT); cfg.dynamicSmemBytes = P->cl_smem;
  cfg.stream = P->L.st; cfg.attrs = at; cfg.numAttrs = 1;
  const size_t t0 = P->L.tbegin();
  cudaError_t e = P->b == 16 ? cudaLaunchKernelEx(&cfg, k_cluster_factor<16>, a)
                : P->b == 32 ? cudaLaunchKernelEx(&cfg, k_cluster_factor<32>, a)
                             : cudaLaunchKernelEx(&cfg, k_cluster_factor<64>, a);
  CUDA_TRY(e);
  P->L.launches += 1;
  P->L.tend(t0, TSQR_KCLASS_CLUSTER, 4.0 * (double)P->m * P->n * P->n, 16.0 * (double)P->m * P->n);
  P->allreduces = reductions_of(P->algo, P->k);
  for (int j = 0; j < P->k; ++j) TRY(panel_done(P, j));
  return TSQR_OK;
}

const char* status_names[] = {"TSQR_OK", "TSQR_ERR_INVALID_ARG", "TSQR_ERR_UNSUPPORTED", "TSQR_ERR_CUDA",
                              "TSQR_ERR_NCCL", "TSQR_ERR_BREAKDOWN", "TSQR_ERR_WORKSPACE"};

}  // namespace

// =========================================================================================
// C ABI
// =========================================================================================
extern "C" {

const char* tsqr_status_string(tsqr_status s) {
  if ((int)s < 0 || (int)s > 6) return "TSQR_UNKNOWN";
  return status_names[(int)s];
}

const char* tsqr_last_error(void) { return g_err; }

size_t tsqr_workspace_bytes(int64_t m_local, int32_t n, int32_t panel_b, int32_t nranks, tsqr_algo algo) {
  (void)nranks;
  if (check_shape(m_local, n, panel_b, algo) != TSQR_OK) return 0;
  Carve c;
  return carve(c, nullptr, m_local, n, panel_b, algo);
}

tsqr_status tsqr_create(tsqr_plan_t* plan, int64_t m_local, int32_t n, int32_t panel_b, void* nccl_comm,
                        tsqr_algo algo, void* cuda_stream, void* workspace, size_t workspace_bytes) {
  if (!plan) { set_err("plan == NULL"); return TSQR_ERR_INVALID_ARG; }
  *plan = nullptr;
  tsqr_status st = check_shape(m_local, n, panel_b, algo);
  size_t need = st == TSQR_OK ? tsqr_workspace_bytes(m_local, n, panel_b, 1, algo) : 0;
  if (st == TSQR_OK && (!workspace || workspace_bytes < need || (reinterpret_cast<uintptr_t>(workspace) % kAlign))) {
    set_err("workspace NULL, smaller than %zu bytes or not 256-byte aligned", need);
    st = TSQR_ERR_WORKSPACE;
  }
  ncclComm_t comm = reinterpret_cast<ncclComm_t>(nccl_comm);
  int nranks = 1, rank = 0;
  int64_t m_global = m_local;
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  if (comm) {
    NCCL_TRY(ncclCommCount(comm, &nranks));
    NCCL_TRY(ncclCommUserRank(comm, &rank));
    // collective argument validation: [n, b, algo, valid] min/max and sum(m_local)
    int64_t h[6] = {n, panel_b, (int64_t)algo, st == TSQR_OK ? 1 : 0, m_local, 0};
    int64_t* d = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), 3 * 6 * sizeof(int64_t), stream));
    CUDA_TRY(cudaMemcpyAsync(d, h, sizeof(h), cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(d + 6, h, sizeof(h), cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaMemcpyAsync(d + 12, h, sizeof(h), cudaMemcpyHostToDevice, stream));
    NCCL_TRY(ncclGroupStart());
    NCCL_TRY(ncclAllReduce(d, d, 6, ncclInt64, ncclMin, comm, stream));
    NCCL_TRY(ncclAllReduce(d + 6, d + 6, 6, ncclInt64, ncclMax, comm, stream));
    NCCL_TRY(ncclAllReduce(d + 12, d + 12, 6, ncclInt64, ncclSum, comm, stream));
    NCCL_TRY(ncclGroupEnd());
    int64_t r[18];
    CUDA_TRY(cudaMemcpyAsync(r, d, sizeof(r), cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    CUDA_TRY(cudaFreeAsync(d, stream));
    if (r[0] != r[6] || r[1] != r[7] || r[2] != r[8]) {
      set_err("ranks disagree on n / panel_b / algo");
      return TSQR_ERR_INVALID_ARG;
    }
    if (r[3] == 0) {
      if (st == TSQR_OK) { set_err("another rank rejected its arguments"); st = TSQR_ERR_INVALID_ARG; }
      return st;
    }
    if (r[12 + 4] < n) { set_err("global m < n"); return TSQR_ERR_INVALID_ARG; }
    m_global = r[12 + 4];
  } else {
    if (st != TSQR_OK) return st;
    if (m_local < n) { set_err("m < n"); return TSQR_ERR_INVALID_ARG; }
  }
  if (st != TSQR_OK) return st;
  tsqr_plan_s* p = new (std::nothrow) tsqr_plan_s();
  if (!p) return TSQR_ERR_INVALID_ARG;
  p->m = m_local; p->m_global = m_global; p->n = n; p->b = panel_b; p->k = n / panel_b; p->algo = algo;
  p->comm = comm; p->nranks = nranks; p->rank = rank; p->stream = stream;
  Carve c;
  c.base = reinterpret_cast<char*>(workspace);
  carve(c, p, m_local, n, panel_b, algo);
  p->L.st = stream;
  p->L.status = p->status;
  p->L.timer = &p->timer;
  if (comm) {
    const tsqr_status fs = setup_fused_allreduce(p);
    if (fs != TSQR_OK) {
      delete p;
      return fs;
    }
  }
  setup_cluster_path(p);
  {
    const char* la = std::getenv("TSQR_LOOKAHEAD");
    if (la && std::atoi(la) != 0 && tsqr_set_lookahead(p, 1) != TSQR_OK) {
      delete p;
      return TSQR_ERR_CUDA;
    }
  }
  *plan = p;
  return TSQR_OK;
}

static tsqr_status enqueue_factor(tsqr_plan_t P, double* A, int64_t lda, double* R, int32_t ldr) {
  P->L.launches = 0;
  P->allreduces = 0;
  P->sticky = TSQR_OK;
  if (P->cluster) return launch_cluster(P, A, lda, R, ldr);  // clears the status word itself
  CUDA_TRY(cudaMemsetAsync(P->status, 0, 16 * sizeof(int), P->L.st));
  k_zero2d<<<grid_1d((int64_t)P->n * P->n), 256, 0, P->L.st>>>(R, ldr, P->n, P->n);
  CUDA_TRY(cudaGetLastError());
  P->L.launches++;
  const int n = P->n, b = P->b;
  tsqr_status s = TSQR_OK;
  switch (P->algo) {
    case TSQR_CQR:
      s = cqr(P, A, lda, n, R, ldr, 1, 1, 1);
      break;
    case TSQR_CQR2:
      s = cqr2_block(P, A, lda, n, R, ldr);
      break;
    case TSQR_CQRGS:
      s = cqrgs_pass(P, A, lda, R, ldr, 1);
      break;
    case TSQR_CQR2GS:
      if (P->k == 1) {  // b == n: CQR2GS falls back to CholeskyQR2
        s = cqr2_block(P, A, lda, n, R, ldr);
        break;
      }
      k_zero2d<<<grid_1d((int64_t)n * n), 256, 0, P->L.st>>>(P->R1, n, n, n);
      k_zero2d<<<grid_1d((int64_t)n * n), 256, 0, P->L.st>>>(P->R2, n, n, n);
      P->L.launches += 2;
      s = cqrgs_pass(P, A, lda, P->R1, n, 1);
      if (s == TSQR_OK) s = cqrgs_pass(P, A, lda, P->R2, n, 2);
      if (s == TSQR_OK) s = P->L.trimul(P->R2, n, P->R1, n, R, ldr, n);
      break;
    case TSQR_MCQR2GS:
    case TSQR_MCQR2GS_ADAPTIVE:
      s = run_mcqr2gs(P, A, lda, R, ldr);
      break;
    case TSQR_SCQR3:
      s = run_scqr3(P, A, lda, R, ldr);
      break;
    case TSQR_SCQR:
      s = scqr(P, A, lda, R, ldr);
      break;
  }
  (void)b;
  return s;
}

tsqr_status tsqr_factor(tsqr_plan_t P, double* A, int64_t lda, double* R, int32_t ldr) {
  if (!P) { set_err("plan == NULL"); return TSQR_ERR_INVALID_ARG; }
  if ((!A && P->m > 0) || !R || lda < std::max<int64_t>(1, P->m) || ldr < P->n ||
      (reinterpret_cast<uintptr_t>(A) & 7u) || (reinterpret_cast<uintptr_t>(R) & 7u)) {
    set_err("bad A/R pointer or leading dimension");
    return TSQR_ERR_INVALID_ARG;
  }
  P->sticky = TSQR_OK;
  if (P->use_graph && !P->gstream) {
    if (cudaStreamCreateWithFlags(&P->gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&P->ev_out, cudaEventDisableTiming) != cudaSuccess) {
      (void)cudaGetLastError();
      P->use_graph = false;
    }
  }
  if (!P->use_graph) {
    if (P->timer.graph_recs) P->timer.drop_recs();
    P->L.st = P->stream;
    P->sticky = enqueue_factor(P, A, lda, R, ldr);
    return P->sticky;
  }
  // the graph runs on the plan's own stream, ordered after / before the caller's stream
  CUDA_TRY(cudaEventRecord(P->ev_in, P->stream));
  CUDA_TRY(cudaStreamWaitEvent(P->gstream, P->ev_in, 0));
  const bool same = P->exec && P->gA == A && P->glda == lda && P->gR == R && P->gldr == ldr &&
                    P->gtiming == P->timer.on && P->gpanel == P->panel_events;
  if (!same) {
    // capture the whole factorisation (kernels, NCCL allreduces, timing events) once
    if (P->exec) {
      CUDA_TRY(cudaStreamSynchronize(P->gstream));
      cudaGraphExecDestroy(P->exec);
      P->exec = nullptr;
    }
    P->timer.drop_recs();
    CUDA_TRY(cudaStreamBeginCapture(P->gstream, cudaStreamCaptureModeThreadLocal));
    P->L.st = P->gstream;
    P->timer.capturing = true;
    tsqr_status s = enqueue_factor(P, A, lda, R, ldr);
    P->timer.capturing = false;
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(P->gstream, &g);
    if (s != TSQR_OK || ce != cudaSuccess || !g) {
      if (g) cudaGraphDestroy(g);
      (void)cudaGetLastError();
      if (s == TSQR_OK) set_err("graph capture failed: %s", cudaGetErrorString(ce));
      // fall back to eager enqueueing for this plan
      P->use_graph = false;
      P->timer.drop_recs();
      P->L.st = P->stream;
      P->sticky = enqueue_factor(P, A, lda, R, ldr);
      return P->sticky;
    }
    cudaError_t ie = cudaGraphInstantiate(&P->exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {
      P->exec = nullptr;
      set_err("cudaGraphInstantiate failed: %s", cudaGetErrorString(ie));
      return TSQR_ERR_CUDA;
    }
    P->timer.graph_recs = P->timer.on;
    P->gA = A; P->glda = lda; P->gR = R; P->gldr = ldr; P->gtiming = P->timer.on; P->gpanel = P->panel_events;
  }
  CUDA_TRY(cudaGraphLaunch(P->exec, P->gstream));
  CUDA_TRY(cudaEventRecord(P->ev_out, P->gstream));
  CUDA_TRY(cudaStreamWaitEvent(P->stream, P->ev_out, 0));
  if (P->timer.on) P->timer.pending++;
  return TSQR_OK;
}

tsqr_status tsqr_set_graph(tsqr_plan_t P, int32_t enable) {
  if (!P) return TSQR_ERR_INVALID_ARG;
  P->use_graph = enable != 0;
  if (!P->use_graph && P->exec) {
    CUDA_TRY(cudaStreamSynchronize(P->gstream));
    cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
    P->timer.drop_recs();
  }
  return TSQR_OK;
}

tsqr_status tsqr_wait(tsqr_plan_t P, tsqr_breakdown_info* info) {
  if (!P) { set_err("plan == NULL"); return TSQR_ERR_INVALID_ARG; }
  if (P->sticky != TSQR_OK) return P->sticky;
  int h[16];
  CUDA_TRY(cudaMemcpyAsync(h, P->status, sizeof(h), cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  if (P->timer.on) P->timer.harvest();  // fold this factorisation's events in before a replay reuses them
  if (P->comm) {
    ncclResult_t async_err = ncclSuccess;
    NCCL_TRY(ncclCommGetAsyncError(P->comm, &async_err));
    if (async_err != ncclSuccess) { set_err("NCCL async error: %s", ncclGetErrorString(async_err)); return TSQR_ERR_NCCL; }
  }
  if (h[0] == 5) {
    if (info) {
      info->pass = h[1]; info->panel = h[2]; info->stage = h[3]; info->pivot = h[4];
      double v;
      std::memcpy(&v, &h[6], sizeof(double));
      info->pivot_value = v;
    }
    return TSQR_ERR_BREAKDOWN;
  }
  if (info) std::memset(info, 0, sizeof(*info));
  return TSQR_OK;
}

tsqr_status tsqr_last_counts(tsqr_plan_t P, int64_t* allreduces, int64_t* launches) {
  if (!P) return TSQR_ERR_INVALID_ARG;
  if (allreduces) *allreduces = P->allreduces;
  if (launches) *launches = P->L.launches;
  return TSQR_OK;
}

tsqr_status tsqr_factor_host(tsqr_plan_t P, double* A_host, int64_t lda_host, double* R_host, int32_t ldr_host,
                             double* A_dev, int64_t lda_dev, double* R_dev, int32_t ldr_dev) {
  if (!P || (P->m > 0 && (!A_host || !A_dev)) || !R_host || !R_dev || lda_host < std::max<int64_t>(1, P->m) ||
      ldr_host < P->n) {
    set_err("bad host/device buffers");
    return TSQR_ERR_INVALID_ARG;
  }
  const size_t rowb = sizeof(double) * (size_t)P->m;
  // the panel-wise methods finalise Q one panel at a time: copy Q_j back on a second stream as
  // soon as it is final, overlapping the remaining panels (H2D has to complete first: the first
  // projection reads every column)
  const bool by_panel = P->m > 0 && P->k > 1 && !P->cluster &&  // one launch: nothing to overlap
                        (P->algo == TSQR_MCQR2GS || P->algo == TSQR_MCQR2GS_ADAPTIVE || P->algo == TSQR_CQR2GS);
  if (!P->d2h) {
    CUDA_TRY(cudaStreamCreateWithFlags(&P->d2h, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&P->ev_d2h, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&P->ev_fact, cudaEventDisableTiming));
  }
  if (by_panel && (int)P->ev_panel.size() < P->k) {
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    while ((int)P->ev_panel.size() < P->k) {
      cudaEvent_t e;
      CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      P->ev_panel.push_back(e);
    }
  }
  if (P->m > 0)
    CUDA_TRY(cudaMemcpy2DAsync(A_dev, sizeof(double) * lda_dev, A_host, sizeof(double) * lda_host, rowb, P->n,
                               cudaMemcpyHostToDevice, P->stream));
  P->panel_events = by_panel;
  const tsqr_status fs = tsqr_factor(P, A_dev, lda_dev, R_dev, ldr_dev);
  P->panel_events = false;
  TRY(fs);
  CUDA_TRY(cudaEventRecord(P->ev_fact, P->stream));
  if (by_panel) {
    for (int j = 0; j < P->k; ++j) {
      CUDA_TRY(cudaStreamWaitEvent(P->d2h, P->ev_panel[j], 0));
      CUDA_TRY(cudaMemcpy2DAsync(A_host + (int64_t)j * P->b * lda_host, sizeof(double) * lda_host,
                                 A_dev + (int64_t)j * P->b * lda_dev, sizeof(double) * lda_dev, rowb, P->b,
                                 cudaMemcpyDeviceToHost, P->d2h));
    }
    CUDA_TRY(cudaStreamWaitEvent(P->d2h, P->ev_fact, 0));
  } else {
    CUDA_TRY(cudaStreamWaitEvent(P->d2h, P->ev_fact, 0));
    if (P->m > 0)
      CUDA_TRY(cudaMemcpy2DAsync(A_host, sizeof(double) * lda_host, A_dev, sizeof(double) * lda_dev, rowb, P->n,
                                 cudaMemcpyDeviceToHost, P->d2h));
  }
  CUDA_TRY(cudaMemcpy2DAsync(R_host, sizeof(double) * ldr_host, R_dev, sizeof(double) * ldr_dev,
                             sizeof(double) * P->n, P->n, cudaMemcpyDeviceToHost, P->d2h));
  CUDA_TRY(cudaEventRecord(P->ev_d2h, P->d2h));
  CUDA_TRY(cudaStreamWaitEvent(P->stream, P->ev_d2h, 0));  // tsqr_wait on the plan stream covers the copies
  return TSQR_OK;
}

tsqr_status tsqr_set_timing(tsqr_plan_t P, int32_t enable) {
  if (!P) return TSQR_ERR_INVALID_ARG;
  P->timer.on = enable != 0;
  return TSQR_OK;
}

tsqr_status tsqr_timing_reset(tsqr_plan_t P) {
  if (!P) return TSQR_ERR_INVALID_ARG;
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->timer.reset();
  return TSQR_OK;
}

tsqr_status tsqr_timing(tsqr_plan_t P, int32_t kclass, double* ms, int64_t* launches, double* flops, double* bytes) {
  if (!P || kclass < 0 || kclass >= TSQR_KCLASS_COUNT) return TSQR_ERR_INVALID_ARG;
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  P->timer.harvest();
  if (ms) *ms = P->timer.ms[kclass];
  if (launches) *launches = P->timer.cnt[kclass];
  if (flops) *flops = P->timer.fl[kclass];
  if (bytes) *bytes = P->timer.by[kclass];
  return TSQR_OK;
}

tsqr_status tsqr_data_plane(tsqr_plan_t P, int32_t* plane) {
  if (!P || !plane) return TSQR_ERR_INVALID_ARG;
  *plane = P->L.ar_on ? TSQR_PLANE_FUSED : (P->comm ? TSQR_PLANE_NCCL : TSQR_PLANE_LOCAL);
  return TSQR_OK;
}

tsqr_status tsqr_set_lookahead(tsqr_plan_t P, int32_t enable) {
  if (!P) return TSQR_ERR_INVALID_ARG;
  // mCQR2GS only (the adaptive variant's skip mark is a plan-wide status word the concurrent
  // trailing update would see); the streaming path only
  const bool on = enable != 0 && P->algo == TSQR_MCQR2GS && !P->cluster && P->k > 2;
  if (on && !P->side) {
    CUDA_TRY(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking));
    for (int j = 0; j < P->k; ++j) {
      cudaEvent_t a, b;
      CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      P->ev_fork.push_back(a);
      P->ev_join.push_back(b);
    }
  }
  if (on != P->lookahead && P->exec) {  // the schedule is baked into the captured graph
    CUDA_TRY(cudaStreamSynchronize(P->gstream));
    cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
  }
  P->lookahead = on;
  return TSQR_OK;
}

tsqr_status tsqr_set_adapt_tau(tsqr_plan_t P, double tau) {
  if (!P || !(tau >= 0.0)) return TSQR_ERR_INVALID_ARG;
  if (tau != P->adapt_tau && P->exec) {  // the threshold is a kernel argument of the captured graph
    CUDA_TRY(cudaStreamSynchronize(P->gstream));
    cudaGraphExecDestroy(P->exec);
    P->exec = nullptr;
  }
  P->adapt_tau = tau;
  return TSQR_OK;
}

tsqr_status tsqr_skipped_panels(tsqr_plan_t P, int32_t* panels) {
  if (!P || !panels) return TSQR_ERR_INVALID_ARG;
  int h[16];
  CUDA_TRY(cudaMemcpyAsync(h, P->status, sizeof(h), cudaMemcpyDeviceToHost, P->stream));
  CUDA_TRY(cudaStreamSynchronize(P->stream));
  *panels = P->algo == TSQR_MCQR2GS_ADAPTIVE ? h[9] : 0;
  return TSQR_OK;
}

tsqr_status tsqr_exec_path(tsqr_plan_t P, int32_t* path) {
  if (!P || !path) return TSQR_ERR_INVALID_ARG;
  *path = P->cluster ? TSQR_PATH_CLUSTER : TSQR_PATH_STREAM;
  return TSQR_OK;
}

tsqr_status tsqr_destroy(tsqr_plan_t P) {
  delete P;
  return TSQR_OK;
}

tsqr_status tsqr_nccl_unique_id(void* id128) {
  if (!id128) return TSQR_ERR_INVALID_ARG;
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return TSQR_OK;
}

tsqr_status tsqr_nccl_comm_init(void** comm, int32_t nranks, int32_t rank, const void* id128, int32_t device) {
  if (!comm || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return TSQR_ERR_INVALID_ARG;
  CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  NCCL_TRY(ncclCommInitRank(&c, nranks, id, rank));
  *comm = c;
  return TSQR_OK;
}

tsqr_status tsqr_nccl_comm_destroy(void* comm) {
  if (!comm) return TSQR_OK;
  NCCL_TRY(ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)));
  return TSQR_OK;
}

// ---- step-level entry points (single GPU) ----
// One scratch buffer per device (the split-row partials of tsqr_gram / tsqr_proj and the
// blocked Cholesky's work matrix).  Growing it synchronises the device first, so no kernel
// still reading the old buffer on any stream can see it freed; released at process exit.
namespace {
struct Scratch {
  static constexpr int kMaxDev = 64;
  double* part[kMaxDev] = {};
  size_t cap[kMaxDev] = {};
  ~Scratch() {
    for (int d = 0; d < kMaxDev; ++d)
      if (part[d]) cudaFree(part[d]);  // errors ignored: the context may already be gone
  }
};
Scratch g_scratch;

tsqr_status scratch(size_t doubles, cudaStream_t st, double** out) {
  (void)st;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= Scratch::kMaxDev) { set_err("device index %d out of range", dev); return TSQR_ERR_INVALID_ARG; }
  if (g_scratch.cap[dev] < doubles) {
    if (g_scratch.part[dev]) {
      CUDA_TRY(cudaDeviceSynchronize());
      CUDA_TRY(cudaFree(g_scratch.part[dev]));
      g_scratch.part[dev] = nullptr;
      g_scratch.cap[dev] = 0;
    }
    CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&g_scratch.part[dev]), doubles * sizeof(double)));
    g_scratch.cap[dev] = doubles;
  }
  *out = g_scratch.part[dev];
  return TSQR_OK;
}
}  // namespace

tsqr_status tsqr_gram(const double* X, int64_t ldx, int64_t m, int32_t b, double* W, int32_t ldw, void* cuda_stream) {
  if (!W || (m > 0 && !X) || b < 1 || b > 4096 || ldx < std::max<int64_t>(1, m) || ldw < b) return TSQR_ERR_INVALID_ARG;
  Launcher L;
  L.st = reinterpret_cast<cudaStream_t>(cuda_stream);
  double* part;
  TRY(scratch(atb_part_doubles(m, b, b, true), L.st, &part));
  return L.atb(X, ldx, X, ldx, m, b, b, true, part, W, ldw);
}

tsqr_status tsqr_proj(const double* Lm, int64_t ldl, const double* Rm, int64_t ldr, int64_t m, int32_t p, int32_t q,
                      double* OUT, int32_t ldo, void* cuda_stream) {
  if (!OUT || (m > 0 && (!Lm || !Rm)) || p < 1 || q < 1 || p > 4096 || q > 4096 || ldl < std::max<int64_t>(1, m) ||
      ldr < std::max<int64_t>(1, m) || ldo < p)
    return TSQR_ERR_INVALID_ARG;
  Launcher L;
  L.st = reinterpret_cast<cudaStream_t>(cuda_stream);
  double* part;
  TRY(scratch(atb_part_doubles(m, p, q, false), L.st, &part));
  return L.atb(Lm, ldl, Rm, ldr, m, p, q, false, part, OUT, ldo);
}

tsqr_status tsqr_update(double* X, int64_t ldx, const double* Lm, int64_t ldl, const double* S, int32_t lds, int64_t m,
                        int32_t p, int32_t q, void* cuda_stream) {
  if ((m > 0 && (!X || !Lm)) || !S || p < 1 || q < 1 || p > 4096 || q > 4096 || ldx < std::max<int64_t>(1, m) ||
      ldl < std::max<int64_t>(1, m) || lds < p)
    return TSQR_ERR_INVALID_ARG;
  Launcher L;
  L.st = reinterpret_cast<cudaStream_t>(cuda_stream);
  return L.update(X, ldx, Lm, ldl, S, lds, m, p, q);
}

tsqr_status tsqr_chol_inv(const double* W, int32_t ldw, int32_t b, double* U, int32_t ldu, double* Z, int32_t ldz,
                          int32_t* status_dev, void* cuda_stream) {
  if (!W || !U || !Z || !status_dev || b < 1 || b > 4096 || ldw < b || ldu < b || ldz < b) return TSQR_ERR_INVALID_ARG;
  if (b > 256 && b % 64 != 0) return TSQR_ERR_UNSUPPORTED;
  Launcher L;
  L.st = reinterpret_cast<cudaStream_t>(cuda_stream);
  double* work = nullptr;
  if (b >= 128) TRY(scratch((size_t)b * b, L.st, &work));
  return L.chol_inv(W, ldw, b, U, ldu, Z, ldz, status_dev, 1, 1, 1, work);
}

tsqr_status tsqr_trmm(double* X, int64_t ldx, int64_t m, int32_t b, const double* Z, int32_t ldz, void* cuda_stream) {
  if ((m > 0 && !X) || !Z || ldx < std::max<int64_t>(1, m) || ldz < b) return TSQR_ERR_INVALID_ARG;
  if (!valid_b(b)) return TSQR_ERR_UNSUPPORTED;
  Launcher L;
  L.st = reinterpret_cast<cudaStream_t>(cuda_stream);
  return L.trmm(X, ldx, m, b, Z, ldz);
}

}  // extern "C"
