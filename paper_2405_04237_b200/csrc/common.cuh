// common.cuh -- PTX helpers shared by the sm_100a kernels of libtsqr.
//
// FP64 contractions use mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, the B200 FP64 tensor path;
// tcgen05.mma has no f64 kind).  Fragments (lane = 4*gid + tig):
//   A (8x4, row): a = A[gid][tig]     B (4x8, col): b = B[tig][gid]
//   C (8x8):      c0, c1 = C[gid][2*tig + {0, 1}]
// Operand tiles are staged in shared memory column by column with a padded leading
// dimension LDT == 4 (mod 16) doubles, which makes every fragment load used here
// bank-conflict free (both 16-lane phases of an 8-byte access hit 16 distinct banks).
#pragma once
#include <cuda.h>  // CUtensorMap (type only; the driver entry point is fetched at run time)
#include <cuda_runtime.h>

#include <cstdint>

namespace tsqr {

constexpr int NCW = 8;                    // consumer (math) warps per CTA
constexpr int NTHR = 32 * (NCW + 1);      // + one producer warp
constexpr int PRODUCER = NCW;             // warp index of the producer

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes));
}

// ---- mbarrier (CTA scope) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed (.noinc: the
// barrier's expected count must include this arrival)
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// expect `bytes` of asynchronous (TMA) transactions on `bar` and arrive once
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// TMA bulk copy global -> shared (contiguous bytes, 16-byte aligned, size % 16 == 0);
// completes `bytes` transactions on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 2-D TMA tensor copy of one box (coordinates: x = row, y = column of the column-major
// matrix described by `map`) into shared memory; out-of-bounds elements are zero-filled and
// the full box is counted against the mbarrier's expected transaction bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// 2-D TMA tensor store of one box from shared memory (bulk-group completion); rows / columns
// outside the tensor are not written
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
// 2-D TMA tensor reduce-add of one box from shared memory into global (X[box] += smem box,
// done by the L2; FLOAT64 add is supported on sm_100a -- verified on B200)
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void tma_prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// order this thread's generic-proxy shared-memory writes before later async-proxy accesses
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// named barrier among the NCW consumer warps only (the producer never joins)
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(NCW * 32) : "memory"); }

__device__ __forceinline__ bool failed(const int* status) {
  return status != nullptr && *((volatile const int*)status) != 0;
}

// Producer warp: stage a (TR rows) x (NCOLS columns) tile of column-major G (leading
// dimension ld) starting at (row0, col0) into sm[c*LDT + r] with cp.async.  Rows >= m and
// columns >= colmax are zero-filled (short source size), so ragged tails add nothing.
// V16: 16-byte copies (ld even, G 16-byte aligned), else 8-byte copies.
template <int TR, int LDT, bool V16, int NCOLS>
__device__ __forceinline__ void produce_tile(double* sm, const double* __restrict__ G, int64_t ld, int64_t row0,
                                             int64_t m, int col0, int colmax, int lane) {
#pragma unroll 4
  for (int c = 0; c < NCOLS; ++c) {
    const int gc = col0 + c;
    const bool cv = gc < colmax;
    const double* src = G + (int64_t)(cv ? gc : 0) * ld;
    if (V16) {
#pragma unroll
      for (int rp = lane; rp < TR / 2; rp += 32) {
        const int64_t r = row0 + 2 * rp;
        const int64_t rem = cv ? (m - r) : 0;
        const int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
        cp_async16(sm + c * LDT + 2 * rp, bytes ? (const void*)(src + r) : (const void*)G, bytes);
      }
    } else {
#pragma unroll
      for (int rr = lane; rr < TR; rr += 32) {
        const int64_t r = row0 + rr;
        const int bytes = (cv && r < m) ? 8 : 0;
        cp_async8(sm + c * LDT + rr, bytes ? (const void*)(src + r) : (const void*)G, bytes);
      }
    }
  }
}

// Producer warp, TMA path (ld even, G 16-byte aligned): one cp.async.bulk per column (the
// column's rows are contiguous), issued by the 32 lanes, completing on `bar` which receives
// exactly one arrive.expect_tx per call.  A ragged tail (rows past m, an odd last row) and
// columns >= colmax are written with generic stores (zeros / the odd element) before the
// arrive, followed by a proxy fence.
template <int TR, int LDT, int NCOLS>
__device__ __forceinline__ void produce_tile_tma(double* sm, const double* __restrict__ G, int64_t ld, int64_t row0,
                                                 int64_t m, int col0, int colmax, int lane, uint64_t* bar) {
  int64_t rows64 = m - row0;
  const int rows = rows64 <= 0 ? 0 : (rows64 >= TR ? TR : (int)rows64);
  const int rows2 = rows & ~1;
  int ncv = colmax - col0;
  ncv = ncv < 0 ? 0 : (ncv > NCOLS ? NCOLS : ncv);
  if (rows < TR || ncv < NCOLS) {
    for (int c = lane; c < NCOLS; c += 32) {
      double* d = sm + c * LDT;
      if (c < ncv) {
        const double* src = G + (int64_t)(col0 + c) * ld + row0;
        for (int r = rows2; r < TR; ++r) d[r] = (r < rows) ? src[r] : 0.0;
      } else {
        for (int r = 0; r < TR; ++r) d[r] = 0.0;
      }
    }
    fence_proxy_async();
  }
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(ncv * rows2 * 8));
  __syncwarp();
  if (rows2 > 0)
    for (int c = lane; c < ncv; c += 32)
      bulk_g2s(sm + c * LDT, G + (int64_t)(col0 + c) * ld + row0, (uint32_t)(rows2 * 8), bar);
}

// Upper 8x8 block t (0..35) of a 64x64 Gram: (bi, bj) with bi <= bj, column-major order.
__device__ __forceinline__ void upper_block(int t, int& bi, int& bj) {
  int j = 0;
  while (t > j) {
    t -= j + 1;
    ++j;
  }
  bi = t;
  bj = j;
}

}  // namespace tsqr
