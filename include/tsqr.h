/*
 * tsqr.h -- C ABI of libtsqr: distributed FP64 QR of a tall-and-skinny matrix on
 * B200 GPUs, following arXiv 2405.04237 (Mijic, Kaushik, Davidovic).
 *
 * Problem: A = Q R with A in R^{m x n}, m >= n, Q with orthonormal
 * columns, R upper triangular.  A is distributed in 1-D block rows, one block per
 * GPU (Fig. distA); Q stays distributed and overwrites A in place
 * (P:142); R is computed redundantly and replicated on every rank.
 *
 * Methods (TSQR_ALGO):
 *   TSQR_CQR2     CholeskyQR2: two CholeskyQR passes, R = R2 R1     (Alg. 3)
 *   TSQR_CQR2GS   CholeskyQR2 with block Gram-Schmidt: two passes of the
 *                 distributed CQRGS (Alg. 7), R = R2 R1
 *   TSQR_MCQR2GS  the paper's modified CQR2GS (Alg. 8)
 *   TSQR_CQR      single CholeskyQR pass (Alg. 2)        -- tests
 *   TSQR_CQRGS    single CQRGS pass (Alg. 7)                         -- tests
 *   TSQR_SCQR3    shifted CholeskyQR3 (Alg. 5): sCQR (Alg. 4, P:236-246:
 *                 W = A^T A + s I, s = sqrt(m) u ||A||_F^2, m the global row count,
 *                 u = 2^-53) followed by CQR2; R = R2 R1.  b == n.  3 allreduces.
 *   TSQR_SCQR     single shifted CholeskyQR pass (Alg. 4)           -- tests
 *   TSQR_MCQR2GS_ADAPTIVE  mCQR2GS with the runtime decision on the number of CholeskyQR
 *                 repetitions the paper proposes (DESIGN R-23): after a
 *                 panel's first CholeskyQR (U1, Z = U1^{-1}) the estimate
 *                 E = max(u nu(U1)^2 nu(Z)^2, u nu(R_{1:j,j}) nu(Z)), nu(M) = ||M||_F/sqrt(b),
 *                 decides on the device (identically on every rank) whether the repetition
 *                 (l.7-8; the second CQR of l.1) is skipped: E <= tau (tsqr_set_adapt_tau,
 *                 default 2^-50) -> R_jj = U1.  tau = 0: bitwise TSQR_MCQR2GS
 *
 * Conventions for every entry point:
 *   - Matrices are FP64, COLUMN-MAJOR: element (r, c) of X is X[r + c*ldX].
 *   - A and R passed to tsqr_factor are DEVICE pointers on the plan's device.
 *   - All element offsets are 64-bit (m_local * n may exceed 2^31).
 *   - Functions return a tsqr_status; they never abort the process.  A non-OK
 *     status from tsqr_create leaves *plan == NULL.
 *   - The library performs no host<->device copies of A or R, no cuBLAS/cuSOLVER
 *     calls and has no CPU fallback: every arithmetic step runs in its own sm_100a
 *     kernels.  Cross-GPU sums (nranks > 1) are fused into the split-row reduction kernel:
 *     each rank stores its block sums into every peer's slot of a symmetric NCCL window
 *     (NCCL device API, NVLink load/store) and, after an LSA barrier, adds the nranks slots
 *     in rank order -- deterministic and bitwise identical on every rank (validated on 2
 *     and 4 GPUs; with more than 4 ranks only if TSQR_FUSED_ALLREDUCE=1).  Otherwise, or with
 *     TSQR_NCCL_ALLREDUCE=1 (read at tsqr_create), ncclAllReduce(ncclFloat64, ncclSum).
 *     A plan given a 1-rank communicator runs ncclAllReduce (a copy), or the fused kernel
 *     with TSQR_FUSED_ALLREDUCE=1 -- so both cross-GPU data planes run on one GPU in tests.
 *
 * Citation keys: P:n = line n of the paper's LaTeX source;
 * DESIGN.md lists the readings (R-k) taken where the paper is silent.
 */
#ifndef TSQR_H
#define TSQR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tsqr_plan_s* tsqr_plan_t;

typedef enum {
  TSQR_OK = 0,
  TSQR_ERR_INVALID_ARG = 1, /* bad pointer, size, leading dimension or alignment       */
  TSQR_ERR_UNSUPPORTED = 2, /* valid but not supported in this version (see create)     */
  TSQR_ERR_CUDA = 3,        /* a CUDA runtime call failed (message: tsqr_last_error)    */
  TSQR_ERR_NCCL = 4,        /* an NCCL call failed or the communicator reported an error */
  TSQR_ERR_BREAKDOWN = 5,   /* Cholesky breakdown: a Gram pivot <= 0 or non-finite      */
  TSQR_ERR_WORKSPACE = 6    /* workspace NULL, too small or misaligned                   */
} tsqr_status;

typedef enum {
  TSQR_CQR2 = 0,
  TSQR_CQR2GS = 1,
  TSQR_MCQR2GS = 2,
  TSQR_CQR = 3,
  TSQR_CQRGS = 4,
  TSQR_SCQR3 = 5,
  TSQR_SCQR = 6,
  TSQR_MCQR2GS_ADAPTIVE = 7
} tsqr_algo;

/* Where a Cholesky breakdown happened (identical on every rank, since every rank
 * factors the same allreduced Gram block).  pass: CQRGS pass (1 or 2; always 1 for
 * the other methods); panel: 1-based panel index; stage: which CholeskyQR of that
 * panel (1 = first, 2 = the second "re-orthogonalising" one of CQR2 / Alg. 8 l.8);
 * pivot: 0-based column inside the panel's b x b Gram block; pivot_value: the
 * offending pivot (<= 0, NaN or Inf).  Breakdown rule: unpivoted upper Cholesky
 * W = U^T U fails iff a pivot d is not > 0 or not finite (R-5). */
typedef struct {
  int32_t pass, panel, stage, pivot;
  double pivot_value;
} tsqr_breakdown_info;

/* Bytes of device workspace tsqr_create needs for this problem (0 on invalid
 * arguments).  Depends only on (m_local, n, panel_b, nranks, algo). */
size_t tsqr_workspace_bytes(int64_t m_local, int32_t n, int32_t panel_b, int32_t nranks,
                            tsqr_algo algo);

/* Create a plan.  COLLECTIVE over `nccl_comm` (every rank must call it with the
 * same n, panel_b and algo; m_local may differ per rank).  When nccl_comm is NULL
 * the plan is single-GPU (P = 1).
 *   m_local        rows owned by this rank, >= 0 (sum over ranks >= n)
 *   n              columns, 1 <= n <= 16384
 *   panel_b        panel width b: required n % b == 0 and b = 16, 32 or a
 *                  multiple of 64 up to 4096 (the paper's 400-4000-wide strong-scaling panels,
 *                  P:504, as multiples of 64: DESIGN R-24); for CQR / CQR2 / sCQR(3), b must
 *                  equal n (single panel).  Ragged panels: TSQR_ERR_UNSUPPORTED.
 *   nccl_comm      ncclComm_t (see tsqr_nccl_comm_init) or NULL
 *   algo           method, see tsqr_algo
 *   cuda_stream    cudaStream_t every launch and NCCL call is enqueued on (NULL =
 *                  legacy default stream)
 *   workspace      device buffer of >= tsqr_workspace_bytes(...) bytes, 256-byte
 *                  aligned, owned by the caller and kept alive until destroy
 * All ranks return the same status (arguments are validated with one small
 * allreduce), so a bad argument on one rank cannot deadlock the others.
 * The plan owns only host state; the caller owns A, R, workspace, stream, comm. */
tsqr_status tsqr_create(tsqr_plan_t* plan, int64_t m_local, int32_t n, int32_t panel_b,
                        void* nccl_comm, tsqr_algo algo, void* cuda_stream, void* workspace,
                        size_t workspace_bytes);

/* Factor A = Q R.  COLLECTIVE; asynchronous on the plan's stream.
 *   A    device, m_local x n, column-major, lda >= max(1, m_local); overwritten by
 *        this rank's rows of Q.  8-byte aligned.
 *   R    device, n x n, column-major, ldr >= n; receives the full upper triangle,
 *        exact zeros strictly below the diagonal and a positive diagonal, bitwise
 *        identical on all ranks.
 * Returns TSQR_OK once everything is enqueued; numerical status (breakdown) is
 * reported by tsqr_wait.  After a breakdown the contents of A and R are
 * unspecified.  A plan is bound to one stream and is not thread-safe. */
tsqr_status tsqr_factor(tsqr_plan_t plan, double* A, int64_t lda, double* R, int32_t ldr);

/* Synchronise the plan's stream and return the sticky numerical status of the
 * last tsqr_factor: TSQR_OK or TSQR_ERR_BREAKDOWN (details in *info, may be NULL),
 * or TSQR_ERR_CUDA / TSQR_ERR_NCCL.  Reading the status is the only device->host
 * transfer the library makes. */
tsqr_status tsqr_wait(tsqr_plan_t plan, tsqr_breakdown_info* info);

/* Number of allreduce calls and kernel launches the last tsqr_factor enqueued
 * (4k-2 allreduces for CQR2GS and mCQR2GS, 2 for CQR2; Appendix A.2 of SURVEY).
 * Either pointer may be NULL. */
tsqr_status tsqr_last_counts(tsqr_plan_t plan, int64_t* allreduces, int64_t* launches);

/* Factor from HOST buffers (the end-to-end form of tsqr_factor): A_host (m_local x n,
 * ld lda_host) is copied to the caller's device buffer A_dev (ld lda_dev), factored in
 * place, and Q is copied back over A_host; R is produced in R_dev (device, ldr_dev) and
 * copied to R_host (ld ldr_host).  The host->device copy runs on the plan's stream before
 * the factorisation (every column is read by the first projection); for the panel-wise
 * methods (MCQR2GS, CQR2GS with k > 1) each panel Q_j is copied back on a plan-owned
 * second stream as soon as it is final, overlapping the remaining panels; otherwise Q is
 * copied back after the factorisation.  Copies are cudaMemcpy2DAsync (asynchronous only
 * if the host buffers are pinned, e.g. cudaHostAlloc / torch pin_memory); A_host must
 * not be touched until tsqr_wait returns.  COLLECTIVE like tsqr_factor; completes at
 * tsqr_wait (which orders the plan stream after the copies). */
tsqr_status tsqr_factor_host(tsqr_plan_t plan, double* A_host, int64_t lda_host, double* R_host,
                             int32_t ldr_host, double* A_dev, int64_t lda_dev, double* R_dev,
                             int32_t ldr_dev);

/* Per-kernel-class timing with CUDA events recorded on the plan's stream around every
 * launch of the next tsqr_factor calls (off by default; enabling it adds two event
 * records per launch).  Classes (TSQR_KCLASS_*): 0 Gram (split-row partials + reduce),
 * 1 projection (Y, C), 2 trailing/re-orth update, 3 TRMM (Q = A U^{-1}), 4 Cholesky +
 * inverse, 5 R assembly and other small kernels, 6 allreduce (NCCL), 7 the single-launch
 * cluster factorisation of small problems (tsqr_exec_path == TSQR_PATH_CLUSTER).
 * tsqr_timing synchronises the stream and returns, summed over every launch of `kclass`
 * since the last tsqr_timing_reset: total milliseconds, launch count, and the
 * ALGORITHMIC flops and HBM bytes of those launches (paper's flop counts: Gram m b^2,
 * TRMM m b^2, projection / update 2 m p q; bytes = operands read + written once). */
typedef enum {
  TSQR_KCLASS_GRAM = 0,
  TSQR_KCLASS_PROJ = 1,
  TSQR_KCLASS_UPDATE = 2,
  TSQR_KCLASS_TRMM = 3,
  TSQR_KCLASS_CHOL = 4,
  TSQR_KCLASS_SMALL = 5,
  TSQR_KCLASS_ALLREDUCE = 6,
  TSQR_KCLASS_CLUSTER = 7,
  TSQR_KCLASS_COUNT = 8
} tsqr_kclass;
tsqr_status tsqr_set_timing(tsqr_plan_t plan, int32_t enable);
tsqr_status tsqr_timing_reset(tsqr_plan_t plan);
tsqr_status tsqr_timing(tsqr_plan_t plan, int32_t kclass, double* ms, int64_t* launches, double* flops,
                        double* bytes);

/* CUDA graphs (default on): the first tsqr_factor of a plan captures the whole
 * factorisation (kernels, NCCL allreduces and, if enabled, timing events) into a CUDA graph
 * that later calls with the same A, lda, R, ldr and timing setting replay with one launch.
 * enable = 0 switches to eager enqueueing. */
tsqr_status tsqr_set_graph(tsqr_plan_t plan, int32_t enable);

/* NEXT-f1 look-ahead ("overlap the update of panels with computing the CholeskyQR of the
 * next panel (Algorithm 8 lines 4 and 6)"), TSQR_MCQR2GS on the streaming path with >= 3 panels:
 * after the projection of step j the panel's own columns are updated first, its CholeskyQR chain
 * (l.6-8, incl. the cross-GPU sums) then runs on a second stream while the main stream updates
 * the remaining trailing columns; the two join before step j+1.  The same kernels on the same
 * operands: Q and R are bitwise those of the serial schedule.  enable = 0 (default; also
 * TSQR_LOOKAHEAD=1 at tsqr_create) / 1; silently off where it does not apply.  COLLECTIVE in
 * effect: every rank must use the same setting (the allreduce order is unchanged). */
tsqr_status tsqr_set_lookahead(tsqr_plan_t plan, int32_t enable);

/* TSQR_MCQR2GS_ADAPTIVE: threshold tau of the skip rule (default 2^-50 ~ 8.9e-16; 0 never
 * skips).  Takes effect at the next tsqr_factor (it re-captures the CUDA graph). */
tsqr_status tsqr_set_adapt_tau(tsqr_plan_t plan, double tau);
/* Panels whose CholeskyQR repetition the last factorisation skipped (valid after tsqr_wait;
 * 0 for the other algorithms). */
tsqr_status tsqr_skipped_panels(tsqr_plan_t plan, int32_t* panels);

/* Which cross-GPU data plane the plan's allreduces use: TSQR_PLANE_LOCAL (no communicator,
 * no exchange), TSQR_PLANE_NCCL (k_reduce + ncclAllReduce) or TSQR_PLANE_FUSED (the split-row
 * reduction fused with the cross-GPU sum over NVLink peer memory, k_reduce_allreduce).
 * Decided collectively at tsqr_create, identical on every rank. */
typedef enum { TSQR_PLANE_LOCAL = 0, TSQR_PLANE_NCCL = 1, TSQR_PLANE_FUSED = 2 } tsqr_plane;
tsqr_status tsqr_data_plane(tsqr_plan_t plan, int32_t* plane);

/* Which execution path the plan's tsqr_factor takes (decided at tsqr_create):
 * TSQR_PATH_STREAM  -- one sm_100a kernel per step of the algorithm (split-row Gram and
 *                      projection, Cholesky, TRMM, update, R assembly), replayed as a CUDA graph;
 * TSQR_PATH_CLUSTER -- small problems on one rank (no communicator) whose m x n matrix fits in
 *                      the distributed shared memory of one thread-block cluster (16 CTAs, or 8):
 *                      the whole factorisation in ONE kernel launch, A read once and Q written
 *                      once (the paper's steps in the same order; Q = A U^{-1} as the row-wise
 *                      triangular solve of P:122).  b in {16, 32, 64}.  TSQR_CLUSTER_PATH=0 in
 *                      the environment at tsqr_create disables it. */
typedef enum { TSQR_PATH_STREAM = 0, TSQR_PATH_CLUSTER = 1 } tsqr_path;
tsqr_status tsqr_exec_path(tsqr_plan_t plan, int32_t* path);

/* Destroy the plan (host state, its CUDA graph and, with nranks > 1, the symmetric NCCL
 * window and device communicator of the fused reduce + allreduce).  COLLECTIVE when the plan
 * has a communicator with nranks > 1: every rank destroys its plan, before the
 * communicator. */
tsqr_status tsqr_destroy(tsqr_plan_t plan);

/* Human-readable name of a status; static storage. */
const char* tsqr_status_string(tsqr_status s);

/* Message of the last CUDA/NCCL error seen by this thread (static storage). */
const char* tsqr_last_error(void);

/* NCCL bootstrap.  tsqr_nccl_unique_id writes the 128-byte ncclUniqueId on rank 0;
 * the caller broadcasts those bytes (e.g. over a torch.distributed group) and every
 * rank calls tsqr_nccl_comm_init(&comm, nranks, rank, id, device).  The returned
 * comm is owned by the caller and released with tsqr_nccl_comm_destroy. */
tsqr_status tsqr_nccl_unique_id(void* id128);
tsqr_status tsqr_nccl_comm_init(void** comm, int32_t nranks, int32_t rank, const void* id128,
                                int32_t device);
tsqr_status tsqr_nccl_comm_destroy(void* comm);

/* ------------------------------------------------------------------------- */
/* Step-level entry points (the hot-path steps of SURVEY §8(a), exposed so each */
/* kernel can be checked against the oracle on its own).  All pointers device, */
/* column-major, enqueued on `cuda_stream`, single GPU (no allreduce).  The     */
/* split-row entries (gram, proj, and chol_inv for b >= 128) use a library-   */
/* owned scratch buffer, one per device; growing it synchronises the device     */
/* (cudaDeviceSynchronize) before the old buffer is freed.  Not thread-safe:    */
/* call the step entries from one host thread.  The plan API (tsqr_create /     */
/* tsqr_factor) does not use it.                                                */
/* ------------------------------------------------------------------------- */

/* W (b x b, ldw >= b) = X^T X for X (m x b): the local Gram block (Alg. 2 l.2,
 * P:152; Alg. 7 l.2), upper triangle computed with a fixed split-row
 * partition and a fixed-order reduction, lower triangle mirrored bitwise (R-11).
 * Deterministic.  b in {1..256}. */
tsqr_status tsqr_gram(const double* X, int64_t ldx, int64_t m, int32_t b, double* W, int32_t ldw,
                      void* cuda_stream);

/* OUT (p x q, ldo >= p) = L^T Rm for L (m x p), Rm (m x q): the projection blocks
 * Y = Q_j^T A_trail (Alg. 7 l.7; Alg. 8 l.3) and
 * C = Q_{1:j-1}^T V (Alg. 8 l.7).  Deterministic. p, q <= 4096. */
tsqr_status tsqr_proj(const double* L, int64_t ldl, const double* Rm, int64_t ldr, int64_t m,
                      int32_t p, int32_t q, double* OUT, int32_t ldo, void* cuda_stream);

/* X (m x q) -= L (m x p) * S (p x q), in place (Alg. 7 l.9; Alg. 8 l.4 and
 * l.7).  p, q <= 4096. */
tsqr_status tsqr_update(double* X, int64_t ldx, const double* L, int64_t ldl, const double* S,
                        int32_t lds, int64_t m, int32_t p, int32_t q, void* cuda_stream);

/* Cholesky W = U^T U (upper, unpivoted) and the explicit inverse Z = U^{-1}
 * (Alg. 1 l.2; R-4, R-5).  W b x b (only the upper triangle is read);
 * U and Z receive exact zeros below the diagonal.  On breakdown *status_dev
 * (device int32[8]) is set to {1, pivot, ...} with the pivot value in
 * status_dev[2..3] as a double; otherwise it is left untouched.  b: 16, 32 or a multiple of 64
 * up to 4096 (b > 256: multi-CTA blocked kernels, one launch per block step). */
tsqr_status tsqr_chol_inv(const double* W, int32_t ldw, int32_t b, double* U, int32_t ldu, double* Z,
                          int32_t ldz, int32_t* status_dev, void* cuda_stream);

/* X (m x b) <- X * Z in place for upper-triangular Z (b x b): panel
 * orthogonalisation Q = A R^{-1} with the explicit inverse (Alg. 1 l.3, P:133;
 * R-4).  b <= 256. */
tsqr_status tsqr_trmm(double* X, int64_t ldx, int64_t m, int32_t b, const double* Z, int32_t ldz,
                      void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* TSQR_H */
