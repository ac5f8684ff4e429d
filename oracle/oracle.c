/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the CholeskyQR family of
 * arXiv 2405.04237 ("QR factorization of ill-conditioned tall-and-skinny matrices on
 * distributed-memory systems", Mijic, Kaushik, Davidovic).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2405_04237_b200/), and the
 * CUDA path never calls it.
 *
 * Citation keys: "P:n" is line n of /root/reference/PAPER.md (the paper's LaTeX
 * source); "S:n" is line n of /root/reference/SPEC.md; "R-k" is reading k in
 * DESIGN.md section "Readings of the paper".
 *
 * Conventions
 *   - FP64 IEEE-754, round-to-nearest-even, compiled with -O2 -ffp-contract=off
 *     (no FMA contraction, no fast-math): every product and sum below is rounded
 *     exactly where it is written.
 *   - Matrices are column-major: element (r, c) of X lives at X[r + c*ldx].
 *   - Sums over rows ("Sigma_rows") use the fixed chunked pairwise rule of R-3:
 *     the global row range is cut into chunks of ORC_CHUNK = 256 rows; each chunk
 *     is a plain sequential sum in row order; chunk partials are combined by a
 *     fixed recursive-halving binary tree over the chunk index (mid = lo+(hi-lo)/2).
 *     The result is therefore independent of the number of threads.
 *   - Threads (OpenMP) only evaluate independent subtrees or independent rows.
 *
 * Every function names the passage it follows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define ORC_CHUNK 256

/* status codes */
#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_BREAKDOWN 5
#define ORC_ERR_NOMEM 6

/* algorithms */
#define ORC_CQR2 0
#define ORC_CQR2GS 1
#define ORC_MCQR2GS 2
#define ORC_CQR 3
#define ORC_CQRGS 4
#define ORC_SCQR3 5
#define ORC_SCQR 6
#define ORC_MCQR2GS_ADAPTIVE 7

/* unit roundoff of FP64 round-to-nearest-even: u = 2^-53 */
#define ORC_UNIT_ROUNDOFF 1.1102230246251565e-16

typedef struct {
  int32_t status;      /* ORC_OK or ORC_ERR_* */
  int32_t pass;        /* CQRGS pass (1 or 2) -- CQR2GS only; 1 otherwise */
  int32_t panel;       /* 1-based panel index */
  int32_t stage;       /* which CQR of the panel (1 or 2) */
  int32_t pivot;       /* 0-based pivot index inside the panel's Gram block */
  int32_t pad;
  double pivot_value;  /* the failing pivot d (d <= 0 or non-finite) */
} orc_info;

static int g_threads = 1;
/* number of Sigma_rows reductions performed: each is one Allreduce of the
 * distributed algorithm (Alg. 2 l.4 P:154; Alg. 7 l.3, l.8 P:345) */
static int64_t g_reductions = 0;

/* NEXT-f4: threshold tau of the adaptive repetition rule (mcqr2gs_adaptive below) and
 * the number of panels whose repetition the last adaptive factorisation skipped */
static double g_adapt_tau = 8.8817841970012523e-16; /* 2^-50 (R-23) */
static int64_t g_adapt_skipped = 0;
void orc_set_adapt_tau(double tau) { g_adapt_tau = tau; }
double orc_get_adapt_tau(void) { return g_adapt_tau; }
int64_t orc_adapt_skipped(void) { return g_adapt_skipped; }

void orc_set_threads(int t) { g_threads = t > 0 ? t : 1; }
int orc_get_threads(void) { return g_threads; }
int64_t orc_reduction_count(void) { return g_reductions; }
void orc_reset_reduction_count(void) { g_reductions = 0; }

/* ------------------------------------------------------------------------- */
/* Sigma_rows X^T Y: the chunked pairwise row sum (R-3).                       */
/* Used for: Gram W = A^T A (Alg. 1 l.1; Alg. 2 l.2 + l.4 Allreduce     */
/* P:152-154), projection Y = Q^T A (Alg. 6 l.6 P:296; Alg. 7 l.7-8 P:349-350;  */
/* Alg. 8 l.3 P:464) and re-orthogonalisation C = Q^T V (Alg. 8 l.7 P:468).    */
/* ------------------------------------------------------------------------- */
typedef struct {
  const double* X; int64_t ldx;
  const double* Y; int64_t ldy;
  int64_t m, p, q;  /* X is m x p, Y is m x q; result p x q, column-major ld p */
  int upper;        /* 1: only entries i <= j are computed (Gram) */
} atb_job;

/* leaf: one chunk, plain sequential sum over its rows in row order */
static void atb_leaf(const atb_job* J, int64_t chunk, double* out) {
  int64_t r0 = chunk * ORC_CHUNK, r1 = r0 + ORC_CHUNK;
  if (r1 > J->m) r1 = J->m;
  for (int64_t j = 0; j < J->q; ++j) {
    const double* y = J->Y + j * J->ldy;
    int64_t imax = J->upper ? j + 1 : J->p;
    for (int64_t i = 0; i < imax; ++i) {
      const double* x = J->X + i * J->ldx;
      double s = 0.0;
      for (int64_t r = r0; r < r1; ++r) s += x[r] * y[r];
      out[i + j * J->p] = s;
    }
  }
}

static void mat_add(double* a, const double* b, int64_t len) {
  for (int64_t t = 0; t < len; ++t) a[t] += b[t];
}

/* S(lo,hi) = S(lo,mid) + S(mid,hi), mid = lo + (hi-lo)/2; leaves are chunks.
 * `frontier` (may be NULL) holds precomputed sums of the subtrees at depth `fdepth`. */
typedef struct {
  int64_t lo, hi;
} node_range;

static void atb_node(const atb_job* J, int64_t lo, int64_t hi, double* out, double* scratch) {
  int64_t pq = J->p * J->q;
  if (hi - lo == 1) { atb_leaf(J, lo, out); return; }
  int64_t mid = lo + (hi - lo) / 2;
  atb_node(J, lo, mid, out, scratch);
  atb_node(J, mid, hi, scratch, scratch + pq);
  mat_add(out, scratch, pq);
}

/* enumerate the nodes at depth `d` of the fixed tree (stopping early at leaves) */
static int64_t enum_frontier(int64_t lo, int64_t hi, int d, node_range* outv, int64_t cnt) {
  if (d == 0 || hi - lo == 1) { outv[cnt].lo = lo; outv[cnt].hi = hi; return cnt + 1; }
  int64_t mid = lo + (hi - lo) / 2;
  cnt = enum_frontier(lo, mid, d - 1, outv, cnt);
  return enum_frontier(mid, hi, d - 1, outv, cnt);
}

/* combine frontier sums up the same tree */
static void atb_combine(const atb_job* J, int64_t lo, int64_t hi, int d, const node_range* fr,
                        double* const* frv, int64_t* idx, double* out, double* scratch) {
  int64_t pq = J->p * J->q;
  if (d == 0 || hi - lo == 1) {
    memcpy(out, frv[*idx], (size_t)pq * sizeof(double));
    (*idx)++;
    return;
  }
  int64_t mid = lo + (hi - lo) / 2;
  atb_combine(J, lo, mid, d - 1, fr, frv, idx, out, scratch);
  atb_combine(J, mid, hi, d - 1, fr, frv, idx, scratch, scratch + pq);
  mat_add(out, scratch, pq);
}

static int tree_levels(int64_t nchunks) {
  int l = 1;
  while (((int64_t)1 << (l - 1)) < nchunks) ++l;
  return l + 1;
}

/* out (p x q, ld p) = Sigma_rows X^T Y.  For upper=1 only i<=j is defined (and
 * the lower part of `out` is left zero). Returns ORC_OK or ORC_ERR_NOMEM. */
static int atb(const atb_job* J, double* out) {
  int64_t pq = J->p * J->q;
  memset(out, 0, (size_t)pq * sizeof(double));
  g_reductions++;
  if (J->m == 0 || pq == 0) return ORC_OK;
  int64_t nchunks = (J->m + ORC_CHUNK - 1) / ORC_CHUNK;
  /* frontier depth depends only on the problem (never on the thread count) */
  int d = 0;
  while (d < 8 && ((int64_t)1 << (d + 1)) <= nchunks && ((int64_t)1 << (d + 1)) * pq <= ((int64_t)1 << 27)) ++d;
  int64_t maxnodes = (int64_t)1 << d;
  node_range* fr = (node_range*)malloc(sizeof(node_range) * (size_t)maxnodes);
  int64_t nf = enum_frontier(0, nchunks, d, fr, 0);
  int lv = tree_levels(nchunks);
  double* frbuf = (double*)malloc(sizeof(double) * (size_t)(nf * pq));
  double** frv = (double**)malloc(sizeof(double*) * (size_t)nf);
  int nt = g_threads;
  double* scr = (double*)malloc(sizeof(double) * (size_t)(pq * lv * nt));
  if (!fr || !frbuf || !frv || !scr) { free(fr); free(frbuf); free(frv); free(scr); return ORC_ERR_NOMEM; }
  for (int64_t t = 0; t < nf; ++t) frv[t] = frbuf + t * pq;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int64_t t = 0; t < nf; ++t) {
    double* my = scr + (int64_t)omp_get_thread_num() * pq * lv;
    atb_node(J, fr[t].lo, fr[t].hi, frv[t], my);
  }
  int64_t idx = 0;
  atb_combine(J, 0, nchunks, d, fr, frv, &idx, out, scr);
  free(fr); free(frbuf); free(frv); free(scr);
  return ORC_OK;
}

/* gram(X): W = X^T X, upper triangle computed with the row-sum rule, then the lower
 * triangle mirrored bitwise ("Construct Gram matrix"; R-11). */
int orc_gram(const double* X, int64_t ldx, int64_t m, int64_t b, double* W, int64_t ldw) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!t) return ORC_ERR_NOMEM;
  atb_job J = {X, ldx, X, ldx, m, b, b, 1};
  int rc = atb(&J, t);
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < b; ++i) W[i + j * ldw] = (i <= j) ? t[i + j * b] : t[j + i * b];
  free(t);
  return rc;
}

/* out (p x q) = Sigma_rows X^T Y (projection) */
int orc_atb(const double* X, int64_t ldx, const double* Y, int64_t ldy, int64_t m, int64_t p,
            int64_t q, double* out, int64_t ldo) {
  double* t = (double*)malloc(sizeof(double) * (size_t)(p * q > 0 ? p * q : 1));
  if (!t) return ORC_ERR_NOMEM;
  atb_job J = {X, ldx, Y, ldy, m, p, q, 0};
  int rc = atb(&J, t);
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) out[i + j * ldo] = t[i + j * p];
  free(t);
  return rc;
}

/* chol(W): unpivoted upper Cholesky W = U^T U, right-looking (Alg. 1 l.2, P:132;
 * S:69-77; R-5).  Breakdown iff a pivot d <= 0 or d is not finite: returns the
 * 0-based pivot index in *pivot and d in *pivot_value.  U's strict lower part is
 * set to exact zeros. W is not modified. */
int orc_chol(const double* W, int64_t ldw, int64_t b, double* U, int64_t ldu, int32_t* pivot,
             double* pivot_value) {
  double* S = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!S) return ORC_ERR_NOMEM;
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < b; ++i) S[i + j * b] = W[i + j * ldw];
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i < b; ++i) U[i + j * ldu] = 0.0;
  for (int64_t kk = 0; kk < b; ++kk) {
    double d = S[kk + kk * b];
    if (!(d > 0.0) || !isfinite(d)) {
      if (pivot) *pivot = (int32_t)kk;
      if (pivot_value) *pivot_value = d;
      free(S);
      return ORC_ERR_BREAKDOWN;
    }
    double ukk = sqrt(d);
    U[kk + kk * ldu] = ukk;
    for (int64_t j = kk + 1; j < b; ++j) U[kk + j * ldu] = S[kk + j * b] / ukk;
    /* trailing update of the upper triangle: S_ij -= U_ki U_kj, i <= j */
    for (int64_t j = kk + 1; j < b; ++j)
      for (int64_t i = kk + 1; i <= j; ++i) S[i + j * b] -= U[kk + i * ldu] * U[kk + j * ldu];
  }
  free(S);
  return ORC_OK;
}

/* rsolve(X, U): X <- X U^{-1} for upper-triangular U, by row-wise forward
 * substitution over U's columns, in index order ("Q := A R^{-1} ... trsm", P:122,
 * P:133; R-4). */
void orc_rsolve(double* X, int64_t ldx, int64_t m, int64_t b, const double* U, int64_t ldu) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (int64_t r = 0; r < m; ++r) {
    for (int64_t j = 0; j < b; ++j) {
      double s = X[r + j * ldx];
      for (int64_t i = 0; i < j; ++i) s -= X[r + i * ldx] * U[i + j * ldu];
      X[r + j * ldx] = s / U[j + j * ldu];
    }
  }
}

/* Explicit inverse of an upper-triangular U by column-wise back substitution of
 * U Z = I (the textbook definition of U^{-1}); used only as a test pin for the
 * GPU's explicit-inverse step (R-4). Lower part exact zeros. */
void orc_tri_inv(const double* U, int64_t ldu, int64_t b, double* Z, int64_t ldz) {
  for (int64_t j = 0; j < b; ++j) {
    for (int64_t i = 0; i < b; ++i) Z[i + j * ldz] = 0.0;
    for (int64_t i = j; i >= 0; --i) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int64_t t = i + 1; t <= j; ++t) s -= U[i + t * ldu] * Z[t + j * ldz];
      Z[i + j * ldz] = s / U[i + i * ldu];
    }
  }
}

/* C (p x q) = A (p x r) * B (r x q), plain triple loop, inner index ascending.
 * Used for R := R2 R1 (Alg. 3 l.3; Alg. 6 wrapper l.3) and
 * R_{1:j-1,j} += C U1 (R-8).  upper_tri=1 skips the known-zero region of two
 * upper-triangular factors: only t in [i, j] contributes. */
void orc_matmul(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t p, int64_t r,
                int64_t q, double* C, int64_t ldc, int upper_tri, int accumulate) {
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) {
      double s = 0.0;
      if (upper_tri) {
        if (i <= j)
          for (int64_t t = i; t <= j; ++t) s += A[i + t * lda] * B[t + j * ldb];
      } else {
        for (int64_t t = 0; t < r; ++t) s += A[i + t * lda] * B[t + j * ldb];
      }
      C[i + j * ldc] = accumulate ? C[i + j * ldc] + s : s;
    }
}

/* X (m x q) -= Q (m x p) * Y (p x q), row-local, inner index ascending
 * ("A_{j+1:k} := A_{j+1:k} - Q_j Y", Alg. 6 l.7 P:297; Alg. 7 l.9 P:351;
 * Alg. 8 l.4 P:465 and l.7 P:468). */
void orc_sub_prod(double* X, int64_t ldx, const double* Q, int64_t ldq, const double* Y, int64_t ldy,
                  int64_t m, int64_t p, int64_t q) {
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (int64_t r = 0; r < m; ++r) {
    for (int64_t j = 0; j < q; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < p; ++i) s += Q[r + i * ldq] * Y[i + j * ldy];
      X[r + j * ldx] -= s;
    }
  }
}

/* ------------------------------------------------------------------------- */
/* Algorithms                                                                 */
/* ------------------------------------------------------------------------- */

/* CQR(X): W = gram(X); U = chol(W); X <- X U^{-1}; returns U (Alg. 1 P:125-136,
 * Alg. 2 P:145-160 -- on one address space the Allreduce is the row sum). */
static int cqr(double* X, int64_t ldx, int64_t m, int64_t b, double* U, int64_t ldu, orc_info* info) {
  double* W = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!W) return ORC_ERR_NOMEM;
  int rc = orc_gram(X, ldx, m, b, W, b);
  if (rc == ORC_OK) {
    int32_t piv = -1; double pv = 0.0;
    rc = orc_chol(W, b, b, U, ldu, &piv, &pv);
    if (rc == ORC_ERR_BREAKDOWN && info) { info->pivot = piv; info->pivot_value = pv; }
  }
  if (rc == ORC_OK) orc_rsolve(X, ldx, m, b, U, ldu);
  free(W);
  return rc;
}

/* sCQR(X) -- shifted CholeskyQR (Alg. 4):
 *   G = X^T X                                   (l.1; row sums of R-3)
 *   s = sqrt(m) u ||X||_F^2                     (l.2, "calculate shift"; the conservative
 *                                                Frobenius-norm shift; u = 2^-53)
 *   W = G + s I                                 (l.3)
 *   W = U^T U;  X <- X U^{-1}                   (l.4-5)
 * ||X||_F^2 = sum_j sum_rows x_rj^2 ("summing over the squares of the elements"):
 * the inner row sums are exactly the Gram diagonal G_jj (same products, same R-3 order), so
 * ||X||_F^2 = sum_j G_jj, summed over j in index order.  m is the global row count (on
 * one address space: the rows of X). */
static int scqr(double* X, int64_t ldx, int64_t m, int64_t b, double* U, int64_t ldu, orc_info* info,
                double unit_roundoff) {
  double* W = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!W) return ORC_ERR_NOMEM;
  int rc = orc_gram(X, ldx, m, b, W, b);
  if (rc == ORC_OK) {
    double fro2 = 0.0;
    for (int64_t j = 0; j < b; ++j) fro2 += W[j + j * b];
    const double s = sqrt((double)m) * unit_roundoff * fro2;
    for (int64_t j = 0; j < b; ++j) W[j + j * b] += s;
    int32_t piv = -1; double pv = 0.0;
    rc = orc_chol(W, b, b, U, ldu, &piv, &pv);
    if (rc == ORC_ERR_BREAKDOWN && info) { info->pivot = piv; info->pivot_value = pv; }
  }
  if (rc == ORC_OK) orc_rsolve(X, ldx, m, b, U, ldu);
  free(W);
  return rc;
}

static void zero_mat(double* R, int64_t ldr, int64_t p, int64_t q) {
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < p; ++i) R[i + j * ldr] = 0.0;
}

static int fail(orc_info* info, int rc, int pass, int panel, int stage) {
  if (info) {
    info->status = rc;
    if (rc == ORC_ERR_BREAKDOWN) { info->pass = pass; info->panel = panel; info->stage = stage; }
  }
  return rc;
}

/* CQR2 of an m x b block: U1 = CQR(X); U2 = CQR(X); R = U2 U1 (Alg. 3).
 * Stages 1 and 2 of `panel`. */
static int cqr2_block(double* X, int64_t ldx, int64_t m, int64_t b, double* R, int64_t ldr,
                      int pass, int panel, orc_info* info) {
  double* U1 = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* U2 = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!U1 || !U2) { free(U1); free(U2); return fail(info, ORC_ERR_NOMEM, 0, 0, 0); }
  int rc = cqr(X, ldx, m, b, U1, b, info);
  if (rc != ORC_OK) { free(U1); free(U2); return fail(info, rc, pass, panel, 1); }
  rc = cqr(X, ldx, m, b, U2, b, info);
  if (rc != ORC_OK) { free(U1); free(U2); return fail(info, rc, pass, panel, 2); }
  orc_matmul(U2, b, U1, b, b, b, b, R, ldr, 1, 0);
  free(U1); free(U2);
  return ORC_OK;
}

/* CQRGS(X, b): for j = 1..k: R_jj = CQR(X_j); Y = X_j^T X_{j+1:k};
 * X_{j+1:k} -= X_j Y; R_{j,j+1:k} = Y (Alg. 6; Alg. 7).
 * Ragged last panel allowed. R (n x n) must be zeroed by the caller. */
static int cqrgs(double* X, int64_t ldx, int64_t m, int64_t n, int64_t b, double* R, int64_t ldr,
                 int pass, orc_info* info) {
  int64_t k = (n + b - 1) / b;
  for (int64_t j = 0; j < k; ++j) {
    int64_t c0 = j * b, bj = (c0 + b <= n) ? b : n - c0;
    double* Xj = X + c0 * ldx;
    int rc = cqr(Xj, ldx, m, bj, R + c0 + c0 * ldr, ldr, info);
    if (rc != ORC_OK) return fail(info, rc, pass, (int)j + 1, 1);
    int64_t c1 = c0 + bj, nt = n - c1;
    if (nt > 0) {
      double* Y = R + c0 + c1 * ldr; /* R_{j,j+1:k} := Y */
      rc = orc_atb(Xj, ldx, X + c1 * ldx, ldx, m, bj, nt, Y, ldr);
      if (rc != ORC_OK) return fail(info, rc, 0, 0, 0);
      orc_sub_prod(X + c1 * ldx, ldx, Xj, ldx, Y, ldr, m, bj, nt);
    }
  }
  return ORC_OK;
}

/* Lines 6-8 of Alg. 8 for panel j plus its R bookkeeping (R-8), on the m x
 * (c0 + bj) leading columns of X: X[:, 0:c0] holds Q_{1:j-1} (final), X[:, c0:c0+bj] holds
 * the panel A_j after the line-3/4 projection.
 *     U1 = CQR(A_j)  (A_j <- V1 in place)                        (l.6; R-6)
 *     C = Q_{1:j-1}^T A_j;  A_j -= Q_{1:j-1} C                   (l.7)
 *     U2 = CQR(A_j)  (A_j <- Q_j)                                (l.8)
 *     R_jj = U2 U1;  R_{1:j-1,j} += C U1                         (R-8)
 * R points at R_{1,1} (ld ldr); R_{1:j-1,j} must hold its line-5 contents on entry.  The
 * R-8 identity this implements: A_j = V1 U1 and V1 = Q_{1:j-1} C + Q_j U2, hence
 * A_j = Q_{1:j-1} (C U1) + Q_j (U2 U1) for ANY panel -- so for a panel with a component
 * G = Q_{1:j-1}^T A_j along the earlier panels, R_{1:j-1,j} gains exactly G (in exact
 * arithmetic), which is what tests pin.  `panel` (1-based) labels a breakdown. */
int orc_mcqr2gs_panel(double* X, int64_t ldx, int64_t m, int64_t c0, int64_t bj, double* R, int64_t ldr,
                      int panel, orc_info* info) {
  double* Xj = X + c0 * ldx;
  double* U1 = (double*)malloc(sizeof(double) * (size_t)(bj * bj));
  double* U2 = (double*)malloc(sizeof(double) * (size_t)(bj * bj));
  double* C = (double*)malloc(sizeof(double) * (size_t)((c0 > 0 ? c0 : 1) * bj));
  int rc = ORC_OK;
  if (!U1 || !U2 || !C) { rc = fail(info, ORC_ERR_NOMEM, 0, 0, 0); goto done; }
  /* l.6 */
  rc = cqr(Xj, ldx, m, bj, U1, bj, info);
  if (rc != ORC_OK) { rc = fail(info, rc, 1, panel, 1); goto done; }
  /* l.7 */
  if (c0 > 0) {
    rc = orc_atb(X, ldx, Xj, ldx, m, c0, bj, C, c0);
    if (rc != ORC_OK) goto done;
    orc_sub_prod(Xj, ldx, X, ldx, C, c0, m, c0, bj);
  }
  /* l.8 */
  rc = cqr(Xj, ldx, m, bj, U2, bj, info);
  if (rc != ORC_OK) { rc = fail(info, rc, 1, panel, 2); goto done; }
  /* R assembly (R-8) */
  orc_matmul(U2, bj, U1, bj, bj, bj, bj, R + c0 + c0 * ldr, ldr, 1, 0);
  if (c0 > 0) orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1);
done:
  free(U1); free(U2); free(C);
  return rc;
}

/* mCQR2GS(X, b) (Alg. 8; R-6, R-7, R-8):
 *   [Q_1, R_11] = CQR2(A_1)                                     (l.1)
 *   for j = 2..k:
 *     Y = Q_{j-1}^T A_{:,j:k};  A_{:,j:k} -= Q_{j-1} Y           (l.3-4)
 *     R_{j-1,j:k} = Y                                             (l.5)
 *     lines 6-8 and R_jj, R_{1:j-1,j}: orc_mcqr2gs_panel above      (l.6-8)  */
static int mcqr2gs(double* X, int64_t ldx, int64_t m, int64_t n, int64_t b, double* R, int64_t ldr,
                   orc_info* info) {
  int64_t k = (n + b - 1) / b;
  int64_t b0 = (b <= n) ? b : n;
  int rc = cqr2_block(X, ldx, m, b0, R, ldr, 1, 1, info);
  if (rc != ORC_OK) return rc;
  for (int64_t j = 1; j < k; ++j) {
    int64_t c0 = j * b, bj = (c0 + b <= n) ? b : n - c0;
    int64_t cp = c0 - b; /* previous panel, width b */
    /* l.3-5 */
    double* Y = R + cp + c0 * ldr;
    rc = orc_atb(X + cp * ldx, ldx, X + c0 * ldx, ldx, m, b, n - c0, Y, ldr);
    if (rc != ORC_OK) break;
    orc_sub_prod(X + c0 * ldx, ldx, X + cp * ldx, ldx, Y, ldr, m, b, n - c0);
    /* l.6-8 + R assembly */
    rc = orc_mcqr2gs_panel(X, ldx, m, c0, bj, R, ldr, (int)j + 1, info);
    if (rc != ORC_OK) break;
  }
  return rc;
}

/* Cholesky diagonal ratio rho = max_i U_ii / min_i U_ii of an upper-triangular U with positive
 * diagonal: a LOWER bound of kappa_2(U) (U_ii are the norms of the panel's columns after
 * orthogonalisation against the previous ones), SURVEY NEXT-f4's suggested indicator. */
double orc_diag_ratio(const double* U, int64_t ldu, int64_t b) {
  double mx = U[0], mn = U[0];
  for (int64_t i = 1; i < b; ++i) {
    const double d = U[i + i * ldu];
    if (d > mx) mx = d;
    if (d < mn) mn = d;
  }
  return mx / mn;
}

/* Frobenius condition estimate kappa_F(U) = ||U||_F ||U^{-1}||_F of an upper-triangular U:
 * an UPPER bound of kappa_2(U) (within a factor b of it), from the explicit inverse
 * (orc_tri_inv) -- the quantity the adaptive rule uses (R-23). */
double orc_kappa_f(const double* U, int64_t ldu, int64_t b) {
  double* Z = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!Z) return INFINITY;
  orc_tri_inv(U, ldu, b, Z, b);
  double su = 0.0, sz = 0.0;
  for (int64_t j = 0; j < b; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      su += U[i + j * ldu] * U[i + j * ldu];
      sz += Z[i + j * b] * Z[i + j * b];
    }
  free(Z);
  return sqrt(su) * sqrt(sz);
}

/* The adaptive rule's estimate of the loss of orthogonality one CholeskyQR leaves on panel j
 * (R-23): with Z = U1^{-1} (orc_tri_inv),
 *   own    = u nu(U1)^2 nu(Z)^2            (u kappa(V)^2)
 *   across = u nu(R_{1:j,j}) nu(Z)         (the projection of l.3-4 leaves ~u ||A_j|| along the
 *                                           earlier panels, A_j = Q R_{1:j,j}; the CQR scales it
 *                                           by U1^{-1}: CQRGS's loss of orthogonality)
 * with nu(M) = ||M||_F / sqrt(b), the RMS singular value (1 for an orthonormal panel).
 * E_j = max(own, across).  Rcol points at R_{1,j} (rows 0..c0-1 hold R_{1:j-1,j} = the line-5
 * projections Y of the earlier steps), leading dimension ldr. */
double orc_adapt_estimate(const double* U1, int64_t b, const double* Rcol, int64_t ldr, int64_t c0) {
  double* Z = (double*)malloc(sizeof(double) * (size_t)(b * b));
  if (!Z) return INFINITY;
  orc_tri_inv(U1, b, b, Z, b);
  double su = 0.0, sz = 0.0, sy = 0.0;
  for (int64_t j = 0; j < b; ++j) {
    for (int64_t i = 0; i <= j; ++i) {
      su += U1[i + j * b] * U1[i + j * b];
      sz += Z[i + j * b] * Z[i + j * b];
    }
    for (int64_t i = 0; i < c0; ++i) sy += Rcol[i + j * ldr] * Rcol[i + j * ldr];
  }
  free(Z);
  /* RMS singular values nu(M) = ||M||_F / sqrt(b): 1 for an orthonormal panel, whatever b */
  const double bb = (double)b;
  const double own = ORC_UNIT_ROUNDOFF * (su / bb) * (sz / bb);
  const double across = ORC_UNIT_ROUNDOFF * sqrt((sy + su) / bb) * sqrt(sz / bb);
  return own > across ? own : across;
}

/* Adaptive mCQR2GS ("the condition number steeply decreases as we
 * proceed with the panel processing, opening up a space for further optimisation in reducing
 * the number of flops by applying a runtime decision on how many repetitions of CholeskyQR to
 * perform"; reading R-23).  Alg. 8 with one decision per panel, taken after the panel's FIRST
 * CholeskyQR (U1 = chol(W1), W1 the allreduced Gram -- identical on every rank):
 *     rho_j = orc_diag_ratio(U1)
 *     rho_j <= tau:  the repetition is skipped -- panel 1: no second CQR of l.1, R_11 = U1;
 *                    panel j >= 2: lines 7-8 skipped, R_jj = U1 (R_{1:j-1,j} keeps Y);
 *     otherwise:     Alg. 8 unchanged (second CQR; l.7-8 and R-8 bookkeeping).
 * One CholeskyQR leaves ||Q^T Q - I|| ~ u kappa(panel)^2, so tau bounds the
 * estimated loss by ~u tau^2.  tau = 0 never skips: bitwise mCQR2GS.  tau = +inf always
 * skips: bitwise CQRGS (Alg. 7), whose per-panel steps are then the same operations in the same
 * order.  Panels skipped: orc_adapt_skipped(). */
static int mcqr2gs_adaptive(double* X, int64_t ldx, int64_t m, int64_t n, int64_t b, double* R, int64_t ldr,
                            orc_info* info) {
  int64_t k = (n + b - 1) / b;
  g_adapt_skipped = 0;
  double* U1 = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* U2 = (double*)malloc(sizeof(double) * (size_t)(b * b));
  double* C = (double*)malloc(sizeof(double) * (size_t)(n * b));
  int rc = ORC_OK;
  if (!U1 || !U2 || !C) { rc = fail(info, ORC_ERR_NOMEM, 0, 0, 0); goto done; }
  for (int64_t j = 0; j < k; ++j) {
    int64_t c0 = j * b, bj = (c0 + b <= n) ? b : n - c0;
    double* Xj = X + c0 * ldx;
    if (j > 0) { /* l.3-5 */
      int64_t cp = c0 - b;
      double* Y = R + cp + c0 * ldr;
      rc = orc_atb(X + cp * ldx, ldx, Xj, ldx, m, b, n - c0, Y, ldr);
      if (rc != ORC_OK) goto done;
      orc_sub_prod(Xj, ldx, X + cp * ldx, ldx, Y, ldr, m, b, n - c0);
    }
    /* first CQR: l.1 (first half) / l.6 */
    rc = cqr(Xj, ldx, m, bj, U1, bj, info);
    if (rc != ORC_OK) { rc = fail(info, rc, 1, (int)j + 1, 1); goto done; }
    if (orc_adapt_estimate(U1, bj, R + c0 * ldr, ldr, c0) <= g_adapt_tau) { /* skipped: R_jj = U1 */
      ++g_adapt_skipped;
      for (int64_t jj = 0; jj < bj; ++jj)
        for (int64_t ii = 0; ii <= jj; ++ii) R[c0 + ii + (c0 + jj) * ldr] = U1[ii + jj * bj];
      continue;
    }
    if (c0 > 0) { /* l.7 */
      rc = orc_atb(X, ldx, Xj, ldx, m, c0, bj, C, c0);
      if (rc != ORC_OK) goto done;
      orc_sub_prod(Xj, ldx, X, ldx, C, c0, m, c0, bj);
    }
    rc = cqr(Xj, ldx, m, bj, U2, bj, info); /* second CQR: l.1 (second half) / l.8 */
    if (rc != ORC_OK) { rc = fail(info, rc, 1, (int)j + 1, 2); goto done; }
    orc_matmul(U2, bj, U1, bj, bj, bj, bj, R + c0 + c0 * ldr, ldr, 1, 0);   /* R_jj = U2 U1 */
    if (c0 > 0) orc_matmul(C, c0, U1, bj, c0, bj, bj, R + c0 * ldr, ldr, 0, 1); /* R-8 */
  }
done:
  free(U1); free(U2); free(C);
  return rc;
}

/* Top-level factorisation.  A (m x n, lda >= m) is overwritten with Q; R (n x n,
 * ldr >= n) receives the upper-triangular factor with exact zeros below the
 * diagonal.  b is the panel width (ignored for CQR / CQR2).  Returns ORC_OK,
 * ORC_ERR_ARG, ORC_ERR_BREAKDOWN (details in *info) or ORC_ERR_NOMEM.          */
int orc_factor(double* A, int64_t lda, int64_t m, int64_t n, int64_t b, int algo, double* R,
               int64_t ldr, orc_info* info) {
  if (info) memset(info, 0, sizeof(*info));
  if (!A || !R || m < n || n < 1 || lda < m || ldr < n) return fail(info, ORC_ERR_ARG, 0, 0, 0);
  if ((algo == ORC_CQR2GS || algo == ORC_MCQR2GS || algo == ORC_CQRGS || algo == ORC_MCQR2GS_ADAPTIVE) &&
      (b < 1 || b > n))
    return fail(info, ORC_ERR_ARG, 0, 0, 0);
  zero_mat(R, ldr, n, n);
  int rc = ORC_OK;
  switch (algo) {
    case ORC_CQR: {
      rc = cqr(A, lda, m, n, R, ldr, info);
      if (rc != ORC_OK) rc = fail(info, rc, 1, 1, 1);
      break;
    }
    case ORC_CQR2:
      rc = cqr2_block(A, lda, m, n, R, ldr, 1, 1, info);
      break;
    case ORC_CQRGS:
      rc = cqrgs(A, lda, m, n, b, R, ldr, 1, info);
      break;
    case ORC_CQR2GS: {
      /* R1 = CQRGS(A); R2 = CQRGS(Q1); R = R2 R1 (same b in both passes, R-10) */
      double* R1 = (double*)calloc((size_t)(n * n), sizeof(double));
      double* R2 = (double*)calloc((size_t)(n * n), sizeof(double));
      if (!R1 || !R2) { free(R1); free(R2); return fail(info, ORC_ERR_NOMEM, 0, 0, 0); }
      rc = cqrgs(A, lda, m, n, b, R1, n, 1, info);
      if (rc == ORC_OK) rc = cqrgs(A, lda, m, n, b, R2, n, 2, info);
      if (rc == ORC_OK) orc_matmul(R2, n, R1, n, n, n, n, R, ldr, 1, 0);
      free(R1); free(R2);
      break;
    }
    case ORC_MCQR2GS:
      rc = mcqr2gs(A, lda, m, n, b, R, ldr, info);
      break;
    case ORC_MCQR2GS_ADAPTIVE:
      rc = mcqr2gs_adaptive(A, lda, m, n, b, R, ldr, info);
      break;
    case ORC_SCQR: {
      rc = scqr(A, lda, m, n, R, ldr, info, ORC_UNIT_ROUNDOFF);
      if (rc != ORC_OK) rc = fail(info, rc, 1, 1, 1);
      break;
    }
    case ORC_SCQR3: {
      /* sCQR3 (Alg. 5): [Q1, R1] = sCQR(A); [Q, R2] = CQR2(Q1); R = R2 R1.
       * Breakdown stages: 1 = the shifted CQR, 2 and 3 = the two CQRs of CQR2. */
      double* R1 = (double*)calloc((size_t)(n * n), sizeof(double));
      double* R2 = (double*)calloc((size_t)(n * n), sizeof(double));
      if (!R1 || !R2) { free(R1); free(R2); return fail(info, ORC_ERR_NOMEM, 0, 0, 0); }
      rc = scqr(A, lda, m, n, R1, n, info, ORC_UNIT_ROUNDOFF);
      if (rc != ORC_OK) {
        rc = fail(info, rc, 1, 1, 1);
      } else {
        rc = cqr2_block(A, lda, m, n, R2, n, 1, 1, info);
        if (rc == ORC_ERR_BREAKDOWN && info) info->stage += 1;
      }
      if (rc == ORC_OK) orc_matmul(R2, n, R1, n, n, n, n, R, ldr, 1, 0);
      free(R1); free(R2);
      break;
    }
    default:
      return fail(info, ORC_ERR_ARG, 0, 0, 0);
  }
  if (info) info->status = rc;
  return rc;
}

/* ------------------------------------------------------------------------- */
/* Householder QR (the plain definition of the thin QR): used  */
/* only as a pin on small well-conditioned inputs.  Q (m x n) explicit, R with  */
/* a non-negative diagonal (sign-normalised).                            */
/* ------------------------------------------------------------------------- */
int orc_householder(const double* A, int64_t lda, int64_t m, int64_t n, double* Q, int64_t ldq,
                    double* R, int64_t ldr) {
  if (m < n) return ORC_ERR_ARG;
  double* W = (double*)malloc(sizeof(double) * (size_t)(m * n));
  double* V = (double*)malloc(sizeof(double) * (size_t)(m * n));
  double* beta = (double*)malloc(sizeof(double) * (size_t)n);
  if (!W || !V || !beta) { free(W); free(V); free(beta); return ORC_ERR_NOMEM; }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) W[i + j * m] = A[i + j * lda];
  for (int64_t kk = 0; kk < n; ++kk) {
    /* v = x + sign(x0) ||x|| e0, H = I - beta v v^T */
    double nrm = 0.0;
    for (int64_t i = kk; i < m; ++i) nrm += W[i + kk * m] * W[i + kk * m];
    nrm = sqrt(nrm);
    double x0 = W[kk + kk * m];
    double alpha = (x0 >= 0.0) ? -nrm : nrm;
    for (int64_t i = 0; i < m; ++i) V[i + kk * m] = 0.0;
    for (int64_t i = kk; i < m; ++i) V[i + kk * m] = W[i + kk * m];
    V[kk + kk * m] -= alpha;
    double vv = 0.0;
    for (int64_t i = kk; i < m; ++i) vv += V[i + kk * m] * V[i + kk * m];
    beta[kk] = (vv > 0.0) ? 2.0 / vv : 0.0;
    for (int64_t j = kk; j < n; ++j) {
      double s = 0.0;
      for (int64_t i = kk; i < m; ++i) s += V[i + kk * m] * W[i + j * m];
      s *= beta[kk];
      for (int64_t i = kk; i < m; ++i) W[i + j * m] -= s * V[i + kk * m];
    }
  }
  /* R = upper part of W; Q = H_1 ... H_n [I_n; 0] */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) R[i + j * ldr] = (i <= j) ? W[i + j * m] : 0.0;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  for (int64_t kk = n - 1; kk >= 0; --kk) {
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t i = kk; i < m; ++i) s += V[i + kk * m] * Q[i + j * ldq];
      s *= beta[kk];
      for (int64_t i = kk; i < m; ++i) Q[i + j * ldq] -= s * V[i + kk * m];
    }
  }
  /* sign normalisation: make diag(R) >= 0 */
  for (int64_t i = 0; i < n; ++i) {
    if (R[i + i * ldr] < 0.0) {
      for (int64_t j = i; j < n; ++j) R[i + j * ldr] = -R[i + j * ldr];
      for (int64_t r = 0; r < m; ++r) Q[r + i * ldq] = -Q[r + i * ldq];
    }
  }
  free(W); free(V); free(beta);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Metrics evaluated in double-double (TwoSum / TwoProd via fma, which  */
/* is exact), so the verifier's own error is far below the 1e-13 / 1e-14 gates. */
/* ------------------------------------------------------------------------- */
typedef struct { double hi, lo; } dd;

static inline dd dd_add_d(dd a, double b) {
  double s = a.hi + b;
  double bb = s - a.hi;
  double e = (a.hi - (s - bb)) + (b - bb);
  e += a.lo;
  double h = s + e;
  dd r = {h, e - (h - s)};
  return r;
}
static inline dd dd_add(dd a, dd b) {
  double s = a.hi + b.hi;
  double bb = s - a.hi;
  double e = (a.hi - (s - bb)) + (b.hi - bb);
  e += a.lo + b.lo;
  double h = s + e;
  dd r = {h, e - (h - s)};
  return r;
}
static inline dd dd_prod(double a, double b) {
  double p = a * b;
  dd r = {p, fma(a, b, -p)};
  return r;
}

/* ||Q^T Q - I||_F (un-normalised; divide by sqrt(n) for the paper's P:104 form).
 * Each entry (Q^T Q)_ij is accumulated in double-double over all rows; the
 * difference from delta_ij and the squares are formed in double-double. */
double orc_orthogonality(const double* Q, int64_t ldq, int64_t m, int64_t n) {
  dd total = {0.0, 0.0};
  int64_t npairs = n * (n + 1) / 2;
  double* part = (double*)malloc(sizeof(double) * 2 * (size_t)npairs);
  if (!part) return NAN;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t i = 0; i <= j; ++i) {
      dd s = {0.0, 0.0};
      const double* qi = Q + i * ldq;
      const double* qj = Q + j * ldq;
      for (int64_t r = 0; r < m; ++r) s = dd_add(s, dd_prod(qi[r], qj[r]));
      if (i == j) s = dd_add_d(s, -1.0);
      int64_t t = j * (j + 1) / 2 + i;
      part[2 * t] = s.hi;
      part[2 * t + 1] = s.lo;
    }
  }
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      int64_t t = j * (j + 1) / 2 + i;
      double e = part[2 * t] + part[2 * t + 1];
      dd sq = dd_prod(e, e);
      if (i != j) sq = dd_add(sq, sq);
      total = dd_add(total, sq);
    }
  free(part);
  return sqrt(total.hi + total.lo);
}

/* ||A - Q R||_F / ||A||_F; (QR)_rc accumulated in double-double. */
double orc_residual(const double* A, int64_t lda, const double* Q, int64_t ldq, const double* R,
                    int64_t ldr, int64_t m, int64_t n) {
  dd num = {0.0, 0.0}, den = {0.0, 0.0};
  int nt = g_threads;
  double* pn = (double*)calloc((size_t)(4 * nt), sizeof(double));
  if (!pn) return NAN;
#pragma omp parallel num_threads(nt)
  {
    dd ln = {0.0, 0.0}, ld = {0.0, 0.0};
#pragma omp for schedule(static)
    for (int64_t r = 0; r < m; ++r) {
      for (int64_t c = 0; c < n; ++c) {
        dd s = {0.0, 0.0};
        for (int64_t t = 0; t <= c; ++t) s = dd_add(s, dd_prod(Q[r + t * ldq], R[t + c * ldr]));
        double a = A[r + c * lda];
        dd diff = dd_add_d(s, -a);
        double e = diff.hi + diff.lo;
        ln = dd_add(ln, dd_prod(e, e));
        ld = dd_add(ld, dd_prod(a, a));
      }
    }
    int tid = omp_get_thread_num();
    pn[4 * tid] = ln.hi; pn[4 * tid + 1] = ln.lo; pn[4 * tid + 2] = ld.hi; pn[4 * tid + 3] = ld.lo;
  }
  for (int t = 0; t < nt; ++t) {
    dd a = {pn[4 * t], pn[4 * t + 1]}, b = {pn[4 * t + 2], pn[4 * t + 3]};
    num = dd_add(num, a);
    den = dd_add(den, b);
  }
  free(pn);
  return sqrt((num.hi + num.lo) / (den.hi + den.lo));
}
