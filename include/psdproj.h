/*
 * psdproj.h — C ABI of libpsdproj.so, the B200 (sm_100a) randomized
 * PSD-cone projection.  Plain pointers and sizes only; every array argument
 * is a DEVICE pointer on the plan's device, row-major, with the given leading
 * dimension (in elements).  Calls are enqueued on `stream` (a cudaStream_t;
 * NULL = legacy default stream) and synchronise with it only where the
 * algorithm needs a host decision (symmetry verdict, CholeskyQR breakdown,
 * rank truncation, effective rank), exactly where the reference raises or
 * branches.
 *
 * Each entry point replaces one function of the reference `psdcone` package
 * (/root/reference/pkg/src/psdcone, cited file:line below); INTEGRATION.md
 * shows the ctypes binding a psdcone maintainer would add.
 */
#ifndef PSDPROJ_H
#define PSDPROJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, 1:1 with the reference exception hierarchy (errors.py:4-49). */
enum psd_status {
  PSD_OK = 0,
  PSD_ERR_INVALID_PARAMS = 1,  /* InvalidParams          errors.py:28 */
  PSD_ERR_ASYMMETRIC = 2,      /* AsymmetricMatrixError  errors.py:12 */
  PSD_ERR_RANK_DEFICIENT = 3,  /* RankDeficientSample    errors.py:20 */
  PSD_ERR_ALPHA_TOO_SMALL = 4, /* AlphaTooSmall          errors.py:24 */
  PSD_ERR_CONVERGENCE = 5,     /* ConvergenceFailure     errors.py:16 */
  PSD_ERR_NONSQUARE = 6,       /* NonSquareError         errors.py:8  */
  PSD_ERR_CUDA = 7,            /* CUDA runtime failure (no reference analogue) */
  PSD_ERR_NO_MEMORY = 8        /* device allocation failed */
};

/* flags for psd_ran_proj / psd_range_finder */
#define PSD_FLAG_DIAGNOSTICS 1u   /* residual_frob = ||X - Q Q^T X||_F   (projection.py:109-110) */
#define PSD_FLAG_STRICT 2u        /* RankDeficientSample instead of truncation (sketch.py:86-92) */
#define PSD_FLAG_SKIP_SYMCHECK 4u /* caller already ran psd_require_symmetric on X */
#define PSD_FLAG_ASSUME_SYMMETRIC 8u /* X is bitwise symmetric: X^T·P computed as X·P */
#define PSD_FLAG_FP64_DMMA 16u     /* keep the FP64 n x n products on the DMMA kernel (no INT8 emulation) */
#define PSD_FLAG_FP64_INT8 32u     /* INT8-emulated FP64 products at any n (default: n >= 3072) */

typedef struct psd_plan psd_plan;

/* Stages timed by psd_plan_profile (CUDA events on the caller's stream). */
enum psd_stage {
  PSD_STAGE_SYMCHECK = 0,    /* require_symmetric pass                       */
  PSD_STAGE_SKETCH_GEMM = 1, /* each op(X)·P product (n x n · n x w), DMMA     */
  PSD_STAGE_QR = 2,          /* CholeskyQR (Gram, Cholesky, inverse, apply)  */
  PSD_STAGE_COMPRESS = 3,    /* T = Q^T (X Q)                                */
  PSD_STAGE_EIGH = 4,        /* block-Jacobi eigensolve + sort               */
  PSD_STAGE_RECON = 5,       /* W = Q U, mirrored SYRK reconstruction        */
  PSD_STAGE_DIAG = 6,        /* residual diagnostics                         */
  PSD_STAGE_TOTAL = 7,       /* whole psd_ran_proj call                      */
  PSD_STAGE_INT8_GEMM = 8,   /* INT8 tensor-core kernel inside an emulated FP64 sketch product */
  PSD_NUM_STAGES = 9
};

typedef struct psd_report {
  int32_t effective_rank;  /* ProjectionReport.effective_rank (projection.py:115) */
  int32_t basis_width;     /* ProjectionReport.basis_width    (projection.py:118) */
  int32_t used_transpose;  /* 1 if X^T multiplies ran on the transposed-operand kernel */
  int32_t qr_passes;       /* CholeskyQR passes of the final orthonormalisation */
  int32_t qr_shifted;      /* 1 if a shifted CholeskyQR pass was needed */
  int32_t eig_sweeps;      /* block-Jacobi sweeps of the k x k eigensolve */
  int32_t gpu_launches;    /* kernels this call launched */
  int32_t sketch_engine;   /* n x n products ran on: 0 FP64 DMMA, 1 INT8-emulated FP64 (Ozaki II),
                              2 3xTF32, 3 X·P on INT8 and X^T·P on DMMA (X not bitwise symmetric) */
  double residual_frob;    /* PSD_FLAG_DIAGNOSTICS only, else NaN */
  double max_abs;          /* max|x_ij| (symmetric.py:51) */
  double sym_defect;       /* max|x_ij - x_ji| (symmetric.py:52) */
  double alpha_used;       /* alpha (ran_proj_scal) or 0 */
  int32_t recon_engine;    /* reconstruction SYRK ran on: 0 FP64 DMMA (or 3xTF32 for FP32),
                              1 INT8 tensor cores (Ozaki I digit slices, ozaki_syrk.cu) */
  int32_t reserved0;
} psd_report;

/* Thread-local description of the last non-OK status. */
const char* psd_last_error(void);
const char* psd_version(void);

/* Workspace for problems with dimension <= n and sketch width <= width on
 * `device`.  A plan is not thread-safe; use one per host thread / stream. */
int psd_plan_create(psd_plan** plan, int64_t n, int32_t width, int32_t device);
void psd_plan_destroy(psd_plan* plan);
/* Bytes of device memory the plan holds. */
int64_t psd_plan_bytes(const psd_plan* plan);
/* Stage profiling.  enable: 1 on, 0 off, -1 unchanged.  When ms_out /
 * counts_out (HOST, PSD_NUM_STAGES each) are non-NULL they receive the
 * accumulated milliseconds / event pairs per psd_stage; reset != 0 zeroes
 * the accumulators afterwards. */
int psd_plan_profile(psd_plan* plan, int32_t enable, double* ms_out, int32_t* counts_out,
                     int32_t reset);
/* Pipelining hint for a batch of projections (C3's 16 sequential projections;
 * the reference projects one matrix per call, projection.py:92-119): the NEXT
 * psd_ran_proj call on this plan will project x_next (n x n FP64, device,
 * leading dimension ldx).  That call starts x_next's require_symmetric pass
 * and its INT8-engine residue planes on a low-priority side stream once its
 * own n x n products are done, so they run under its latency-bound CholeskyQR
 * and eigensolver; the call after it consumes them (same pointer, n, ldx)
 * instead of reading X again.  Results are identical to unhinted calls; the
 * caller must not modify x_next until it has been projected.  The hint is
 * used by exactly one call (NULL clears it); FP32 / DMMA-engine calls ignore it. */
int psd_plan_prefetch(psd_plan* plan, const double* x_next, int64_t n, int64_t ldx);
/* The same for the FP32 path (psd_ran_proj_f32): x_next's require_symmetric pass fused with
 * its tf32 split runs on the side stream under the current call's QR / eigensolver. */
int psd_plan_prefetch_f32(psd_plan* plan, const float* x_next, int64_t n, int64_t ldx);

/* require_symmetric — symmetric.py:39-57.  tol < 0 selects the reference
 * default 1e-10*max(1, max|x|).  stats_out (HOST, 3 doubles) receives
 * {max|x|, max|x - x^T|, 1.0 if bitwise symmetric else 0.0}. */
int psd_require_symmetric(psd_plan* plan, const double* x, int64_t n, int64_t ldx, double tol,
                          double* stats_out, void* stream);

/* power_iteration — sketch.py:96-114: exactly n_iter normalised products of
 * (X - shift*I) from v0 (device, length n), returns ||(X - shift I) v||_2, or
 * 0 when an iterate is annihilated.  result: HOST double. */
int psd_power_iteration(psd_plan* plan, const double* x, int64_t n, int64_t ldx, double shift,
                        const double* v0, int32_t n_iter, double* result, void* stream);

/* min_eig_magnitude — sketch.py:117-129 (Alg. 5) with start vectors v1, v2. */
int psd_min_eig_magnitude(psd_plan* plan, const double* x, int64_t n, int64_t ldx,
                          const double* v1, const double* v2, int32_t n_iter, double* result,
                          void* stream);
/* The same with flags: PSD_FLAG_ASSUME_SYMMETRIC (the caller verified X bitwise symmetric, as
 * project() does with require_symmetric first, projection.py:189) lets every product read only
 * X's lower triangle (n % 64 == 0): half the HBM bytes of the 2(N+1) passes. */
int psd_min_eig_magnitude_ex(psd_plan* plan, const double* x, int64_t n, int64_t ldx,
                             const double* v1, const double* v2, int32_t n_iter, uint32_t flags,
                             double* result, void* stream);

/* range_finder — sketch.py:53-93: basis (m x width, ld ldb) of the range of
 * (X X^T)^q X Omega for an m x n X, Omega = omega (n x width, ld ldo).  alpha > 0 sketches
 * B = (X + alpha I)/alpha instead (projection.py:139-140).  *width_out =
 * number of columns kept by the 1e-12*||Y||_F truncation. */
int psd_range_finder(psd_plan* plan, const double* x, int64_t m, int64_t n, int64_t ldx,
                     const double* omega, int64_t ldo, int32_t width, int32_t q, double alpha,
                     uint32_t flags, double* basis, int64_t ldb, int32_t* width_out,
                     void* stream);

/* eigh — symmetric.py:68-86 for an m x m symmetric matrix: values descending,
 * each vector's largest-|entry| positive.  a is overwritten. */
int psd_eigh(psd_plan* plan, double* a, int32_t m, int64_t lda, double* values, double* vectors,
             int64_t ldv, int32_t* sweeps_out, void* stream);

/* ran_proj (alpha == 0) — projection.py:92-119, Alg. 2;
 * ran_proj_scal (alpha > 0) — projection.py:122-159, Alg. 3.
 * omega: n x (k+l) Gaussian test matrix (ld ldo) — the reference's draw at
 * sketch.py:75, passed in so both sides see identical inputs.
 * result: n x n (ld ldr) or NULL; factors_w: n x (k+l) (ld ldw) or NULL —
 * the first report->effective_rank columns receive W; factors_d: k+l or NULL.
 * report: HOST. */
int psd_ran_proj(psd_plan* plan, const double* x, int64_t n, int64_t ldx, const double* omega,
                 int64_t ldo, int32_t k, int32_t l, int32_t q, double alpha, uint32_t flags,
                 double* result, int64_t ldr, double* factors_w, int64_t ldw, double* factors_d,
                 psd_report* report, void* stream);

/* FP32 path of ran_proj / ran_proj_scal (BASELINE config 3 "fp32"; no
 * reference counterpart — the reference casts to float64 at sketch.py:66).
 * x, omega, result: fp32; every n x n product runs as 3xTF32 on the tcgen05
 * tensor cores (TMEM accumulators), the power scheme is always
 * re-orthonormalised, QR / eigh stay FP64.  Same flags and report as
 * psd_ran_proj (PSD_FLAG_DIAGNOSTICS is ignored: residual_frob = NaN). */
int psd_ran_proj_f32(psd_plan* plan, const float* x, int64_t n, int64_t ldx, const float* omega,
                     int64_t ldo, int32_t k, int32_t l, int32_t q, double alpha, uint32_t flags,
                     float* result, int64_t ldr, double* factors_w, int64_t ldw, double* factors_d,
                     psd_report* report, void* stream);

/* FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme II, 16 moduli;
 * test entry, allocates its own scratch): C (fp64, m x n) = A (m x k) · P (k x n),
 * all row-major, n <= 512. */
int psd_gemm_f64_ozaki(const double* a, int64_t lda, const double* p, int64_t ldp, int64_t m,
                       int64_t n, int64_t k, double* c, int64_t ldc, void* stream);

/* The same emulated FP64 GEMM for a general A streamed in row chunks, with a
 * caller-owned device workspace (replaces the DGEMM of sketch.py:75/:82 and
 * projection.py:104 for a row block X_g of a sharded X):
 * C = A·P, or C = (A·P + alpha·S)/alpha when alpha > 0 (B = (X+αI)/α with S the
 * rows of P matching the rows of A).  chunk_rows <= 0 picks 8192.  Panels wider
 * than 512 columns run as column groups of <= 512 (TMEM budget).
 * psd_gemm_f64_int8_ws_bytes reports the workspace size for (m, n, k, chunk_rows). */
int psd_gemm_f64_int8_ws_bytes(int64_t m, int64_t n, int64_t k, int64_t chunk_rows, int64_t* bytes);
int psd_gemm_f64_int8(const double* a, int64_t lda, const double* p, int64_t ldp, int64_t m, int64_t n,
                      int64_t k, double* c, int64_t ldc, double alpha, const double* s, int64_t lds,
                      void* ws, int64_t ws_bytes, int64_t chunk_rows, void* stream);

/* Reconstruction X = W diag(d) W^T (projection.py:72-78, d > 0) on the INT8
 * tensor cores (test entry, allocates its own scratch): V = W diag(sqrt d) split
 * into 7 signed base-128 int8 digit planes per row-scaled 49-bit integer, the
 * 28 digit products of level <= 6 accumulated exactly in s32 TMEM, levels
 * combined in FP64; lower 128x32 tiles stored twice (bitwise-symmetric result).
 * W n x r row-major (r <= 640), result n x n. */
int psd_syrk_f64_int8(const double* w, int64_t ldw, const double* d, int64_t n, int32_t r,
                      double* result, int64_t ldr, void* stream);

/* The 3xTF32 tcgen05 GEMM itself (test entry; allocates its own scratch):
 * mode 0: C (fp64, m x n) = A · B^T; mode 1: mirrored fp32 C (m == n) from
 * the lower tiles of A · B^T; mode 2: as mode 0 with `a` given transposed
 * (k x m, ld lda — the M-contiguous operand path the FP32 projection uses).
 * A m x k, B n x k, fp32 row-major. */
int psd_gemm_tf32x3(int32_t mode, const float* a, int64_t lda, const float* b, int64_t ldb,
                    int64_t m, int64_t n, int64_t k, void* c, int64_t ldc, void* stream);

/* Dense X = sym(W diag(d) W^T) for W n x r (ld ldw), d[r] — the reconstruction
 * of projection.py:72-78 (and of exact_psd_projection, symmetric.py:109-114):
 * lower tiles on the FP64 tensor cores, each tile stored twice (mirrored). */
int psd_reconstruct(psd_plan* plan, const double* w, int64_t n, int64_t ldw, const double* d,
                    int32_t r, double* result, int64_t ldr, void* stream);

/* symmetrize — symmetric.py:31-36, in place: a <- (a + a^T)/2 (m x m). */
int psd_symmetrize(double* a, int64_t m, int64_t lda, void* stream);

/* The FP64 DMMA GEMM itself: C (M x N) = op_A · op_B with
 * a_layout 0: A[m*lda + k] (row-major M x K), 1: A[k*lda + m] (A^T stored);
 * b_layout 0: B[k*ldb + n] (row-major K x N), 1: B[n*ldb + k] (B^T stored);
 * epilogue 0: C = acc; 1: C = (acc + alpha*S)/alpha; 2: C = S - acc;
 *          3: mirrored lower-tile store (M == N, a_layout 0, b_layout 1).
 * ws/ws_elems: split-K scratch (may be NULL → no split). */
int psd_gemm_f64(int32_t a_layout, int32_t b_layout, const double* a, int64_t lda, const double* b,
                 int64_t ldb, double* c, int64_t ldc, int32_t m, int32_t n, int32_t k,
                 int32_t epilogue, double alpha, const double* s, int64_t lds, double* ws,
                 int64_t ws_elems, void* stream);

/* One CholeskyQR factor step on an m x m Gram matrix (m <= ~600):
 * L = chol(G + shift I) and, when no pivot failed, rinv = L^-T (upper).
 * status (DEVICE, 4 doubles) = {first failing pivot + 1 or 0, trace(G),
 * min L_ii, max L_ii}.  g is not modified. */
int psd_chol_inv(const double* g, int32_t m, int64_t ldg, double shift, double* l, int64_t ldl,
                 double* rinv, int64_t ldr, double* scratch, double* status, void* stream);

/* out[i][j] = w[i][j] * d[j] (i < rows, j < cols): the (w_kept * d_kept) of
 * projection.py:77. */
int psd_scale_columns(const double* w, int64_t ldw, const double* d, double* out, int64_t ldo,
                      int64_t rows, int32_t cols, void* stream);

/* out[0] = max |x_ij| over a rows x cols block (one HBM pass). */
int psd_max_abs(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                void* stream);

/* Rows [r0, r1) of the exactly symmetric n x n matrix S = lowtri-mirror(A·B^T)
 * (A, B: n x k, 16-byte aligned, even ld): every value is computed once on a
 * lower tile and stored at (i,j) and (j,i), so row blocks produced by
 * different ranks assemble into a bitwise-symmetric matrix.  out: (r1-r0) x n. */
int psd_syrk_window(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t n,
                    int32_t k, int64_t r0, int64_t r1, double* out, int64_t ldo, void* stream);

/* out[i - r0][j] = beta·out[i - r0][j] + scale·z(min(i,j), max(i,j)) for rows
 * [r0, r0+rows), j < n: rows of a symmetric N(0,1) matrix keyed on (seed,
 * unordered index pair) — identical on every rank that generates them. */
int psd_fill_sym_gaussian(double* out, int64_t ldo, int64_t r0, int64_t rows, int64_t n,
                          uint64_t seed, double scale, double beta, void* stream);

/* Symmetry statistics of one block pair of a row-sharded X (require_symmetric,
 * symmetric.py:39-57, when X's (i,j) and (j,i) entries live on different ranks —
 * SURVEY §8(e)): a = X[rows_g, cols_h] (rows x cols), b = X[rows_h, cols_g]
 * (cols x rows).  Accumulates into the DEVICE array stats[3] = {max|x|,
 * max|a_ij - b_ji|, flags (1: not bitwise equal, 2: non-finite) stored as the
 * bits of an int in stats[2]}; reset != 0 zeroes stats first.  Asynchronous. */
int psd_pair_defect(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t rows,
                    int64_t cols, double* stats, int32_t reset, void* stream);

/* ---- solver loop (sdls.py:76-89, :221-245; BASELINE config 5) ---------- */
/* x = cr + Σ_i y_i A_i: x ← copy(cr) (n x n, the C/ρ term), then for every
 * distinct stored position p: x[pos[p]] += Σ_{t ∈ [ptr[p], ptr[p+1])}
 * y[econ[t]]·evals[t] in stored order (assemble_dual_matrix, sdls.py:83-89). */
int psd_sdls_assemble(const double* cr, int64_t n, const int64_t* pos, const int32_t* ptr,
                      const int32_t* econ, const double* evals, const double* y, int32_t npos,
                      double* x, void* stream);
/* t_i = Tr(A_i X₊) with X₊ = sym((W·D)·Wᵀ) evaluated on A_i's stored entries
 * (rows/cols/vals grouped by constraint, cptr[m+1]); wd = W·diag(d), n x r
 * (constraint_traces, sdls.py:76-80, on the factored projection). */
int psd_sdls_traces(const double* wd, const double* w, int64_t ldw, int32_t r, const int32_t* rows,
                    const int32_t* cols, const double* vals, const int32_t* cptr, int32_t m,
                    double* t, void* stream);
/* t_i = Tr(A_i X) = Σ v·X[row][col] over A_i's stored entries for a dense
 * n x n X (constraint_traces, sdls.py:76-80 — the exact / polar projectors). */
int psd_sdls_traces_dense(const double* x, int64_t ldx, const int32_t* rows, const int32_t* cols,
                          const double* vals, const int32_t* cptr, int32_t m, double* t,
                          void* stream);
/* grad = b − t; out[0] = ‖grad‖; if out[0] > eps: y += beta·grad (sdls.py:236-245). */
int psd_sdls_step(const double* b, const double* t, double* y, double* grad, int32_t m,
                  double beta, double eps, double* out, void* stream);

/* Device-side N(0,1) fill (Philox4x32-10 + Box-Muller) for callers that do
 * not need the reference's numpy stream (benchmarks, solver loops). */
int psd_fill_gaussian(double* out, int64_t rows, int32_t cols, int64_t ld, uint64_t seed,
                      uint64_t offset, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PSDPROJ_H */
