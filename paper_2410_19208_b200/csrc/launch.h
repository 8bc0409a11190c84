// Host-side launchers for the sm_100a kernels (internal to libpsdproj.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_f64.cuh"

namespace psd {

// Kernels launched by this library on the calling thread (reported to callers
// as psd_report.gpu_launches).
extern thread_local int g_launch_count;
inline void count_launch(int k = 1) { g_launch_count += k; }

struct DeviceInfo {
  int sms = 148;
  size_t max_smem = 227 * 1024;
};
const DeviceInfo& device_info();

// ---- GEMM (DMMA) ------------------------------------------------------------
struct GemmOp {
  int a_layout = A_MK, b_layout = B_KN;
  const double* A = nullptr;
  long long lda = 0;
  const double* B = nullptr;
  long long ldb = 0;
  double* C = nullptr;
  long long ldc = 0;
  int M = 0, N = 0, K = 0;
  int epi = EPI_STORE;
  double alpha = 1.0;
  const double* S = nullptr;
  long long lds = 0;
  double* partials = nullptr;  // EPI_RESID: one double per CTA
  int max_splits = 256;        // 1 forces a single pass (required for SUB/MIRROR/RESID)
  int win0 = 0, win1 = 0;      // EPI_MIRROR row window (win1 = 0 → all rows); TMA path only
};
// Launches the DMMA GEMM, splitting K when that shortens the critical path.
// `ws` must hold ws_elems doubles for split-K partials.  Returns the number
// of kernel launches issued (1 or 2), or <0 on error.
int gemm_f64(const GemmOp& op, double* ws, size_t ws_elems, cudaStream_t st);
// Number of partial sums a RESID launch may write (size of `partials`; zero it first).
long long gemm_resid_ctas(const GemmOp& op);
// TMA-fed warp-specialised path (gemm_tma.cu); −2 = operands not TMA-aligned.
int gemm_f64_tma(const GemmOp& op, double* ws, size_t ws_elems, cudaStream_t st);
long long gemm_tma_resid_parts(const GemmOp& op);

// ---- 3xTF32 tcgen05 GEMM (gemm_tc32.cu): C = A·Bᵀ, A M×K and B N×K fp32 -------
// operands given as tf32 hi/lo pairs (K contiguous, ld % 4 == 0, 16-B aligned).
struct Tc32Op {
  const float *a_hi = nullptr, *a_lo = nullptr;
  long long lda = 0;
  long long lda_lo = 0;       // 0: same as lda
  const float *b_hi = nullptr, *b_lo = nullptr;
  long long ldb = 0;
  int M = 0, N = 0, K = 0;
  int mode = 0;               // 0: fp64 result c64 (split-K partials in ws), 1: mirrored fp32 c32 (M == N)
  double* c64 = nullptr;
  long long ldc64 = 0;
  double alpha = 0.0;         // mode 0, α > 0: c64 = (acc + α·S)/α
  const double* S = nullptr;
  long long lds = 0;
  float* c32 = nullptr;
  long long ldc32 = 0;
  float* ws = nullptr;
  size_t ws_elems = 0;
  int max_splits = 8;
  bool a_mn = false;          // A given as Aᵀ (K×M row-major, ld lda): M-contiguous TMA loads
};
// ---- FP64 GEMM emulated on INT8 tensor cores (ozaki.cu): C (M×N) = A (M×K) · P (K×N) ----
// A is given as prepared residues (oz_prepare_rows): ar[ℓ][M][ldar] int8 + row exponents e[M].
struct OzOp {
  const int8_t* ar = nullptr;
  long long ldar = 0;
  const int* e = nullptr;
  const double* P = nullptr;   // K×N row-major fp64 panel
  long long ldp = 0;
  int M = 0, N = 0, K = 0;
  int8_t* br = nullptr;        // scratch: [16][round16(N)][ldbr] int8
  long long ldbr = 0;
  int* f = nullptr;            // scratch: N column exponents
  uint8_t* res = nullptr;      // scratch: residue partials
  size_t res_elems = 0;
  double* C = nullptr;
  long long ldc = 0;
  long long ar_rows = 0;       // rows per A residue plane (0: M) — a transposed panel as A
  double alpha = 0.0;          // α > 0: C = (acc + α·S)/α
  const double* S = nullptr;
  long long lds = 0;
  cudaEvent_t ev_gemm[2] = {nullptr, nullptr};   // optional: recorded around the INT8 kernel
};
// device→host read of a few status bytes that does not queue behind DMA copies
// (kernel store into host-mapped memory, then a stream sync); > 64 KB: cudaMemcpy
cudaError_t read_small(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t st);
cudaError_t read_small2(void* host_dst, const void* dev_src, size_t bytes, void* host_dst2, const void* dev_src2,
                        size_t bytes2, cudaStream_t st);
// enqueue a status read (≤ 4 KB) without draining the stream; collect with read_small_wait
cudaError_t read_small_async(const void* dev_src, size_t bytes, cudaStream_t st);
cudaError_t read_small_wait(void* host_dst, size_t bytes);
// copy a few device bytes into caller-owned host-mapped memory (its device alias) on `st`
void copy_to_mapped(void* mapped_dev_dst, const void* dev_src, size_t bytes, cudaStream_t st);
int oz_num_moduli();
long long oz_max_k();   // largest K the exact CRT reconstruction admits (2^18)
// residues of X's rows when the high words of max_j |x_ij| are already known (rowmax_hi,
// from sym_stats): one pass over X
// grid > 0: that many CTAs instead of the persistent default (short-lived CTAs for work on a
// low-priority side stream that must yield SMs to the caller's stream — the pipelined prefetch)
void oz_prepare_rows_max(const double* x, long long rows, long long cols, long long ldx,
                         const unsigned* rowmax_hi, int* e, int8_t* r, long long ldr, cudaStream_t st,
                         long long grid = 0, int threads = 256);
void oz_prepare_rows(const double* x, long long rows, long long cols, long long ldx, int* e, int8_t* r,
                     long long ldr, cudaStream_t st);
int oz_gemm(const OzOp& op, cudaStream_t st);
int oz_prepare_panel(const OzOp& op, cudaStream_t st);
int oz_gemm_prepared(const OzOp& op, cudaStream_t st);
size_t oz_stream_ws_bytes(long long m, long long n, long long k, long long chunk);
int oz_gemm_stream(const double* a, long long lda, const double* P, long long ldp, long long m, int n,
                   long long k, double* c, long long ldc, double alpha, const double* S, long long lds,
                   void* ws, size_t ws_bytes, long long chunk, cudaStream_t st);
// X̂₊ = W·diag(d)·Wᵀ (n×n, bitwise symmetric) on the INT8 tensor cores (ozaki_syrk.cu);
// W n×r (ld ldw), d[r] > 0; ws ≥ oz_syrk_ws_bytes(n, r).  0 ok, < 0 rejected.
size_t oz_syrk_ws_bytes(long long n, int r);
int oz_syrk(const double* w, long long n, int r, long long ldw, const double* d, double* c, long long ldc,
            void* ws, size_t ws_bytes, cudaStream_t st);
// Returns the K-split count used (≥ 1) or < 0 on error (−2 alignment, −3 workspace).
int gemm_tf32x3(const Tc32Op& op, cudaStream_t st);
long long tc32_ws_elems(long long M, int N, int max_splits);
// require_symmetric statistics of a square fp32 X (as sym_stats) fused with its tf32 hi/lo split;
// hi == nullptr (also for split_rows_f32): raw mode, X itself serves as hi, only lo is written.
void symsplit_f32(const float* x, long long n, long long ldx, double* stats, float* hi, float* lo,
                  long long ldh, cudaStream_t st, long long grid = 0);
void split_rows_f32(const float* x, long long rows, long long cols, long long ldx, float* hi,
                    float* lo, long long ldh, long long cols_pad, cudaStream_t st);
void split_rows_f64(const double* x, long long rows, int cols, long long ldx, const double* scale,
                    float* hi, float* lo, long long ldh, int cols_pad, cudaStream_t st);
void split_transpose(const double* P, long long n, int w, long long ldp, float* hi, float* lo,
                     long long ldt, int w_rows, cudaStream_t st);

// ---- memory-bound kernels --------------------------------------------------
// stats[0] = max|x|, stats[1] = max|x - xᵀ|, ((int*)(stats+2))[0] = flags
// (bit0: not bitwise symmetric, bit1: NaN/Inf present). stats zeroed inside.
void pair_defect(const double* a, long long lda, const double* b, long long ldb, long long rows,
                 long long cols, double* stats, bool reset, cudaStream_t st);
void sym_stats(const double* x, long long n, long long ldx, double* stats, cudaStream_t st,
               unsigned* rowmax = nullptr, long long grid = 0);
// out[0] = max |G − I| over a w×w Gram (single block)
void identity_defect(const double* g, int w, long long ldg, double* out, cudaStream_t st);
void sym_stats_f32(const float* x, long long n, long long ldx, double* stats, cudaStream_t st);
void convert_f32_f64(const float* src, long long lds, double* dst, long long ldd, long long rows,
                     int cols, cudaStream_t st);
// x ← (x + xᵀ)/2 for a small m×m matrix (in place, exact mirror).
void symmetrize_small(double* x, int m, long long ld, cudaStream_t st);
void philox_normal(double* out, long long rows, int cols, long long ld, uint64_t seed,
                   uint64_t offset, cudaStream_t st);
// rows [r0, r0+rows) of a symmetric N(0,1) matrix keyed on (seed, min(i,j), max(i,j))
void sym_gaussian_rows(double* out, long long ldo, long long r0, long long rows, long long n,
                       uint64_t seed, double scale, double beta, cudaStream_t st);
// y = (X − shift·I)·v ; partials[b] = Σ_{rows of block b} y²; returns #blocks.
int gemv_shift(const double* x, long long n, long long ldx, const double* v, double shift,
               double* y, double* partials, cudaStream_t st);
int gemv_blocks(long long n);
// the same product for a BITWISE-symmetric X from its lower triangle (n % 64 == 0, see symv_ok);
// ws ≥ symv_ws_elems(n) doubles; returns the partials count (≤ gemv_blocks(n))
bool symv_ok(const double* x, long long n, long long ldx, const double* v);
size_t symv_ws_elems(long long n);
int symv_shift(const double* x, long long n, long long ldx, const double* v, double shift, double* y,
               double* partials, double* ws, cudaStream_t st);
// nrm = sqrt(Σ partials); if nrm ≤ floor set *flag; v = y / nrm. out[0] = nrm.
void normalize(const double* y, const double* partials, int nparts, long long n, double floor,
               double* v, double* out, int* flag, cudaStream_t st);
void sum_partials(const double* partials, long long nparts, double* out, int do_sqrt,
                  cudaStream_t st);
// Split-K reduction with the GEMM epilogues; mode EPI_STORE/SHIFT/SUB or 10 (= symmetric).
void splitk_reduce(const double* ws, int splits, long long split_stride, int M, int N,
                   long long ldw, double* C, long long ldc, int mode, double alpha,
                   const double* S, long long lds, cudaStream_t st);
void copy_matrix(const double* src, long long lds, double* dst, long long ldd, long long rows,
                 int cols, cudaStream_t st);
void fill_zero(double* dst, long long ld, long long rows, long long cols, cudaStream_t st);
void scale_columns(const double* w, long long ldw, const double* d, double* out, long long ldo,
                   long long rows, int cols, cudaStream_t st);
void gather_columns(const double* src, long long lds, const int* idx, int ncols, double* dst,
                    long long ldd, long long rows, cudaStream_t st);
void add_diag(double* a, long long ld, int m, double s, cudaStream_t st);
// out[0] = max |x| over a rows×cols block (deterministic: non-negative u64 max)
void max_abs(const double* x, long long rows, long long cols, long long ldx, double* out,
             cudaStream_t st);
void set_identity(double* a, long long ld, int m, cudaStream_t st);

// ---- small dense (w×w) kernels ---------------------------------------------
// Blocked right-looking Cholesky A = L Lᵀ in place (lower), ld = lda.
// info[0] = 0 ok, j+1 = first failing pivot.  Upper triangle zeroed.
int cholesky_lower(double* a, long long lda, int m, int* info, double* ws, size_t ws_elems,
                   cudaStream_t st);
// rinv = (Lᵀ)⁻¹ (upper triangular), from lower-triangular L.
void tri_inv_upper_from_lower(const double* l, long long ldl, int m, double* rinv,
                              long long ldr, cudaStream_t st);
// One launch: L = chol(G + shift I) and (when no pivot failed) Rinv = L⁻ᵀ;
// status = {info, trace(G), min L_ii, max L_ii}.
int chol_inv(const double* G, long long ldg, int m, double shift, double* L, long long ldl,
             double* Rinv, long long ldr, double* Xs, double* status, cudaStream_t st);
// Faster two-launch variant (warp-register diagonal blocks + parallel block
// inverse); dinv scratch: ceil(m/32)·32·32 doubles.  Same outputs as chol_inv.
int chol_fast(const double* G, long long ldg, int m, double shift, double* L, long long ldl,
              double* Rinv, long long ldr, double* Dinv, double* status, cudaStream_t st,
              double shift_factor = 0.0, double* L1 = nullptr, double* Rinv1 = nullptr,
              double* Dinv1 = nullptr, double* status1 = nullptr);
// rdiag[i] *= L[i][i]
void accumulate_diag(const double* l, long long ldl, int m, double* rdiag, cudaStream_t st);
// Symmetric eigensolver (block Jacobi, jacobi.cu).
// a (m×m, destroyed), values[m], v (m×m).  Enqueued only: returns 0 (< 0: launch /
// workspace error); *dsweeps (DEVICE int) receives the sweep count, or −1 on
// non-convergence, for the caller's next status read.
int jacobi_eigh(double* a, long long lda, int m, double* values, double* v, long long ldv,
                double* ws, size_t ws_elems, int* dsweeps, cudaStream_t st);
size_t jacobi_ws_elems(int m);
// Sort eigenpairs descending, sign-fix columns (symmetric.py:80-85).
// vals_out[m], vecs_out (m×m, ld), npos[0] = #(vals − offset > 0).
void sort_eigs(const double* vals, const double* vecs, long long ldv, int m, double offset,
               double* vals_out, double* vecs_out, long long ldo, int* npos, int* perm,
               cudaStream_t st);

// ---- solver loop (sdls_kernels.cu) -------------------------------------------
void sdls_assemble(const double* cr, long long n, const long long* pos, const int* ptr,
                   const int* econ, const double* evals, const double* y, int npos, double* x,
                   cudaStream_t st);
void sdls_traces(const double* wd, const double* w, long long ldw, int r, const int* rows,
                 const int* cols, const double* vals, const int* cptr, int m, double* t,
                 cudaStream_t st);
void sdls_traces_dense(const double* x, long long ldx, const int* rows, const int* cols,
                       const double* vals, const int* cptr, int m, double* t, cudaStream_t st);
void sdls_step(const double* b, const double* t, double* y, double* grad, int m, double beta,
               double eps, double* out, cudaStream_t st);

}  // namespace psd
