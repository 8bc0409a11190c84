// C ABI (include/psdproj.h) and the host-side orchestration of the randomized
// PSD projection on one B200.  Every numeric step runs in the sm_100a kernels
// of this library; the host only sequences launches and takes the decisions
// the reference takes on the host (raise / truncate / count).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <functional>
#include <string>
#include <vector>

#include "launch.h"
#include "psdproj.h"

using ll = long long;

namespace psd {
thread_local int g_launch_count = 0;
}

struct psd_plan {
  int device = 0;
  ll n = 0;
  int w = 0;
  ll ldp = 0;  // leading dimension of n×w panels
  double* panel[6] = {};
  double *G = nullptr, *L = nullptr, *Rinv = nullptr, *T = nullptr, *V = nullptr, *U = nullptr;
  double *vals = nullptr, *vals_sorted = nullptr, *rdiag = nullptr, *dvec = nullptr;
  int* ints = nullptr;  // perm[w], npos, info, flags
  double* ws = nullptr;
  size_t ws_elems = 0;
  double* jws = nullptr;
  size_t jws_elems = 0;
  double *gy = nullptr, *gv = nullptr, *gpart = nullptr, *stats = nullptr, *scal = nullptr;
  double* qrstat = nullptr;
  double* symv_ws = nullptr;   // tile partials of the symmetric GEMV (power iteration on a bitwise-symmetric X)
  size_t symv_elems = 0;
  bool symv_failed = false;
  bool span_host = false;   // power-step QRs on the host-driven loop (set while redoing a call)
  double* dinv = nullptr;  // ceil(w/32) diagonal-block inverses (32×32) for chol_fast
  double *L1 = nullptr, *Rinv1 = nullptr, *dinv1 = nullptr;   // shifted CholeskyQR candidate
  bool oz_gram = false;   // CholeskyQR Grams on the INT8 engine (set per call by psd_ran_proj)
  // the Gram's own INT8-engine buffers (panel residues, column exponents, partials): ≈ 16·w·n
  // bytes, so the FP32 path (which has no X residue planes) can use it too
  int8_t* g_br = nullptr;
  int* g_f = nullptr;
  uint8_t* g_res = nullptr;
  size_t g_res_elems = 0;
  ll g_ldk = 0;
  bool g_failed = false;
  // g_br / g_f hold the residue planes of this n×w panel (set by the last INT8 Gram; cleared by
  // every write to a panel) — the compression product X·Q and the Gram QᵀC reuse them
  const double* gq_P = nullptr;
  ll gq_ld = 0, gq_n = 0;
  int gq_w = 0;
  int gparts = 0;
  double* rpart = nullptr;
  ll rparts = 0;
  // FP32 path (ensure_f32)
  float *xh = nullptr, *xl = nullptr, *f[4] = {}, *ws32 = nullptr;
  // FP64-on-INT8 (Ozaki II) path (ensure_oz): X residues, panel residues, exponents, partials
  int8_t *oz_ar = nullptr, *oz_br = nullptr;
  int *oz_e = nullptr, *oz_f = nullptr;
  unsigned* oz_rowmax = nullptr;  // high words of max_j |x_ij| from the symmetry pass (row scales)
  uint8_t* oz_res = nullptr;
  ll oz_ldk = 0;
  bool oz_failed = false;
  size_t oz_res_elems = 0;
  ll ldx32 = 0;
  size_t ws32_elems = 0;
  std::vector<void*> allocs;
  size_t bytes = 0;
  // pipelined batch (psd_plan_prefetch): the next X's symmetry pass and residue planes are
  // prepared on a low-priority side stream into the *_alt buffers while this call's QR /
  // eigensolver run; calls involved run on `work`, a high-priority stream joined to the
  // caller's, so their CTAs are dispatched ahead of the side stream's.
  cudaStream_t work = nullptr, side = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_fork = nullptr, ev_pf_stats = nullptr,
              ev_pf_done = nullptr;
  int8_t* oz_ar_alt = nullptr;
  int* oz_e_alt = nullptr;
  unsigned* oz_rowmax_alt = nullptr;
  double* stats_alt = nullptr;
  unsigned char *pf_host = nullptr, *pf_dev = nullptr;   // mapped statistics of the prefetched X
  const double* hint_x = nullptr;   // set by psd_plan_prefetch, consumed by the next call
  ll hint_n = 0, hint_ldx = 0;
  const double* pf_x = nullptr;     // prefetched (in flight or done on `side`)
  ll pf_n = 0, pf_ldx = 0;
  bool pf_ready = false;
  bool pf_failed = false;
  // FP32 path (psd_plan_prefetch_f32): the next X's symmetry pass fused with its tf32 lo split
  const float* hint_x32 = nullptr;
  const float* pf_x32 = nullptr;
  bool pf_f32 = false;              // the prefetch in flight is an FP32 one
  float* xl_alt = nullptr;
  bool pf32_failed = false;
  // stage profiling (psd_plan_profile): CUDA events on the caller's stream
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  double stage_ms[PSD_NUM_STAGES] = {};
  int stage_cnt[PSD_NUM_STAGES] = {};
};

namespace {

thread_local std::string g_err;

cudaEvent_t take_event(psd_plan* p) {
  cudaEvent_t e;
  if (!p->ev_pool.empty()) {
    e = p->ev_pool.back();
    p->ev_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}

// RAII stage marker: records start/stop events on `st` when profiling is on.
struct Stage {
  psd_plan* p;
  int id;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  Stage(psd_plan* p_, int id_, cudaStream_t st_) : p(p_), id(id_), st(st_) {
    if (p->prof) {
      a = take_event(p);
      cudaEventRecord(a, st);
    }
  }
  void close() {
    if (p->prof && a) {
      cudaEvent_t b = take_event(p);
      cudaEventRecord(b, st);
      p->marks.push_back({id, {a, b}});
      a = nullptr;
    }
  }
  ~Stage() { close(); }
};

// Fold recorded marks into the per-stage totals (stream must be synchronised).
void collect_marks(psd_plan* p) {
  for (auto& m : p->marks) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, m.second.first, m.second.second) == cudaSuccess) {
      p->stage_ms[m.first] += ms;
      p->stage_cnt[m.first] += 1;
    }
    p->ev_pool.push_back(m.second.first);
    p->ev_pool.push_back(m.second.second);
  }
  p->marks.clear();
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(PSD_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

#define PSD_CUDA_CHECK(expr, where)                \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

#define PSD_TRY(expr)          \
  do {                         \
    int _s = (expr);           \
    if (_s != PSD_OK) return _s; \
  } while (0)

// Calls on one device are serialized (each holds its device's lock until its final
// stream synchronisation): the persistent tcgen05 kernels (TMEM-resident for their
// lifetime) and the cooperative Jacobi grid must not share a GPU with another call's
// copies of themselves — three host threads projecting concurrently on separate
// streams deadlocked the device in a round-2 experiment.
std::recursive_mutex& device_mutex(int dev) {
  static std::recursive_mutex mu[16];
  return mu[dev & 15];
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

double* alloc(psd_plan* p, size_t elems) {
  void* ptr = nullptr;
  const size_t b = std::max<size_t>(elems, 2) * sizeof(double);
  if (cudaMalloc(&ptr, b) != cudaSuccess) return nullptr;
  p->allocs.push_back(ptr);
  p->bytes += b;
  return static_cast<double*>(ptr);
}

int sync(cudaStream_t st, const char* where) {
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, where);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, where);
  return PSD_OK;
}

int launched(int k) {
  if (k > 0) psd::count_launch(k);
  return k;
}

// C = op(X)·P  (op = X or Xᵀ); alpha > 0 fuses B = (X + αI)/α: C = (acc + α·P)/α
// X is rows×cols; op(X) = X (M=rows, K=cols) or Xᵀ (M=cols, K=rows).
int xmul_rect(psd_plan* p, const double* x, ll rows, ll cols, ll ldx, const double* P, ll ldP,
              int w, double* out, ll ldo, double alpha, bool transpose, cudaStream_t st) {
  Stage mark(p, PSD_STAGE_SKETCH_GEMM, st);
  if (out == p->gq_P) p->gq_P = nullptr;
  psd::GemmOp op;
  op.a_layout = transpose ? psd::A_KM : psd::A_MK;
  op.b_layout = psd::B_KN;
  op.A = x;
  op.lda = ldx;
  op.B = P;
  op.ldb = ldP;
  op.C = out;
  op.ldc = ldo;
  op.M = (int)(transpose ? cols : rows);
  op.N = w;
  op.K = (int)(transpose ? rows : cols);
  op.epi = alpha > 0.0 ? psd::EPI_SHIFT : psd::EPI_STORE;
  op.alpha = alpha;
  op.S = P;
  op.lds = ldP;
  op.max_splits = 16;   // wave quantisation at small n (config 2: 128 tiles on 148 SMs)
  const int r = psd::gemm_f64(op, p->ws, p->ws_elems, st);
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "unsupported GEMM layout");
  return PSD_OK;
}

int xmul(psd_plan* p, const double* x, ll n, ll ldx, const double* P, ll ldP, int w, double* out,
         ll ldo, double alpha, bool transpose, cudaStream_t st) {
  return xmul_rect(p, x, n, n, ldx, P, ldP, w, out, ldo, alpha, transpose, st);
}

// G (w×w, ld w) = Aᵀ·B for n×w panels A, B (symmetrised when A == B or sym)
// G = YᵀY (w×w) as an exact-integer Gram on the INT8 tensor cores (Ozaki II): Y's column
// scales and transposed residues (the panel preparation of the X·P products) serve as
// both operands — A = Yᵀ is B's residue planes read row-wise — K = n unsplit up to 2^15
// per split, CRT on the w×w output only.  Bitwise symmetric (the integer sums are).
int ensure_gram_oz(psd_plan* p) {
  if (p->g_ldk) return PSD_OK;
  if (p->g_failed || p->w > 512) return -1;
  const int L = psd::oz_num_moduli();
  const ll ldk = (p->n + 127) / 128 * 128;
  const ll wpad = (p->w + 15) / 16 * 16;
  auto balloc = [&](size_t bytes) -> void* { return static_cast<void*>(alloc(p, (bytes + 7) / 8)); };
  p->g_br = static_cast<int8_t*>(balloc((size_t)L * wpad * ldk));
  p->g_f = static_cast<int*>(balloc((size_t)wpad * sizeof(int)));
  p->g_res_elems = (size_t)L * 8 * wpad * (wpad + 16);
  p->g_res = static_cast<uint8_t*>(balloc(p->g_res_elems));
  if (!p->g_br || !p->g_f || !p->g_res) {
    cudaGetLastError();
    p->g_failed = true;
    return -1;
  }
  cudaMemset(p->g_br, 0, (size_t)L * wpad * ldk);   // K padding stays zero
  // cudaMemset is asynchronous on the legacy stream: finish it before any call on a
  // non-blocking stream (the caller's or the plan's pipelined `work` stream) writes here
  cudaDeviceSynchronize();
  p->g_ldk = ldk;
  return PSD_OK;
}

int gram_oz(psd_plan* p, const double* Y, ll ld, ll n, int w, double* G, cudaStream_t st) {
  if (ensure_gram_oz(p) != PSD_OK) return -1;
  psd::OzOp op;
  op.P = Y;
  op.ldp = ld;
  op.N = w;
  op.K = (int)n;
  op.br = p->g_br;
  op.ldbr = p->g_ldk;
  op.f = p->g_f;
  if (psd::oz_prepare_panel(op, st) != 0) return -1;
  p->gq_P = Y;
  p->gq_ld = ld;
  p->gq_n = n;
  p->gq_w = w;
  op.ar = op.br;
  op.ldar = op.ldbr;
  op.ar_rows = (w + 15) / 16 * 16;
  op.e = op.f;
  op.M = w;
  op.res = p->g_res;
  op.res_elems = p->g_res_elems;
  op.C = G;
  op.ldc = w;
  return psd::oz_gemm_prepared(op, st) < 0 ? -1 : 0;
}

// G = AᵀB for A ≠ B on the INT8 engine when A's planes are already in g_br (the compression
// Gram QᵀC after the verification Gram of Q): B's panel is prepared into oz_br (free once the
// product that read it has run), A = Qᵀ is g_br read row-wise.
int gram2_oz(psd_plan* p, const double* A, const double* B, ll ld, ll n, int w, double* G, cudaStream_t st) {
  if (!(p->gq_P == A && p->gq_ld == ld && p->gq_n == n && p->gq_w == w) || !p->oz_br || p->w > 512 ||
      p->g_ldk != p->oz_ldk)
    return -1;
  psd::OzOp op;
  op.P = B;
  op.ldp = ld;
  op.N = w;
  op.K = (int)n;
  op.br = p->oz_br;
  op.ldbr = p->oz_ldk;
  op.f = p->oz_f;
  if (psd::oz_prepare_panel(op, st) != 0) return -1;
  op.ar = p->g_br;
  op.ldar = p->g_ldk;
  op.ar_rows = (w + 15) / 16 * 16;
  op.e = p->g_f;
  op.M = w;
  op.res = p->g_res;
  op.res_elems = p->g_res_elems;
  op.C = G;
  op.ldc = w;
  return psd::oz_gemm_prepared(op, st) < 0 ? -1 : 0;
}

int panel_tn(psd_plan* p, const double* A, const double* B, ll ld, ll n, int w, double* G,
             bool sym, cudaStream_t st) {
  if (A == B && p->oz_gram && w <= 512 && n <= psd::oz_max_k() && gram_oz(p, A, ld, n, w, G, st) == 0)
    return PSD_OK;   // else (buffers unavailable): the DMMA Gram below
  if (A != B && p->oz_gram && n <= psd::oz_max_k() && gram2_oz(p, A, B, ld, n, w, G, st) == 0) {
    if (sym) psd::symmetrize_small(G, w, w, st);
    return PSD_OK;
  }
  psd::GemmOp op;
  op.a_layout = psd::A_KM;
  op.b_layout = psd::B_KN;
  op.A = A;
  op.lda = ld;
  op.B = B;
  op.ldb = ld;
  op.C = G;
  op.ldc = w;
  op.M = w;
  op.N = w;
  op.K = (int)n;
  op.epi = psd::EPI_STORE;
  op.max_splits = 256;
  const int r = psd::gemm_f64(op, p->ws, p->ws_elems, st);
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "unsupported GEMM layout");
  if (sym) {
    psd::symmetrize_small(G, w, w, st);
  }
  return PSD_OK;
}

// out (n×N) = A (n×K, lda) · B (K×N, ldb)
int panel_nn(psd_plan* p, const double* A, ll lda, const double* B, ll ldb, double* out, ll ldo,
             ll n, int K, int N, cudaStream_t st) {
  if (out == p->gq_P) p->gq_P = nullptr;
  psd::GemmOp op;
  op.a_layout = psd::A_MK;
  op.b_layout = psd::B_KN;
  op.A = A;
  op.lda = lda;
  op.B = B;
  op.ldb = ldb;
  op.C = out;
  op.ldc = ldo;
  op.M = (int)n;
  op.N = N;
  op.K = K;
  op.epi = psd::EPI_STORE;
  op.max_splits = 1;
  const int r = psd::gemm_f64(op, p->ws, p->ws_elems, st);
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "unsupported GEMM layout");
  return PSD_OK;
}

__global__ void fill_value_kernel(double* a, int m, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) a[i] = v;
}

__global__ void clip_values_kernel(const double* vals, int m, double offset, double scale,
                                   double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = (vals[i] - offset) * scale;
}

constexpr int kSpanRedo = -100;   // internal: redo the range finder with host-decided power-step QRs

struct QrInfo {
  int passes = 0;
  int shifted = 0;
  double frob = 0.0;  // ‖Y‖_F of the input panel
  bool zero = false;  // Y == 0
  std::vector<double> rdiag;   // |R_ii| when read together with the last status (no extra round trip)
  int span_redo = 0;           // a device-decided power-step QR missed its one-pass acceptance
};

// The final QR's first two passes without host round trips: the same candidate rule on the
// device, |R_ii| accumulated from the chosen factor, and the pass's status (plus the power-step
// redo flag) saved for the host to replay the decisions after one read (cholqr below).
__global__ void qr_select_final_kernel(const double* __restrict__ stat, double* __restrict__ rinv,
                                       const double* __restrict__ rinv1, const double* __restrict__ l,
                                       const double* __restrict__ l1, int w, double* __restrict__ rdiag,
                                       double* __restrict__ save, const int* __restrict__ redo) {
  __shared__ int shift_s;
  if (threadIdx.x == 0) {
    const double info = stat[0], mn = stat[2], mx = stat[3];
    const bool bad = info != 0.0 || !isfinite(mn) || !isfinite(mx);
    const double kest = mn > 0.0 ? mx / mn : INFINITY;
    shift_s = (bad || kest > 3e6) ? 1 : 0;
  }
  if (threadIdx.x < 16) save[threadIdx.x] = threadIdx.x == 15 ? (double)*redo : stat[threadIdx.x];
  __syncthreads();
  const bool shift = shift_s != 0;
  const double* ls = shift ? l1 : l;
  if (rdiag)
    for (int i = threadIdx.x; i < w; i += blockDim.x) rdiag[i] *= fabs(ls[(long long)i * w + i]);
  if (shift)
    for (long long e = threadIdx.x; e < (long long)w * w; e += blockDim.x) rinv[e] = rinv1[e];
}

// Power-step (span-only) CholeskyQR without a host round trip: the candidate choice of the
// host loop below (shift iff Cholesky breakdown or κ-estimate > 3e6) made on the device, and
// a flag raised when the pass would not have been accepted there (shifted, κ-estimate > 1e4,
// zero or non-finite Gram); the final QR reads the flag with its status, and a raised flag
// makes the caller redo the range finder with the host-driven loop.
__global__ void qr_select_kernel(const double* __restrict__ stat, double* __restrict__ rinv,
                                 const double* __restrict__ rinv1, long long elems, int* redo) {
  __shared__ int shift_s;
  if (threadIdx.x == 0) {
    const double info = stat[0], trace = stat[1], mn = stat[2], mx = stat[3];
    const bool bad = info != 0.0 || !isfinite(mn) || !isfinite(mx);
    const double kest = mn > 0.0 ? mx / mn : INFINITY;
    const bool shift = bad || kest > 3e6;
    shift_s = shift ? 1 : 0;
    if (shift || kest > 1e4 || !(trace > 0.0) || !isfinite(trace) || stat[8] != 0.0) atomicOr(redo, 1);
  }
  __syncthreads();
  if (shift_s)
    for (long long e = threadIdx.x; e < elems; e += blockDim.x) rinv[e] = rinv1[e];
}

// CholeskyQR2 with shifted passes (shifted CholeskyQR3 when ill-conditioned).
// Orthonormalises the n×w panel in `bufs[cur]`; `bufs[tmp]` is scratch.
// On return *qidx is the buffer index holding Q; rdiag (if non-null) holds
// Π_pass |L_ii| = |R_ii| of Y = Q·R.
//
// `span_only` (the power-iteration stabilisation of sketch.py:78/:80): the
// next product only needs a well-conditioned basis of span(Y) — the final
// result depends on the span alone — so one unshifted pass with κ²u ≲ 1e-12
// is accepted instead of two.
int cholqr(psd_plan* p, double** bufs, int cur, int tmp, ll n, int w, double* rdiag, int* qidx,
           QrInfo* info, cudaStream_t st, bool span_only = false, bool device_decided = false) {
  Stage mark(p, PSD_STAGE_QR, st);
  const ll ld = p->ldp;
  const double u0 = 1.1102230246251565e-16;
  if (span_only && device_decided) {   // one pass, candidate chosen on the device (see qr_select_kernel)
    PSD_TRY(panel_tn(p, bufs[cur], bufs[cur], ld, n, w, p->G, true, st));
    const double sfac = 11.0 * ((double)n * w + (double)w * (w + 1)) * u0;
    if (psd::chol_fast(p->G, w, w, 0.0, p->L, w, p->Rinv, w, p->dinv, p->qrstat, st, sfac, p->L1,
                       p->Rinv1, p->dinv1, p->qrstat + 8) != 0)
      return fail(PSD_ERR_INVALID_PARAMS, "width %d too large for the CholeskyQR kernel", w);
    qr_select_kernel<<<1, 1024, 0, st>>>(p->qrstat, p->Rinv, p->Rinv1, (long long)w * w, p->ints + p->w + 4);
    launched(1);
    PSD_TRY(panel_nn(p, bufs[cur], ld, p->Rinv, w, bufs[tmp], ld, n, w, w, st));
    info->passes = 1;
    *qidx = tmp;
    return PSD_OK;
  }
  if (rdiag) {
    fill_value_kernel<<<(w + 255) / 256, 256, 0, st>>>(rdiag, w, 1.0);
    launched(1);
  }
  int unshifted_run = 0;
  double kest0 = 0.0;
  bool verified = false;
  const double u = 1.1102230246251565e-16;
  // host decision of one pass from its status (the loop below, or replayed for deferred passes)
  // → 1: stop with Y == 0, < 0: error; sets shift
  auto decide = [&](const double* hs2, int pass, bool& shift) -> int {
    const double trace = hs2[1];
    if (pass == 0) {
      info->frob = std::sqrt(std::max(trace, 0.0));
      if (trace == 0.0) {
        info->zero = true;
        return 1;
      }
    }
    if (!std::isfinite(trace)) return fail(PSD_ERR_CONVERGENCE, "non-finite Gram matrix in QR");
    const bool bad = hs2[0] != 0.0 || !std::isfinite(hs2[2]) || !std::isfinite(hs2[3]);
    const double kest = (hs2[2] > 0.0) ? hs2[3] / hs2[2] : INFINITY;
    if (pass == 0) kest0 = kest;
    shift = bad || kest > 3e6;
    if (shift) {
      // Fukaya et al. shifted CholeskyQR: s = 11(mn + n(n+1))·u·‖Y‖² (candidate 1)
      if (hs2[8] != 0.0)
        return fail(PSD_ERR_CONVERGENCE, "shifted CholeskyQR broke down (pivot %d)", (int)hs2[8]);
      info->shifted = 1;
    }
    info->passes++;
    unshifted_run = shift ? 0 : unshifted_run + 1;
    if ((unshifted_run >= 2 && kest0 <= 1e4) || (span_only && !shift && kest <= 1e4)) verified = true;
    return PSD_OK;
  };
  int first = 0;
  static const bool defer_on = [] { const char* e = getenv("PSD_QR_DEFER"); return !(e && e[0] == '0'); }();
  if (!span_only && defer_on) {
    // the first two passes with device-side candidate choice, then ONE read of both statuses
    // (and |R_ii|): the host replays the loop's decisions; identical kernels and results
    constexpr int kDefer = 2;
    const int c0 = cur;
    const double sfac = 11.0 * ((double)n * w + (double)w * (w + 1)) * u;
    for (int pass = 0; pass < kDefer; ++pass) {
      PSD_TRY(panel_tn(p, bufs[cur], bufs[cur], ld, n, w, p->G, true, st));
      if (psd::chol_fast(p->G, w, w, 0.0, p->L, w, p->Rinv, w, p->dinv, p->qrstat, st, sfac, p->L1,
                         p->Rinv1, p->dinv1, p->qrstat + 8) != 0)
        return fail(PSD_ERR_INVALID_PARAMS, "width %d too large for the CholeskyQR kernel", w);
      qr_select_final_kernel<<<1, 1024, 0, st>>>(p->qrstat, p->Rinv, p->Rinv1, p->L, p->L1, w, rdiag,
                                                 p->qrstat + 16 + 16 * pass, p->ints + p->w + 4);
      launched(1);
      PSD_TRY(panel_nn(p, bufs[cur], ld, p->Rinv, w, bufs[tmp], ld, n, w, w, st));
      std::swap(cur, tmp);
    }
    double saved[2 * 16];
    if (rdiag) info->rdiag.assign(w, 0.0);
    PSD_CUDA_CHECK(psd::read_small2(saved, p->qrstat + 16, sizeof(saved), rdiag ? info->rdiag.data() : nullptr,
                                    rdiag, rdiag ? w * sizeof(double) : 0, st),
                   "qr status");
    PSD_TRY(sync(st, "cholesky"));
    info->span_redo = (int)saved[16 + 15];
    for (int pass = 0; pass < kDefer; ++pass) {
      bool shift = false;
      const int r = decide(saved + 16 * pass, pass, shift);
      if (r == 1) {   // Y == 0 (the passes after it computed nothing the caller uses)
        *qidx = c0;
        return PSD_OK;
      }
      if (r != PSD_OK) return r;
      if (verified) break;   // only after the second pass (unshifted_run ≥ 2 or span rule)
    }
    if (verified) {
      *qidx = cur;
      return PSD_OK;
    }
    info->rdiag.clear();   // not final yet
    first = kDefer;
  }
  for (int pass = first; pass < 10; ++pass) {
    PSD_TRY(panel_tn(p, bufs[cur], bufs[cur], ld, n, w, p->G, true, st));
    if (unshifted_run >= 2) {
      // verification Gram after two unshifted passes: accept if ‖QᵀQ − I‖_max small
      // (checked before factoring it, so an accepted basis costs no third Cholesky)
      psd::identity_defect(p->G, w, w, p->scal + 3, st);
      double dev = 0.0;
      // the final QR's |R_ii| (accumulated through the last pass) ride along with the defect
      if (rdiag) info->rdiag.assign(w, 0.0);
      PSD_CUDA_CHECK(psd::read_small2(&dev, p->scal + 3, sizeof(double), rdiag ? info->rdiag.data() : nullptr,
                                      rdiag, rdiag ? w * sizeof(double) : 0, st),
                     "orthogonality defect");
      PSD_TRY(sync(st, "orthogonality defect"));
      if (dev <= 1e-13 * std::max(1, w)) {
        verified = true;
        break;
      }
      info->rdiag.clear();
    }
    // both candidates at once: unshifted (L, Rinv) and Fukaya-shifted (L1, Rinv1) with
    // s = 11(nw + w(w+1))·u·trace(G) — the fallback costs no extra launch or round trip
    const double sfac = 11.0 * ((double)n * w + (double)w * (w + 1)) * u;
    if (psd::chol_fast(p->G, w, w, 0.0, p->L, w, p->Rinv, w, p->dinv, p->qrstat, st, sfac, p->L1,
                       p->Rinv1, p->dinv1, p->qrstat + 8) != 0)
      return fail(PSD_ERR_INVALID_PARAMS, "width %d too large for the CholeskyQR kernel", w);
    double hs2[16];
    PSD_CUDA_CHECK(psd::read_small2(hs2, p->qrstat, sizeof(hs2), &info->span_redo, p->ints + p->w + 4,
                                    sizeof(int), st),
                   "qr status");
    PSD_TRY(sync(st, "cholesky"));
    bool shift = false;
    const int r = decide(hs2, pass, shift);
    if (r == 1) {
      *qidx = cur;
      return PSD_OK;
    }
    if (r != PSD_OK) return r;
    const double* Lsel = shift ? p->L1 : p->L;
    const double* Rsel = shift ? p->Rinv1 : p->Rinv;
    if (rdiag) psd::accumulate_diag(Lsel, w, w, rdiag, st);
    PSD_TRY(panel_nn(p, bufs[cur], ld, Rsel, w, bufs[tmp], ld, n, w, w, st));
    std::swap(cur, tmp);
    if (verified) break;
  }
  if (!verified) return fail(PSD_ERR_CONVERGENCE, "CholeskyQR did not reach orthogonality");
  *qidx = cur;
  return PSD_OK;
}

struct SymInfo {
  double max_abs = 0.0, defect = 0.0;
  bool bitwise = true, nonfinite = false;
};

int symcheck(psd_plan* p, const double* x, ll n, ll ldx, SymInfo* si, cudaStream_t st,
             unsigned* rowmax = nullptr) {
  {
    Stage mark(p, PSD_STAGE_SYMCHECK, st);
    psd::sym_stats(x, n, ldx, p->stats, st, rowmax);
  }
  double h[3];
  PSD_CUDA_CHECK(psd::read_small(h, p->stats, 3 * sizeof(double), st),
                 "stats");
  PSD_TRY(sync(st, "symmetry check"));
  int flags = 0;
  std::memcpy(&flags, &h[2], sizeof(int));
  si->max_abs = h[0];
  si->defect = h[1];
  si->bitwise = (flags & 1) == 0;
  si->nonfinite = (flags & 2) != 0;
  return PSD_OK;
}

// Range finder core (sketch.py:53-93).  Returns index of the buffer holding
// the basis (columns compacted to *width_out).  bufs: 3 panel buffers.
// X is m×n (m == n for the projections); Ω is n×w; the basis is m×w.
// op(X)·P for an n×w panel P: transpose=true asks for Xᵀ·P (sketch.py:79).
using MulFn = std::function<int(const double* P, ll ldP, int w, double* out, ll ldo, bool transpose)>;

int range_finder_core(psd_plan* p, const MulFn& mul, ll m, ll n, const double* omega, ll ldo, int w,
                      int q, bool always_stabilize, bool strict, double** bufs, int* qidx,
                      int* width_out, QrInfo* qi, cudaStream_t st,
                      const std::function<int()>& after_first = nullptr,
                      const std::function<void()>& before_final_qr = nullptr) {
  const ll ld = p->ldp;
  p->gq_P = nullptr;   // planes of an earlier call's panels are never reused
  const bool stabilize = q >= 2 || always_stabilize;               // sketch.py:74
  // power-step QRs decided on the device (no host round trip) unless a redo asked otherwise
  static const bool dev_span_on = [] { const char* e = getenv("PSD_SPAN_DEVICE"); return !(e && e[0] == '0'); }();
  const bool dev_span = stabilize && !p->span_host && dev_span_on;
  if (dev_span) PSD_CUDA_CHECK(cudaMemsetAsync(p->ints + p->w + 4, 0, sizeof(int), st), "span flag");
  int y = 0;
  PSD_TRY(mul(omega, ldo, w, bufs[0], ld, false));                 // :75
  // deferred input validation (psd_ran_proj): the host collects the symmetry statistics
  // while the first product runs, before anything depends on them
  if (after_first) PSD_TRY(after_first());
  for (int it = 0; it < q; ++it) {                                 // :76-82
    QrInfo tmp;
    if (stabilize) PSD_TRY(cholqr(p, bufs, y, (y + 1) % 3, m, w, nullptr, &y, &tmp, st, true, dev_span));
    const int z = (y + 1) % 3;
    // z = xᵀ @ y (sketch.py:79); for bitwise-symmetric X this equals X·Y exactly
    PSD_TRY(mul(bufs[y], ld, w, bufs[z], ld, true));
    int zq = z;
    if (stabilize) PSD_TRY(cholqr(p, bufs, z, (z + 1) % 3, n, w, nullptr, &zq, &tmp, st, true, dev_span));
    const int ny = (zq + 1) % 3;
    PSD_TRY(mul(bufs[zq], ld, w, bufs[ny], ld, false));
    y = ny;
  }
  n = m;  // the final QR and gather act on the m×w sample
  // the n×n products of the range finder are all enqueued: a pipelined batch starts the
  // next matrix's preparation here (psd_plan_prefetch)
  if (before_final_qr) before_final_qr();
  int qb = y;
  const int rcq = cholqr(p, bufs, y, (y + 1) % 3, n, w, p->rdiag, &qb, qi, st);   // :84-85
  if (dev_span) {   // a power step needed the host loop (also when the final QR failed after it): redo
    int fl = qi->span_redo;
    if (rcq != PSD_OK && psd::read_small(&fl, p->ints + p->w + 4, sizeof(int), st) != cudaSuccess) fl = 0;
    if (fl) return kSpanRedo;
  }
  PSD_TRY(rcq);
  if (qi->zero) {
    *width_out = 0;
    *qidx = qb;
    return PSD_OK;
  }
  std::vector<double> rd(w);
  if ((int)qi->rdiag.size() == w) {
    rd = qi->rdiag;   // read with the verification Gram's defect
  } else {
    PSD_CUDA_CHECK(psd::read_small(rd.data(), p->rdiag, w * sizeof(double), st), "rdiag");
    PSD_TRY(sync(st, "rdiag"));
  }
  std::vector<int> keep;
  for (int i = 0; i < w; ++i)
    if (rd[i] > 1e-12 * qi->frob) keep.push_back(i);               // :86
  if ((int)keep.size() < w) {
    if (strict)
      return fail(PSD_ERR_RANK_DEFICIENT, "sampled matrix has numerical rank %d < %d",
                  (int)keep.size(), w);
    if (!keep.empty()) {
      int* didx = p->ints;  // perm area reused
      PSD_CUDA_CHECK(cudaMemcpyAsync(didx, keep.data(), keep.size() * sizeof(int),
                                     cudaMemcpyHostToDevice, st),
                     "keep idx");
      const int dst = (qb + 1) % 3;
      if (bufs[dst] == p->gq_P) p->gq_P = nullptr;
      psd::gather_columns(bufs[qb], ld, didx, (int)keep.size(), bufs[dst], ld, n, st);
      qb = dst;
    }
  }
  *width_out = (int)keep.size();
  *qidx = qb;
  return PSD_OK;
}

int ensure_oz(psd_plan* p);
int ensure_pipeline(psd_plan* p);
int ensure_pipeline32(psd_plan* p);
int ensure_f32(psd_plan* p, bool need_hi);

}  // namespace

extern "C" {

const char* psd_last_error(void) { return g_err.c_str(); }

const char* psd_version(void) {
  return "psdproj 0.2.0 (sm_100a: FP64 as exact INT8 tcgen05 emulation (Ozaki II products, Ozaki I SYRK) "
         "or FP64 DMMA; FP32 as 3xTF32 tcgen05)";
}

int psd_plan_create(psd_plan** out, int64_t n, int32_t width, int32_t device) {
  if (!out) return fail(PSD_ERR_INVALID_PARAMS, "null plan pointer");
  if (n < 1 || width < 1 || width > n)
    return fail(PSD_ERR_INVALID_PARAMS, "plan needs 1 <= width <= n (n=%lld, width=%d)", (ll)n, width);
  DeviceGuard g(device);
  psd_plan* p = new psd_plan();
  p->device = device;
  p->n = n;
  p->w = width;
  p->ldp = (width + 1) / 2 * 2;
  const size_t panel = (size_t)n * p->ldp;
  const size_t sq = (size_t)width * width;
  bool ok = true;
  for (int i = 0; i < 6; ++i) ok &= (p->panel[i] = alloc(p, panel)) != nullptr;
  ok &= (p->G = alloc(p, sq)) != nullptr;
  ok &= (p->L = alloc(p, sq)) != nullptr;
  ok &= (p->Rinv = alloc(p, sq)) != nullptr;
  ok &= (p->L1 = alloc(p, sq)) != nullptr;
  ok &= (p->Rinv1 = alloc(p, sq)) != nullptr;
  ok &= (p->dinv1 = alloc(p, (size_t)((width + 31) / 32) * 1024)) != nullptr;
  ok &= (p->T = alloc(p, sq)) != nullptr;
  ok &= (p->V = alloc(p, sq)) != nullptr;
  ok &= (p->U = alloc(p, sq)) != nullptr;
  ok &= (p->vals = alloc(p, width)) != nullptr;
  ok &= (p->vals_sorted = alloc(p, width)) != nullptr;
  ok &= (p->rdiag = alloc(p, width)) != nullptr;
  ok &= (p->dvec = alloc(p, width)) != nullptr;
  ok &= (p->ints = reinterpret_cast<int*>(alloc(p, width + 8))) != nullptr;
  p->ws_elems = std::max<size_t>((size_t)4 * n * p->ldp, (size_t)256 * width * p->ldp);
  p->ws_elems = std::max<size_t>(p->ws_elems, std::min<size_t>((size_t)16 * n * p->ldp, (size_t)64 << 20));
  p->ws_elems = std::max<size_t>(p->ws_elems, 1 << 20);
  ok &= (p->ws = alloc(p, p->ws_elems)) != nullptr;
  p->jws_elems = psd::jacobi_ws_elems(width);
  ok &= (p->jws = alloc(p, p->jws_elems)) != nullptr;
  p->gparts = psd::gemv_blocks(n);
  ok &= (p->gy = alloc(p, n)) != nullptr;
  ok &= (p->gv = alloc(p, n)) != nullptr;
  ok &= (p->gpart = alloc(p, p->gparts)) != nullptr;
  ok &= (p->stats = alloc(p, 4)) != nullptr;
  ok &= (p->scal = alloc(p, 8)) != nullptr;
  ok &= (p->qrstat = alloc(p, 48)) != nullptr;   // [0, 8): unshifted candidate, [8, 16): shifted; [16, 48): deferred passes
  ok &= (p->dinv = alloc(p, (size_t)((width + 31) / 32) * 1024)) != nullptr;
  psd::GemmOp rop;
  rop.M = (int)n;
  rop.N = (int)n;
  p->rparts = psd::gemm_resid_ctas(rop);
  ok &= (p->rpart = alloc(p, p->rparts)) != nullptr;
  if (!ok) {
    psd_plan_destroy(p);
    return fail(PSD_ERR_NO_MEMORY, "device allocation failed for plan n=%lld width=%d", (ll)n, width);
  }
  *out = p;
  return PSD_OK;
}

void psd_plan_destroy(psd_plan* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  if (p->side) cudaStreamSynchronize(p->side);   // a prefetch may still be writing the alt planes
  if (p->work) cudaStreamSynchronize(p->work);
  for (cudaEvent_t e : {p->ev_in, p->ev_out, p->ev_fork, p->ev_pf_stats, p->ev_pf_done})
    if (e) cudaEventDestroy(e);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->work) cudaStreamDestroy(p->work);
  if (p->pf_host) cudaFreeHost(p->pf_host);
  for (auto& m : p->marks) {
    p->ev_pool.push_back(m.second.first);
    p->ev_pool.push_back(m.second.second);
  }
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  for (void* a : p->allocs) cudaFree(a);
  delete p;
}

int64_t psd_plan_bytes(const psd_plan* p) { return p ? (int64_t)p->bytes : 0; }

int psd_plan_prefetch(psd_plan* p, const double* x_next, int64_t n, int64_t ldx) {
  if (!p) return fail(PSD_ERR_INVALID_PARAMS, "null plan");
  if (x_next && (n < 1 || n > p->n || ldx < n))
    return fail(PSD_ERR_INVALID_PARAMS, "prefetch hint outside the plan (n=%lld, ldx=%lld)", (ll)n, (ll)ldx);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  p->hint_x = x_next;
  p->hint_x32 = nullptr;
  p->hint_n = x_next ? n : 0;
  p->hint_ldx = x_next ? ldx : 0;
  if (x_next && n < 3072) p->hint_x = nullptr;   // INT8 engine only (its size rule)
  if (p->hint_x && !p->work) {   // the call's streams exist before it decides to run on them
    DeviceGuard g(p->device);
    if (ensure_oz(p) != PSD_OK || ensure_pipeline(p) != PSD_OK) {
      cudaGetLastError();
      p->hint_x = nullptr;   // no room for a second set of planes: unpipelined calls
    }
  }
  return PSD_OK;
}

int psd_plan_prefetch_f32(psd_plan* p, const float* x_next, int64_t n, int64_t ldx) {
  if (!p) return fail(PSD_ERR_INVALID_PARAMS, "null plan");
  if (x_next && (n < 1 || n > p->n || ldx < n))
    return fail(PSD_ERR_INVALID_PARAMS, "prefetch hint outside the plan (n=%lld, ldx=%lld)", (ll)n, (ll)ldx);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  p->hint_x = nullptr;
  p->hint_x32 = x_next;
  p->hint_n = x_next ? n : 0;
  p->hint_ldx = x_next ? ldx : 0;
  if (p->hint_x32 && !p->xl_alt) {   // the call's streams and planes exist before it runs on them
    DeviceGuard g(p->device);
    if (ensure_f32(p, false) != PSD_OK || ensure_pipeline32(p) != PSD_OK) {
      cudaGetLastError();
      p->hint_x32 = nullptr;
    }
  }
  return PSD_OK;
}

int psd_require_symmetric(psd_plan* p, const double* x, int64_t n, int64_t ldx, double tol,
                          double* stats_out, void* stream) {
  if (!p || !x) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (n < 1) return fail(PSD_ERR_NONSQUARE, "matrix dimension must be at least 1");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SymInfo si;
  PSD_TRY(symcheck(p, x, n, ldx, &si, st));
  if (stats_out) {
    stats_out[0] = si.max_abs;
    stats_out[1] = si.defect;
    stats_out[2] = si.bitwise ? 1.0 : 0.0;
  }
  if (si.nonfinite) return fail(PSD_ERR_CONVERGENCE, "matrix has non-finite entries");
  if (tol < 0.0) tol = 1e-10 * std::max(1.0, si.max_abs);
  if (si.defect > tol)
    return fail(PSD_ERR_ASYMMETRIC,
                "matrix is not symmetric: max asymmetry %.3e exceeds tolerance %.3e", si.defect, tol);
  return PSD_OK;
}

// sym: X is bitwise symmetric (caller-checked) — the products read only its lower triangle
// (psd::symv_shift, half the HBM bytes) when the shape allows, else the row GEMV
static int power_iteration_impl(psd_plan* p, const double* x, ll n, ll ldx, double shift,
                                const double* v0, int n_iter, double* result, cudaStream_t st,
                                bool sym = false) {
  const double floor = 2.2250738585072014e-308 * (double)n;  // finfo.tiny·n (sketch.py:107)
  int* flag = p->ints + p->w + 2;
  PSD_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int), st), "flag");
  if (sym && psd::symv_ok(x, n, ldx, v0) && !p->symv_failed && p->symv_elems < psd::symv_ws_elems(n)) {
    p->symv_ws = alloc(p, psd::symv_ws_elems(p->n));   // once per plan (the old block is kept, small)
    if (p->symv_ws) {
      p->symv_elems = psd::symv_ws_elems(p->n);
    } else {
      cudaGetLastError();
      p->symv_failed = true;
    }
  }
  const bool use_symv = sym && psd::symv_ok(x, n, ldx, v0) && p->symv_elems >= psd::symv_ws_elems(n);
  auto product = [&](const double* v) {
    return use_symv ? psd::symv_shift(x, n, ldx, v, shift, p->gy, p->gpart, p->symv_ws, st)
                    : psd::gemv_shift(x, n, ldx, v, shift, p->gy, p->gpart, st);
  };
  const double* v = v0;
  for (int it = 0; it < n_iter; ++it) {
    const int nb = product(v);
    psd::normalize(p->gy, p->gpart, nb, n, floor, p->gv, p->scal, flag, st);
    v = p->gv;
  }
  const int nb = product(v);
  psd::sum_partials(p->gpart, nb, p->scal + 1, 1, st);
  double h[2];
  int hflag = 0;
  PSD_CUDA_CHECK(psd::read_small(h, p->scal, 2 * sizeof(double), st), "pi");
  PSD_CUDA_CHECK(psd::read_small(&hflag, flag, sizeof(int), st), "pi flag");
  PSD_TRY(sync(st, "power iteration"));
  *result = hflag ? 0.0 : h[1];
  return PSD_OK;
}

int psd_power_iteration(psd_plan* p, const double* x, int64_t n, int64_t ldx, double shift,
                        const double* v0, int32_t n_iter, double* result, void* stream) {
  if (!p || !x || !v0 || !result) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (n_iter < 1) return fail(PSD_ERR_INVALID_PARAMS, "power iteration needs n_iter >= 1, got %d", n_iter);
  if (n < 1 || n > p->n) return fail(PSD_ERR_INVALID_PARAMS, "n=%lld outside plan", (ll)n);
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  return power_iteration_impl(p, x, n, ldx, shift, v0, n_iter, result,
                              static_cast<cudaStream_t>(stream));
}

int psd_min_eig_magnitude(psd_plan* p, const double* x, int64_t n, int64_t ldx, const double* v1,
                          const double* v2, int32_t n_iter, double* result, void* stream) {
  return psd_min_eig_magnitude_ex(p, x, n, ldx, v1, v2, n_iter, 0u, result, stream);
}

int psd_min_eig_magnitude_ex(psd_plan* p, const double* x, int64_t n, int64_t ldx, const double* v1,
                             const double* v2, int32_t n_iter, uint32_t flags, double* result, void* stream) {
  if (!p || !x || !v1 || !v2 || !result) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (n_iter < 1) return fail(PSD_ERR_INVALID_PARAMS, "power iteration needs n_iter >= 1, got %d", n_iter);
  if (n < 1 || n > p->n) return fail(PSD_ERR_INVALID_PARAMS, "n=%lld outside plan", (ll)n);
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool sym = (flags & PSD_FLAG_ASSUME_SYMMETRIC) != 0;
  double s1 = 0.0, s2 = 0.0;
  PSD_TRY(power_iteration_impl(p, x, n, ldx, 0.0, v1, n_iter, &s1, st, sym));   // sketch.py:126
  PSD_TRY(power_iteration_impl(p, x, n, ldx, s1, v2, n_iter, &s2, st, sym));    // sketch.py:127-128
  *result = std::fabs(s1 - s2);
  return PSD_OK;
}

int psd_range_finder(psd_plan* p, const double* x, int64_t m, int64_t n, int64_t ldx,
                     const double* omega, int64_t ldo, int32_t width, int32_t q, double alpha,
                     uint32_t flags, double* basis, int64_t ldb, int32_t* width_out,
                     void* stream) {
  if (!p || !x || !omega || !basis || !width_out) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (q < 0) return fail(PSD_ERR_INVALID_PARAMS, "power exponent q must be >= 0, got %d", q);
  if (m < 1 || n < 1) return fail(PSD_ERR_INVALID_PARAMS, "expected a matrix, got shape (%lld, %lld)", (ll)m, (ll)n);
  if (width < 1 || width > std::min(m, n))
    return fail(PSD_ERR_INVALID_PARAMS, "k+l = %d exceeds min(m, n) = %lld", width, (ll)std::min(m, n));
  if (std::max(m, n) > p->n || width > p->w)
    return fail(PSD_ERR_INVALID_PARAMS, "problem exceeds plan capacity");
  if (alpha > 0.0 && m != n) return fail(PSD_ERR_INVALID_PARAMS, "scaled sketch needs a square matrix");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  psd::g_launch_count = 0;
  p->oz_gram = false;
  bool use_t = (m != n) || !(flags & PSD_FLAG_ASSUME_SYMMETRIC);
  if (use_t && m == n) {
    SymInfo si;
    PSD_TRY(symcheck(p, x, n, ldx, &si, st));
    use_t = !si.bitwise;
  }
  double* bufs[3] = {p->panel[0], p->panel[1], p->panel[2]};
  int qb = 0, wk = 0;
  QrInfo qi;
  const MulFn mul = [&](const double* P, ll ldP, int w, double* out, ll ldo2, bool t) {
    return xmul_rect(p, x, m, n, ldx, P, ldP, w, out, ldo2, alpha, t && use_t, st);
  };
  int rc = range_finder_core(p, mul, m, n, omega, ldo, width, q, false, (flags & PSD_FLAG_STRICT) != 0, bufs,
                             &qb, &wk, &qi, st);
  if (rc == kSpanRedo) {   // a device-decided power-step QR needed more passes: host-driven redo
    qi = QrInfo();
    p->span_host = true;
    rc = range_finder_core(p, mul, m, n, omega, ldo, width, q, false, (flags & PSD_FLAG_STRICT) != 0, bufs,
                           &qb, &wk, &qi, st);
    p->span_host = false;
  }
  PSD_TRY(rc);
  if (wk > 0) {
    psd::copy_matrix(bufs[qb], p->ldp, basis, ldb, m, wk, st);
  }
  *width_out = wk;
  return sync(st, "range finder");
}

int psd_eigh(psd_plan* p, double* a, int32_t m, int64_t lda, double* values, double* vectors,
             int64_t ldv, int32_t* sweeps_out, void* stream) {
  if (!p || !a || !values || !vectors) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (m < 1 || m > p->w) return fail(PSD_ERR_INVALID_PARAMS, "eigh size %d outside plan", m);
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  psd::symmetrize_small(a, m, lda, st);  // eigh validates/uses the symmetric part
  if (psd::jacobi_eigh(a, lda, m, p->vals, p->V, m, p->jws, p->jws_elems, p->ints + p->w + 1, st) < 0)
    return fail(PSD_ERR_CONVERGENCE, "Jacobi eigensolver could not be launched");
  psd::sort_eigs(p->vals, p->V, m, m, 0.0, values, vectors, ldv, p->ints + p->w, p->ints, st);
  int h[2] = {0, 0};   // {npos, sweeps}: one status read
  PSD_CUDA_CHECK(psd::read_small(h, p->ints + p->w, sizeof(h), st), "eigh status");
  PSD_TRY(sync(st, "eigh"));
  if (h[1] < 0) return fail(PSD_ERR_CONVERGENCE, "Jacobi eigensolver did not converge");
  if (sweeps_out) *sweeps_out = h[1];
  return PSD_OK;
}

}  // extern "C"

namespace {

// FP32 path buffers (allocated on first use): tf32 hi/lo of X, four operand
// scratch buffers (transposed panels / reconstruction factors), split-K partials.
int ensure_f32(psd_plan* p, bool need_hi) {
  if (need_hi && !p->xh) {
    const size_t xsz = (size_t)p->n * ((p->n + 31) / 32 * 32);
    p->xh = reinterpret_cast<float*>(alloc(p, (xsz + 1) / 2));
    if (!p->xh) return fail(PSD_ERR_NO_MEMORY, "device allocation failed for the FP32 hi buffer");
  }
  if (p->xl) return PSD_OK;
  const ll ld = (p->n + 31) / 32 * 32;
  const ll wp = (p->w + 15) / 16 * 16;
  const size_t xsz = (size_t)p->n * ld;
  const size_t fsz = (size_t)std::max(wp * ld, p->n * wp);
  const size_t wsz = (size_t)psd::tc32_ws_elems(p->n, p->w, 32);
  auto falloc = [&](size_t elems) { return reinterpret_cast<float*>(alloc(p, (elems + 1) / 2)); };
  bool ok = (p->xl = falloc(xsz)) != nullptr;
  for (int i = 0; i < 4; ++i) ok &= (p->f[i] = falloc(fsz)) != nullptr;
  ok &= (p->ws32 = falloc(wsz)) != nullptr;
  if (!ok) return fail(PSD_ERR_NO_MEMORY, "device allocation failed for the FP32 buffers (n=%lld)", p->n);
  p->ldx32 = ld;
  p->ws32_elems = wsz;
  return PSD_OK;
}

// Ozaki-II buffers (allocated on first use): 16 int8 residue planes of X
// (n × ldk each), panel residues, exponents, per-split residue partials.
int ensure_oz(psd_plan* p) {
  if (p->oz_ldk) return PSD_OK;
  if (p->oz_failed) return PSD_ERR_NO_MEMORY;
  const int L = psd::oz_num_moduli();
  const ll ldk = (p->n + 127) / 128 * 128;
  const int groups = (int)((p->w + 511) / 512);
  const ll gw_pad = ((p->w + groups - 1) / groups + 15) / 16 * 16;
  const ll wpad = gw_pad * groups;   // column groups of ≤ 512 (TMEM), each padded to 16
  auto balloc = [&](size_t bytes) -> void* {
    return static_cast<void*>(alloc(p, (bytes + 7) / 8));
  };
  p->oz_ar = static_cast<int8_t*>(balloc((size_t)L * p->n * ldk));
  p->oz_br = static_cast<int8_t*>(balloc((size_t)L * wpad * ldk));
  p->oz_e = static_cast<int*>(balloc((size_t)p->n * sizeof(int)));
  p->oz_rowmax = static_cast<unsigned*>(balloc((size_t)p->n * sizeof(unsigned)));
  p->oz_f = static_cast<int*>(balloc((size_t)wpad * sizeof(int)));
  p->oz_res_elems = (size_t)L * 8 * p->n * (gw_pad + 16);
  p->oz_res = static_cast<uint8_t*>(balloc(p->oz_res_elems));
  if (!p->oz_ar || !p->oz_br || !p->oz_e || !p->oz_f || !p->oz_res || !p->oz_rowmax) {
    p->oz_failed = true;
    return fail(PSD_ERR_NO_MEMORY, "device allocation failed for the INT8-emulation buffers");
  }
  p->oz_ldk = ldk;
  cudaMemset(p->oz_ar, 0, (size_t)L * p->n * ldk);   // K padding stays zero
  cudaMemset(p->oz_br, 0, (size_t)L * wpad * ldk);
  cudaDeviceSynchronize();   // legacy-stream memsets done before non-blocking streams write here
  return PSD_OK;
}

// Pipelining state (psd_plan_prefetch): streams, events, the mapped statistics slot and a
// second set of X residue planes / exponents / row maxima (allocated on first use).
// streams, events and the mapped statistics slot (shared by the FP64 and FP32 prefetch)
bool ensure_pipe_common(psd_plan* p) {
  if (p->work) return true;
  int least = 0, greatest = 0;
  bool ok = cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess;
  ok = ok && cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, least) == cudaSuccess;
  for (cudaEvent_t* e : {&p->ev_in, &p->ev_out, &p->ev_fork, &p->ev_pf_stats, &p->ev_pf_done})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaHostAlloc(reinterpret_cast<void**>(&p->pf_host), 64, cudaHostAllocMapped) == cudaSuccess;
  ok = ok && cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->pf_dev), p->pf_host, 0) == cudaSuccess;
  if (!p->stats_alt) ok = ok && (p->stats_alt = alloc(p, 4)) != nullptr;
  // `work` last: its existence marks the common state complete
  ok = ok && cudaStreamCreateWithPriority(&p->work, cudaStreamNonBlocking, greatest) == cudaSuccess;
  if (!ok) cudaGetLastError();
  return ok;
}

int ensure_pipeline(psd_plan* p) {
  if (p->oz_ar_alt) return PSD_OK;
  if (p->pf_failed || !p->oz_ldk) return -1;
  bool ok = ensure_pipe_common(p);
  if (ok) {
    const size_t planes = (size_t)psd::oz_num_moduli() * p->n * p->oz_ldk;
    p->oz_ar_alt = static_cast<int8_t*>(static_cast<void*>(alloc(p, (planes + 7) / 8)));
    p->oz_e_alt = reinterpret_cast<int*>(alloc(p, ((size_t)p->n + 1) / 2));
    p->oz_rowmax_alt = reinterpret_cast<unsigned*>(alloc(p, ((size_t)p->n + 1) / 2));
    ok = p->oz_ar_alt && p->oz_e_alt && p->oz_rowmax_alt;
    if (ok) ok = cudaMemset(p->oz_ar_alt, 0, planes) == cudaSuccess;   // K padding stays zero
    if (ok) ok = cudaDeviceSynchronize() == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    p->pf_failed = true;   // no room: calls run unpipelined
    p->oz_ar_alt = nullptr;
    return -1;
  }
  return PSD_OK;
}

int ensure_pipeline32(psd_plan* p) {
  if (p->xl_alt) return PSD_OK;
  if (p->pf32_failed || !p->xl) return -1;
  bool ok = ensure_pipe_common(p);
  if (ok) ok = (p->xl_alt = reinterpret_cast<float*>(alloc(p, ((size_t)p->n * p->ldx32 + 1) / 2))) != nullptr;
  if (!ok) {
    cudaGetLastError();
    p->pf32_failed = true;
    p->xl_alt = nullptr;
    return -1;
  }
  return PSD_OK;
}

// FP32: the next X's require_symmetric statistics fused with its tf32 lo split (X itself is
// the hi operand) into the alternate lo plane, on the side stream.
void launch_prefetch32(psd_plan* p, const float* x, ll n, ll ldx, cudaStream_t st) {
  cudaEventRecord(p->ev_fork, st);
  cudaStreamWaitEvent(p->side, p->ev_fork, 0);
  const ll nt = (n + 63) / 64;
  psd::symsplit_f32(x, n, ldx, p->stats_alt, nullptr, p->xl_alt, p->ldx32, p->side,
                    std::max<ll>(1, nt * (nt + 1) / 2 / 16));
  psd::copy_to_mapped(p->pf_dev, p->stats_alt, 3 * sizeof(double), p->side);
  cudaEventRecord(p->ev_pf_stats, p->side);
  cudaEventRecord(p->ev_pf_done, p->side);
  p->pf_x = nullptr;
  p->pf_x32 = x;
  p->pf_f32 = true;
  p->pf_n = n;
  p->pf_ldx = ldx;
  p->pf_ready = true;
}

// Enqueue the hinted next X's require_symmetric pass (statistics → mapped slot) and its
// residue planes on the side stream, ordered after everything enqueued on `st` so far.
// Short-lived CTAs (16 tile pairs / 2 rows each) so the work yields SMs to `st`'s
// latency-bound kernels between CTAs; the side stream has the lowest priority.
void launch_prefetch(psd_plan* p, const double* x, ll n, ll ldx, cudaStream_t st) {
  cudaEventRecord(p->ev_fork, st);
  cudaStreamWaitEvent(p->side, p->ev_fork, 0);
  static const int pairs = [] { const char* e = getenv("PSD_PF_PAIRS"); return e ? std::max(1, atoi(e)) : 16; }();
  static const int rows = [] { const char* e = getenv("PSD_PF_ROWS"); return e ? std::max(1, atoi(e)) : 2; }();
  const ll nt = (n + 63) / 64;
  psd::sym_stats(x, n, ldx, p->stats_alt, p->side, p->oz_rowmax_alt, std::max<ll>(1, nt * (nt + 1) / 2 / pairs));
  psd::copy_to_mapped(p->pf_dev, p->stats_alt, 3 * sizeof(double), p->side);
  cudaEventRecord(p->ev_pf_stats, p->side);
  static const int pf_threads = [] { const char* e = getenv("PSD_PF_THREADS"); return e ? atoi(e) : 256; }();
  psd::oz_prepare_rows_max(x, n, n, ldx, p->oz_rowmax_alt, p->oz_e_alt, p->oz_ar_alt, p->oz_ldk, p->side,
                           std::max<ll>(1, n / rows), pf_threads);
  cudaEventRecord(p->ev_pf_done, p->side);
  p->pf_x = x;
  p->pf_x32 = nullptr;
  p->pf_f32 = false;
  p->pf_n = n;
  p->pf_ldx = ldx;
  p->pf_ready = true;
}

// X·P (X bitwise symmetric, residues prepared) as 16 INT8 GEMMs + CRT, panels
// wider than 512 columns (TMEM) in column groups of ≤ 512.
int xmul_oz(psd_plan* p, ll n, const double* P, ll ldP, int w, double* out, ll ldo, double alpha,
            cudaStream_t st) {
  Stage mark(p, PSD_STAGE_SKETCH_GEMM, st);
  const int groups = (w + 511) / 512;
  // the panel's planes are already in g_br (the verification Gram of the final Q): no preparation
  const bool reuse = groups == 1 && p->gq_P == P && p->gq_ld == ldP && p->gq_n == n && p->gq_w == w &&
                     p->g_ldk == p->oz_ldk;
  if (out == p->gq_P) p->gq_P = nullptr;
  const int gw = (w + groups - 1) / groups;
  const ll gw_pad = (gw + 15) / 16 * 16;
  for (int g = 0; g < groups; ++g) {
    const int c0 = g * gw;
    psd::OzOp op;
    op.ar = p->oz_ar;
    op.ldar = p->oz_ldk;
    op.e = p->oz_e;
    op.P = P + c0;
    op.ldp = ldP;
    op.M = (int)n;
    op.N = std::min(gw, w - c0);
    op.K = (int)n;
    op.br = p->oz_br + (size_t)g * psd::oz_num_moduli() * gw_pad * p->oz_ldk;
    op.ldbr = p->oz_ldk;
    op.f = p->oz_f + (size_t)g * gw_pad;
    op.res = p->oz_res;
    op.res_elems = p->oz_res_elems;
    op.C = out + c0;
    op.ldc = ldo;
    op.alpha = alpha;
    op.S = P + c0;
    op.lds = ldP;
    if (reuse) {
      op.br = p->g_br;
      op.ldbr = p->g_ldk;
      op.f = p->g_f;
    }
    if (p->prof) {
      op.ev_gemm[0] = take_event(p);
      op.ev_gemm[1] = take_event(p);
    }
    const int r = reuse ? psd::oz_gemm_prepared(op, st) : psd::oz_gemm(op, st);
    if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "INT8-emulated GEMM rejected its operands (%d)", r);
    if (p->prof) p->marks.push_back({PSD_STAGE_INT8_GEMM, {op.ev_gemm[0], op.ev_gemm[1]}});
  }
  return PSD_OK;
}

// X·P on the 3xTF32 tensor-core path: P (fp64 n×w) → tf32 hi/lo, transposed
// to the K-major B operand; fp32 partials reduced into the fp64 panel `out`.
int xmul_tc32(psd_plan* p, ll n, const float* xhi, ll ldhi, const double* P, ll ldP, int w,
              double* out, ll ldo, double alpha, cudaStream_t st) {
  Stage mark(p, PSD_STAGE_SKETCH_GEMM, st);
  if (out == p->gq_P) p->gq_P = nullptr;
  psd::split_transpose(P, n, w, ldP, p->f[0], p->f[1], p->ldx32, w, st);
  psd::Tc32Op op;
  op.a_hi = xhi;
  op.a_lo = p->xl;
  op.lda = ldhi;
  op.lda_lo = p->ldx32;
  op.b_hi = p->f[0];
  op.b_lo = p->f[1];
  op.ldb = p->ldx32;
  op.M = (int)n;
  op.N = w;
  op.K = (int)n;
  op.mode = 0;
  op.c64 = out;
  op.ldc64 = ldo;
  op.alpha = alpha;
  op.S = P;
  op.lds = ldP;
  op.ws = p->ws32;
  op.ws_elems = p->ws32_elems;
  const int r = psd::gemm_tf32x3(op, st);
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "3xTF32 GEMM rejected its operands (%d)", r);
  return PSD_OK;
}

// require_symmetric on the fp32 X fused with its tf32 split (one HBM pass);
// raw: X itself is the hi operand and only lo is written.
int symcheck32(psd_plan* p, const float* x, ll n, ll ldx, bool raw, SymInfo* si, cudaStream_t st) {
  {
    Stage mark(p, PSD_STAGE_SYMCHECK, st);
    psd::symsplit_f32(x, n, ldx, p->stats, raw ? nullptr : p->xh, p->xl, p->ldx32, st);
  }
  double h[3];
  PSD_CUDA_CHECK(psd::read_small(h, p->stats, 3 * sizeof(double), st),
                 "stats");
  PSD_TRY(sync(st, "symmetry check"));
  int flags = 0;
  std::memcpy(&flags, &h[2], sizeof(int));
  si->max_abs = h[0];
  si->defect = h[1];
  si->bitwise = (flags & 1) == 0;
  si->nonfinite = (flags & 2) != 0;
  return PSD_OK;
}

// x64 (FP64 path) or x32 (FP32 path: 3xTF32 tensor-core GEMMs, FP64 QR/eigh,
// power-scheme multiplies always re-orthonormalised — SURVEY §7 step 8).
static int ran_proj_impl(psd_plan* p, const double* x64, const float* x32, int64_t n, int64_t ldx,
                         const double* omega64, const float* omega32, int64_t ldo, int32_t k,
                         int32_t l, int32_t q, double alpha, uint32_t flags, double* result64,
                         float* result32, int64_t ldr, double* factors_w, int64_t ldw,
                         double* factors_d, psd_report* rep, void* stream) {
  const bool f32 = x32 != nullptr;
  if (k < 1) return fail(PSD_ERR_INVALID_PARAMS, "target rank k must be >= 1, got %d", k);
  if (l < 0) return fail(PSD_ERR_INVALID_PARAMS, "oversampling l must be >= 0, got %d", l);
  if (q < 0) return fail(PSD_ERR_INVALID_PARAMS, "power exponent q must be >= 0, got %d", q);
  if (n < 1) return fail(PSD_ERR_NONSQUARE, "matrix dimension must be at least 1");
  const int w = k + l;
  if (n > p->n || std::min<ll>(w, n) > p->w)
    return fail(PSD_ERR_INVALID_PARAMS, "problem exceeds plan capacity");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  psd::g_launch_count = 0;
  p->oz_gram = false;
  p->gq_P = nullptr;
  psd_report r{};
  r.residual_frob = NAN;
  r.alpha_used = alpha;
  const bool have_result = f32 ? result32 != nullptr : result64 != nullptr;

  // require_symmetric (projection.py:100 / :132) + alpha_tol (projection.py:133-137)
  // With PSD_FLAG_SKIP_SYMCHECK the caller has run require_symmetric and the
  // alpha_tol test itself and tells us via PSD_FLAG_ASSUME_SYMMETRIC whether
  // X is bitwise symmetric (then Xᵀ·P == X·P exactly).
  bool use_t = !(flags & PSD_FLAG_ASSUME_SYMMETRIC);
  // FP32: X itself is the tf32 "hi" operand when its rows are TMA-addressable
  const bool raw = f32 && ldx % 4 == 0 && (uintptr_t)x32 % 16 == 0 && !getenv("PSD_TF32_RNA");
  if (f32) PSD_TRY(ensure_f32(p, !raw));
  const float* xhi = raw ? x32 : p->xh;
  const ll ldhi = raw ? ldx : p->ldx32;
  // FP64 n×n products on the INT8 tensor cores (Ozaki II) when X is bitwise
  // symmetric (Xᵀ·P = X·P, the residues of X's rows serve both); PSD_FP64_OZAKI=0
  // keeps them on the FP64 DMMA kernel.
  static const bool oz_on = [] {
    const char* e = getenv("PSD_FP64_OZAKI");
    return !(e && e[0] == '0');
  }();
  // below n ≈ 3k the per-product residue/CRT passes cost more than DMMA saves
  // (C1 n=1000: 606 vs 697 projections/s; n=2048 par; n=4096: 227 vs 205)
  const bool oz_size = (n >= 3072 || (flags & PSD_FLAG_FP64_INT8)) && n <= psd::oz_max_k();
  bool oz = !f32 && oz_on && oz_size && !(flags & PSD_FLAG_FP64_DMMA);
  // reconstruction SYRK on the INT8 engine too (PSD_OZ_SYRK=0 keeps it on DMMA)
  static const bool oz_syrk_on = [] {
    const char* e = getenv("PSD_OZ_SYRK");
    return !(e && e[0] == '0');
  }();
  if (oz && ensure_oz(p) != PSD_OK) {   // no room for the residue planes: DMMA products
    cudaGetLastError();
    oz = false;
  }
  // pipelined batch (psd_plan_prefetch): the hint names the NEXT call's X; a finished
  // prefetch of THIS call's X replaces the symmetry pass and the residue preparation
  const double* hint_x = p->hint_x;
  const float* hint_x32 = p->hint_x32;
  const ll hint_n = p->hint_n, hint_ldx = p->hint_ldx;
  p->hint_x = nullptr;
  p->hint_x32 = nullptr;
  bool consumed = false;
  // FP32 X usable as the raw tf32 hi operand (ldx % 4, 16-byte aligned; see symcheck32)
  auto raw32 = [](const float* x, ll ld) { return ld % 4 == 0 && (uintptr_t)x % 16 == 0 && !getenv("PSD_TF32_RNA"); };
  if (p->pf_ready && p->pf_f32) {
    if (f32 && p->pf_x32 == x32 && p->pf_n == n && p->pf_ldx == ldx && raw32(x32, ldx) && p->xl &&
        !(flags & PSD_FLAG_SKIP_SYMCHECK)) {
      PSD_CUDA_CHECK(cudaStreamWaitEvent(st, p->ev_pf_done, 0), "prefetch join");
      std::swap(p->xl, p->xl_alt);
      consumed = true;
    }
    p->pf_ready = false;
  }
  if (p->pf_ready) {
    if (oz && p->pf_x == x64 && p->pf_n == n && p->pf_ldx == ldx && !(flags & PSD_FLAG_SKIP_SYMCHECK)) {
      PSD_CUDA_CHECK(cudaStreamWaitEvent(st, p->ev_pf_done, 0), "prefetch join");
      std::swap(p->oz_ar, p->oz_ar_alt);
      std::swap(p->oz_e, p->oz_e_alt);
      std::swap(p->oz_rowmax, p->oz_rowmax_alt);
      consumed = true;
    }
    p->pf_ready = false;   // a mismatched prefetch is dropped (the side stream stays ordered)
  }
  // PSD_PREFETCH=0: off; =eigh: start before the eigensolver (default: before the final QR —
  // measured at C3 30.4 → 32.5–33.4 projections/s; starting at the first product or before
  // the eigensolver gained less: the side stream only gets SMs once the products are done)
  static const int pf_at = [] {
    const char* e = getenv("PSD_PREFETCH");
    return (e && e[0] == '0') ? 0 : (e && e[0] == 'e') ? 2 : 1;
  }();
  const bool prefetch_next = hint_x && oz && pf_at != 0 && hint_n >= 3072 && hint_n <= p->n &&
                             hint_ldx >= hint_n && ensure_pipeline(p) == PSD_OK;
  const bool prefetch_next32 = hint_x32 && f32 && raw && pf_at != 0 && hint_n <= p->n && hint_ldx >= hint_n &&
                               raw32(hint_x32, hint_ldx) && ensure_pipeline32(p) == PSD_OK;
  bool have_rowmax = false;
  // require_symmetric's verdict (and alpha_tol) — evaluated now for FP32, and for FP64 once
  // the first product is enqueued (sym_pending): the statistics travel through an
  // event-tracked mapped-memory read, so the GPU never idles on this host round trip.
  // Nothing observable (the result, factors) is written before the verdict.
  bool sym_pending = false;
  bool sym_prefetched = false;   // the verdict comes from the prefetch's mapped slot
  auto judge = [&](const SymInfo& si) -> int {
    r.max_abs = si.max_abs;
    r.sym_defect = si.defect;
    if (si.nonfinite) return fail(PSD_ERR_CONVERGENCE, "matrix has non-finite entries");
    const double tol = 1e-10 * std::max(1.0, si.max_abs);
    if (si.defect > tol)
      return fail(PSD_ERR_ASYMMETRIC,
                  "matrix is not symmetric: max asymmetry %.3e exceeds tolerance %.3e", si.defect,
                  tol);
    if (alpha > 0.0) {
      const double alpha_tol = 1e-12 * std::max(1.0, si.max_abs);
      if (alpha <= alpha_tol)
        return fail(PSD_ERR_ALPHA_TOO_SMALL,
                    "alpha = %.3e is at or below tolerance %.3e; input is numerically PSD", alpha,
                    alpha_tol);
    }
    use_t = use_t && !si.bitwise && !f32;
    return PSD_OK;
  };
  auto resolve_sym = [&]() -> int {
    if (!sym_pending) return PSD_OK;
    sym_pending = false;
    double h[3];
    if (sym_prefetched) {
      PSD_CUDA_CHECK(cudaEventSynchronize(p->ev_pf_stats), "prefetched stats");
      std::memcpy(h, p->pf_host, sizeof(h));
    } else {
      PSD_CUDA_CHECK(psd::read_small_wait(h, sizeof(h)), "stats");
    }
    SymInfo si;
    int fl = 0;
    std::memcpy(&fl, &h[2], sizeof(int));
    si.max_abs = h[0];
    si.defect = h[1];
    si.bitwise = (fl & 1) == 0;
    si.nonfinite = (fl & 2) != 0;
    PSD_TRY(judge(si));
    r.used_transpose = use_t ? 1 : 0;
    r.sketch_engine = oz ? (use_t ? 3 : 1) : 0;
    return PSD_OK;
  };
  if (!(flags & PSD_FLAG_SKIP_SYMCHECK)) {
    if (f32 && consumed) {   // the verdict of the prefetched symsplit pass
      PSD_CUDA_CHECK(cudaEventSynchronize(p->ev_pf_stats), "prefetched stats");
      double h[3];
      std::memcpy(h, p->pf_host, sizeof(h));
      SymInfo si;
      int fl = 0;
      std::memcpy(&fl, &h[2], sizeof(int));
      si.max_abs = h[0];
      si.defect = h[1];
      si.bitwise = (fl & 1) == 0;
      si.nonfinite = (fl & 2) != 0;
      PSD_TRY(judge(si));
    } else if (f32) {
      SymInfo si;
      PSD_TRY(symcheck32(p, x32, n, ldx, raw, &si, st));
      PSD_TRY(judge(si));
    } else if (consumed) {
      sym_pending = true;
      sym_prefetched = true;
    } else {
      {
        Stage mark(p, PSD_STAGE_SYMCHECK, st);
        psd::sym_stats(x64, n, ldx, p->stats, st, oz ? p->oz_rowmax : nullptr);
      }
      PSD_CUDA_CHECK(psd::read_small_async(p->stats, 3 * sizeof(double), st), "stats");
      sym_pending = true;
      have_rowmax = oz;
    }
  }
  if (w > n) {
    PSD_TRY(resolve_sym());
    return fail(PSD_ERR_INVALID_PARAMS, "k+l = %d exceeds min(m, n) = %lld", w, (ll)n);
  }
  // FP32: Xᵀ·P is taken as X·P — X passed the 1e-10·max|X| symmetry test, far
  // below the path's 1e-4 tolerance.
  if (f32) use_t = false;
  r.used_transpose = use_t ? 1 : 0;

  const ll ld = p->ldp;
  double* bufs[3] = {p->panel[0], p->panel[1], p->panel[2]};
  const double* omega = omega64;
  ll ldo_eff = ldo;
  if (f32) {
    if (flags & PSD_FLAG_SKIP_SYMCHECK)
      psd::split_rows_f32(x32, n, n, ldx, raw ? nullptr : p->xh, p->xl, p->ldx32, n, st);
    // Ω (fp32) → fp64 panel in the Gram/Cholesky workspace-free buffer panel[3]
    psd::convert_f32_f64(omega32, ldo, p->panel[3], ld, n, w, st);
    omega = p->panel[3];
    ldo_eff = ld;
  }
  // 3: X·P products on the INT8 engine, Xᵀ·P (X not bitwise symmetric) on DMMA
  r.sketch_engine = f32 ? 2 : (oz ? (use_t ? 3 : 1) : 0);
  static const bool oz_gram_on = [] { const char* e = getenv("PSD_OZ_GRAM"); return !(e && e[0] == '0'); }();
  // Grams on the INT8 engine wherever it pays (same size rule as the products; the
  // FP32 path's QR is FP64 too)
  p->oz_gram = oz_gram_on && oz_on && oz_size && !(flags & PSD_FLAG_FP64_DMMA);
  if (oz && !consumed) {
    Stage mark(p, PSD_STAGE_SKETCH_GEMM, st);
    if (have_rowmax)   // row scales from the symmetry pass: one read of X
      psd::oz_prepare_rows_max(x64, n, n, ldx, p->oz_rowmax, p->oz_e, p->oz_ar, p->oz_ldk, st);
    else
      psd::oz_prepare_rows(x64, n, n, ldx, p->oz_e, p->oz_ar, p->oz_ldk, st);
  }
  const MulFn mul = [&](const double* P, ll ldP, int ww, double* out, ll ldo2, bool t) {
    if (f32) return xmul_tc32(p, n, xhi, ldhi, P, ldP, ww, out, ldo2, alpha, st);
    if (oz && !(t && use_t)) return xmul_oz(p, n, P, ldP, ww, out, ldo2, alpha, st);
    return xmul(p, x64, n, ldx, P, ldP, ww, out, ldo2, alpha, t && use_t, st);
  };
  int qb = 0, wk = 0;
  QrInfo qi;
  auto start_prefetch = [&]() {
    if (prefetch_next) launch_prefetch(p, hint_x, hint_n, hint_ldx, st);
    if (prefetch_next32) launch_prefetch32(p, hint_x32, hint_n, hint_ldx, st);
  };
  bool pf_started = false;
  auto start_once = [&]() {
    if (!pf_started) start_prefetch();
    pf_started = true;
  };
  auto run_rf = [&]() {
    return range_finder_core(p, mul, n, n, omega, ldo_eff, w, q, f32, (flags & PSD_FLAG_STRICT) != 0, bufs,
                             &qb, &wk, &qi, st, resolve_sym,
                             pf_at == 1 ? std::function<void()>(start_once) : nullptr);
  };
  int rc = run_rf();
  if (rc == kSpanRedo) {   // a device-decided power-step QR needed more passes: host-driven redo
    qi = QrInfo();
    p->span_host = true;
    rc = run_rf();
    p->span_host = false;
  }
  PSD_TRY(rc);
  PSD_TRY(resolve_sym());
  r.qr_passes = qi.passes;
  r.qr_shifted = qi.shifted;
  r.basis_width = wk;
  auto zero_result = [&]() {
    if (f32) cudaMemset2DAsync(result32, ldr * sizeof(float), 0, n * sizeof(float), n, st);
    else psd::fill_zero(result64, ldr, n, n, st);
  };
  if (wk == 0) {  // _zero_report (projection.py:81-89)
    if (have_result) zero_result();
    r.effective_rank = 0;
    r.gpu_launches = psd::g_launch_count;
    if (rep) *rep = r;
    return sync(st, "zero report");
  }
  double* Q = bufs[qb];
  double* C = p->panel[3];
  double* W = p->panel[4];
  double* WD = p->panel[5];

  // compression T = sym(Qᵀ X Q) or sym(Qᵀ B Q)  (projection.py:104 / :143)
  PSD_TRY(mul(Q, ld, wk, C, ld, false));
  {
    Stage mark(p, PSD_STAGE_COMPRESS, st);
    PSD_TRY(panel_tn(p, Q, C, ld, n, wk, p->T, true, st));
  }
  if (pf_at == 2) start_prefetch();
  // eigh (projection.py:105 → symmetric.py:68-86)
  Stage eig_mark(p, PSD_STAGE_EIGH, st);
  if (psd::jacobi_eigh(p->T, wk, wk, p->vals, p->V, wk, p->jws, p->jws_elems, p->ints + p->w + 1, st) < 0)
    return fail(PSD_ERR_CONVERGENCE, "eigen-decomposition failed: Jacobi could not be launched");
  const double offset = alpha > 0.0 ? 1.0 : 0.0;  // max(D − 1, 0) for Alg. 3
  psd::sort_eigs(p->vals, p->V, wk, wk, offset, p->vals_sorted, p->U, wk, p->ints + p->w,
                 p->ints, st);
  int eh[2] = {0, 0};   // {npos, sweeps}: the eigensolver's one host round trip
  PSD_CUDA_CHECK(psd::read_small(eh, p->ints + p->w, sizeof(eh), st), "eigh status");
  PSD_TRY(sync(st, "eigh"));
  if (eh[1] < 0) return fail(PSD_ERR_CONVERGENCE, "eigen-decomposition failed: Jacobi did not converge");
  r.eig_sweeps = eh[1];
  const int npos = eh[0];
  eig_mark.close();
  r.effective_rank = npos;
  Stage recon_mark(p, PSD_STAGE_RECON, st);
  // d = clipped[keep]·scale (projection.py:75-77)
  clip_values_kernel<<<(wk + 255) / 256, 256, 0, st>>>(p->vals_sorted, wk, offset,
                                                        alpha > 0.0 ? alpha : 1.0, p->dvec);
  launched(1);
  if (npos > 0) {
    // W = Q·U₊ ; WD = W·diag(d) ; X̂₊ = WD·Wᵀ on lower tiles, mirrored
    PSD_TRY(panel_nn(p, Q, ld, p->U, wk, W, ld, n, wk, npos, st));
    if (have_result && f32) {
      const int rp = (npos + 15) / 16 * 16;
      psd::split_rows_f64(W, n, npos, ld, p->dvec, p->f[0], p->f[1], rp, rp, st);
      psd::split_rows_f64(W, n, npos, ld, nullptr, p->f[2], p->f[3], rp, rp, st);
      psd::Tc32Op op;
      op.a_hi = p->f[0];
      op.a_lo = p->f[1];
      op.lda = rp;
      op.b_hi = p->f[2];
      op.b_lo = p->f[3];
      op.ldb = rp;
      op.M = (int)n;
      op.N = (int)n;
      op.K = npos;
      op.mode = 1;
      op.c32 = result32;
      op.ldc32 = ldr;
      const int rr = psd::gemm_tf32x3(op, st);
      if (rr < 0) return fail(PSD_ERR_INVALID_PARAMS, "3xTF32 reconstruction rejected its operands (%d)", rr);
    } else if (have_result && oz && oz_syrk_on && npos <= 640) {
      // V = W·diag(√d) as 7 int8 digit planes, X̂₊ = V·Vᵀ from 28 exact slice products
      // per K step on the INT8 tensor cores (Ozaki I, ozaki_syrk.cu); the X residue
      // partials buffer is dead here and holds the planes.
      const int rr = psd::oz_syrk(W, n, npos, ld, p->dvec, result64, ldr, p->oz_res, p->oz_res_elems, st);
      if (rr < 0) return fail(PSD_ERR_INVALID_PARAMS, "INT8 reconstruction rejected its operands (%d)", rr);
      r.recon_engine = 1;
    } else if (have_result) {
      psd::scale_columns(W, ld, p->dvec, WD, ld, n, npos, st);
      psd::GemmOp op;
      op.a_layout = psd::A_MK;
      op.b_layout = psd::B_NK;
      op.A = WD;
      op.lda = ld;
      op.B = W;
      op.ldb = ld;
      op.C = result64;
      op.ldc = ldr;
      op.M = (int)n;
      op.N = (int)n;
      op.K = npos;
      op.epi = psd::EPI_MIRROR;
      op.max_splits = 1;
      psd::gemm_f64(op, p->ws, p->ws_elems, st);
    }
    if (factors_w) {
      psd::copy_matrix(W, ld, factors_w, ldw, n, npos, st);
    }
    if (factors_d) {
      PSD_CUDA_CHECK(cudaMemcpyAsync(factors_d, p->dvec, npos * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st),
                     "factors d");
    }
  } else if (have_result) {
    zero_result();
  }
  recon_mark.close();
  if ((flags & PSD_FLAG_DIAGNOSTICS) && !f32) {
    Stage diag_mark(p, PSD_STAGE_DIAG, st);
    // ‖X − Q(QᵀX)‖_F with QᵀX = (XᵀQ)ᵀ (projection.py:110)
    PSD_TRY(xmul(p, x64, n, ldx, Q, ld, wk, C, ld, 0.0, use_t, st));
    psd::GemmOp op;
    op.a_layout = psd::A_MK;
    op.b_layout = psd::B_NK;
    op.A = Q;
    op.lda = ld;
    op.B = C;
    op.ldb = ld;
    op.C = nullptr;
    op.M = (int)n;
    op.N = (int)n;
    op.K = wk;
    op.epi = psd::EPI_RESID;
    op.S = x64;
    op.lds = ldx;
    op.partials = p->rpart;
    op.max_splits = 1;
    PSD_CUDA_CHECK(cudaMemsetAsync(p->rpart, 0, psd::gemm_resid_ctas(op) * sizeof(double), st),
                   "resid partials");
    psd::gemm_f64(op, p->ws, p->ws_elems, st);
    psd::sum_partials(p->rpart, psd::gemm_resid_ctas(op), p->scal + 2, 1, st);
    PSD_CUDA_CHECK(psd::read_small(&r.residual_frob, p->scal + 2, sizeof(double), st),
                   "residual");
  }
  PSD_TRY(sync(st, "ran_proj"));
  r.gpu_launches = psd::g_launch_count;
  if (rep) *rep = r;
  return PSD_OK;
}

}  // namespace

extern "C" {

int psd_ran_proj(psd_plan* p, const double* x, int64_t n, int64_t ldx, const double* omega,
                 int64_t ldo, int32_t k, int32_t l, int32_t q, double alpha, uint32_t flags,
                 double* result, int64_t ldr, double* factors_w, int64_t ldw, double* factors_d,
                 psd_report* rep, void* stream) {
  if (!p || !x || !omega) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaStream_t st = caller;
  // a call in a pipelined batch runs on the plan's high-priority stream, joined to the
  // caller's at both ends (its CTAs are dispatched ahead of the side stream's)
  const bool piped = (p->hint_x || p->pf_ready) && p->work;
  if (piped) {
    cudaEventRecord(p->ev_in, caller);
    cudaStreamWaitEvent(p->work, p->ev_in, 0);
    st = p->work;
  }
  int status;
  {
    Stage total(p, PSD_STAGE_TOTAL, st);
    status = ran_proj_impl(p, x, nullptr, n, ldx, omega, nullptr, ldo, k, l, q, alpha, flags, result,
                           nullptr, ldr, factors_w, ldw, factors_d, rep, st);
  }
  if (piped) {
    cudaEventRecord(p->ev_out, st);
    cudaStreamWaitEvent(caller, p->ev_out, 0);
  }
  if (p->prof) {
    cudaStreamSynchronize(st);
    collect_marks(p);
  }
  return status;
}

int psd_ran_proj_f32(psd_plan* p, const float* x, int64_t n, int64_t ldx, const float* omega,
                     int64_t ldo, int32_t k, int32_t l, int32_t q, double alpha, uint32_t flags,
                     float* result, int64_t ldr, double* factors_w, int64_t ldw, double* factors_d,
                     psd_report* rep, void* stream) {
  if (!p || !x || !omega) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  const cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaStream_t st = caller;
  const bool piped = (p->hint_x32 || p->pf_ready) && p->work;   // see psd_ran_proj
  if (piped) {
    cudaEventRecord(p->ev_in, caller);
    cudaStreamWaitEvent(p->work, p->ev_in, 0);
    st = p->work;
  }
  int status;
  {
    Stage total(p, PSD_STAGE_TOTAL, st);
    status = ran_proj_impl(p, nullptr, x, n, ldx, nullptr, omega, ldo, k, l, q, alpha, flags, nullptr,
                           result, ldr, factors_w, ldw, factors_d, rep, st);
  }
  if (piped) {
    cudaEventRecord(p->ev_out, st);
    cudaStreamWaitEvent(caller, p->ev_out, 0);
  }
  if (p->prof) {
    cudaStreamSynchronize(st);
    collect_marks(p);
  }
  return status;
}

int psd_syrk_f64_int8(const double* w, int64_t ldw, const double* d, int64_t n, int32_t r,
                      double* result, int64_t ldr, void* stream) {
  if (!w || !d || !result) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (n < 1 || r < 1 || r > 640 || ldw < r || ldr < n) return fail(PSD_ERR_INVALID_PARAMS, "bad syrk shape (r <= 640)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bytes = psd::oz_syrk_ws_bytes(n, r);
  void* ws = nullptr;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(PSD_ERR_NO_MEMORY, "syrk scratch allocation failed");
  }
  int status = PSD_OK;
  const int rr = psd::oz_syrk(w, n, r, ldw, d, result, ldr, ws, bytes, st);
  if (rr < 0) status = fail(PSD_ERR_INVALID_PARAMS, "INT8 SYRK rejected its operands (%d: %s)", rr, cudaGetErrorString(cudaGetLastError()));
  if (status == PSD_OK) status = sync(st, "int8 syrk");
  cudaStreamSynchronize(st);
  cudaFree(ws);
  return status;
}

int psd_gemm_f64_ozaki(const double* a, int64_t lda, const double* pp, int64_t ldp, int64_t m,
                       int64_t nn, int64_t kk, double* c, int64_t ldc, void* stream) {
  if (!a || !pp || !c) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (m < 1 || nn < 1 || nn > 512 || kk < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad ozaki GEMM shape");
  if (kk > psd::oz_max_k()) return fail(PSD_ERR_INVALID_PARAMS, "K exceeds the exact-CRT limit 2^18");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long chunk = m;   // whole A at once (test entry)
  const size_t bytes = psd::oz_stream_ws_bytes(m, nn, kk, chunk);
  void* ws = nullptr;
  if (cudaMalloc(&ws, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(PSD_ERR_NO_MEMORY, "ozaki scratch allocation failed");
  }
  int status = PSD_OK;
  const int r = psd::oz_gemm_stream(a, lda, pp, ldp, m, (int)nn, kk, c, ldc, 0.0, nullptr, 0, ws, bytes,
                                    chunk, st);
  if (r < 0) status = fail(PSD_ERR_INVALID_PARAMS, "ozaki GEMM rejected its operands (%d)", r);
  if (status == PSD_OK) status = sync(st, "ozaki gemm");
  cudaStreamSynchronize(st);
  cudaFree(ws);
  return status;
}

int psd_gemm_f64_int8_ws_bytes(int64_t m, int64_t n, int64_t k, int64_t chunk_rows, int64_t* bytes) {
  if (!bytes) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (m < 1 || n < 1 || k < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad INT8-emulated GEMM shape");
  *bytes = (int64_t)psd::oz_stream_ws_bytes(m, n, k, chunk_rows > 0 ? chunk_rows : 8192);
  return PSD_OK;
}

int psd_gemm_f64_int8(const double* a, int64_t lda, const double* pp, int64_t ldp, int64_t m, int64_t nn,
                      int64_t kk, double* c, int64_t ldc, double alpha, const double* s, int64_t lds,
                      void* ws, int64_t ws_bytes, int64_t chunk_rows, void* stream) {
  if (!a || !pp || !c || !ws) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (m < 1 || nn < 1 || kk < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad INT8-emulated GEMM shape");
  if (alpha > 0.0 && !s) return fail(PSD_ERR_INVALID_PARAMS, "alpha > 0 needs the shift source");
  if (lda < kk || ldp < nn || ldc < nn) return fail(PSD_ERR_INVALID_PARAMS, "leading dimension too small");
  const int r = psd::oz_gemm_stream(a, lda, pp, ldp, m, (int)nn, kk, c, ldc, alpha, s, lds, ws, (size_t)ws_bytes,
                                    chunk_rows > 0 ? chunk_rows : 8192, static_cast<cudaStream_t>(stream));
  if (r == -3) return fail(PSD_ERR_INVALID_PARAMS, "workspace too small (see psd_gemm_f64_int8_ws_bytes)");
  if (r == -4)
    return fail(PSD_ERR_INVALID_PARAMS, "K = %lld exceeds the exact-CRT limit %lld of the INT8 emulation "
                "(use the FP64 DMMA GEMM)", (long long)kk, psd::oz_max_k());
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "INT8-emulated GEMM rejected its operands (%d)", r);
  return PSD_OK;
}

int psd_gemm_tf32x3(int32_t mode, const float* a, int64_t lda, const float* b, int64_t ldb,
                    int64_t m, int64_t nn, int64_t kk, void* c, int64_t ldc, void* stream) {
  if (!a || !b || !c) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (m < 1 || nn < 1 || kk < 1 || mode < 0 || mode > 2 || (mode == 1 && m != nn))
    return fail(PSD_ERR_INVALID_PARAMS, "bad tf32x3 GEMM shape/mode");
  const bool amn = mode == 2;   // a is given transposed (k x m, ld lda)
  if (amn) mode = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ll ldk = (kk + 31) / 32 * 32;
  const ll ldm = (m + 31) / 32 * 32;
  float *ah = nullptr, *al = nullptr, *bh = nullptr, *bl = nullptr, *ws = nullptr;
  const size_t wsz = mode == 0 ? (size_t)psd::tc32_ws_elems(m, (int)nn, std::max<int>(8, (int)((kk + 4095) / 4096))) : 0;
  const size_t asz = amn ? (size_t)kk * ldm : (size_t)m * ldk;
  bool ok = cudaMalloc(&ah, asz * 4) == cudaSuccess &&
            cudaMalloc(&al, asz * 4) == cudaSuccess &&
            cudaMalloc(&bh, (size_t)nn * ldk * 4) == cudaSuccess &&
            cudaMalloc(&bl, (size_t)nn * ldk * 4) == cudaSuccess &&
            (wsz == 0 || cudaMalloc(&ws, wsz * 4) == cudaSuccess);
  int status = PSD_OK;
  if (!ok) {
    status = fail(PSD_ERR_NO_MEMORY, "tf32x3 scratch allocation failed");
  } else {
    if (amn) psd::split_rows_f32(a, kk, m, lda, ah, al, ldm, ldm, st);
    else psd::split_rows_f32(a, m, kk, lda, ah, al, ldk, ldk, st);
    psd::split_rows_f32(b, nn, kk, ldb, bh, bl, ldk, ldk, st);
    psd::Tc32Op op;
    op.a_hi = ah;
    op.a_lo = al;
    op.lda = amn ? ldm : ldk;
    op.a_mn = amn;
    op.b_hi = bh;
    op.b_lo = bl;
    op.ldb = ldk;
    op.M = (int)m;
    op.N = (int)nn;
    op.K = (int)kk;
    op.mode = mode;
    op.c64 = static_cast<double*>(c);
    op.ldc64 = ldc;
    op.c32 = static_cast<float*>(c);
    op.ldc32 = ldc;
    op.ws = ws;
    op.ws_elems = wsz;
    const int r = psd::gemm_tf32x3(op, st);
    if (r < 0) status = fail(PSD_ERR_INVALID_PARAMS, "3xTF32 GEMM rejected its operands (%d)", r);
    if (status == PSD_OK) status = sync(st, "tf32x3 gemm");
  }
  cudaStreamSynchronize(st);
  cudaFree(ah);
  cudaFree(al);
  cudaFree(bh);
  cudaFree(bl);
  cudaFree(ws);
  return status;
}

int psd_plan_profile(psd_plan* p, int32_t enable, double* ms_out, int32_t* counts_out,
                     int32_t reset) {
  if (!p) return fail(PSD_ERR_INVALID_PARAMS, "null plan");
  if (enable >= 0) p->prof = enable != 0;
  for (int i = 0; i < PSD_NUM_STAGES; ++i) {
    if (ms_out) ms_out[i] = p->stage_ms[i];
    if (counts_out) counts_out[i] = p->stage_cnt[i];
    if (reset) {
      p->stage_ms[i] = 0.0;
      p->stage_cnt[i] = 0;
    }
  }
  return PSD_OK;
}

int psd_reconstruct(psd_plan* p, const double* w, int64_t n, int64_t ldw, const double* d,
                    int32_t r, double* result, int64_t ldr, void* stream) {
  if (!p || !w || !d || !result) return fail(PSD_ERR_INVALID_PARAMS, "null argument");
  if (n < 1 || n > p->n || r < 0 || r > p->w) return fail(PSD_ERR_INVALID_PARAMS, "reconstruct shape outside plan");
  DeviceGuard g(p->device);
  std::lock_guard<std::recursive_mutex> dev_lock(device_mutex(p->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (r == 0) {
    psd::fill_zero(result, ldr, n, n, st);
    return sync(st, "reconstruct");
  }
  double* WD = p->panel[5];
  psd::scale_columns(w, ldw, d, WD, p->ldp, n, r, st);
  psd::GemmOp op;
  op.a_layout = psd::A_MK;
  op.b_layout = psd::B_NK;
  op.A = WD;
  op.lda = p->ldp;
  op.B = w;
  op.ldb = ldw;
  op.C = result;
  op.ldc = ldr;
  op.M = (int)n;
  op.N = (int)n;
  op.K = r;
  op.epi = psd::EPI_MIRROR;
  op.max_splits = 1;
  psd::gemm_f64(op, p->ws, p->ws_elems, st);
  return sync(st, "reconstruct");
}

int psd_symmetrize(double* a, int64_t m, int64_t lda, void* stream) {
  if (!a || m < 1) return fail(PSD_ERR_NONSQUARE, "expected a square matrix");
  psd::symmetrize_small(a, (int)m, lda, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "symmetrize");
  return PSD_OK;
}

int psd_gemm_f64(int32_t a_layout, int32_t b_layout, const double* a, int64_t lda, const double* b,
                 int64_t ldb, double* c, int64_t ldc, int32_t m, int32_t n, int32_t k,
                 int32_t epilogue, double alpha, const double* s, int64_t lds, double* ws,
                 int64_t ws_elems, void* stream) {
  if (!a || !b || !c || m < 0 || n < 0 || k < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad gemm arguments");
  if (epilogue < 0 || epilogue > 3) return fail(PSD_ERR_INVALID_PARAMS, "bad epilogue %d", epilogue);
  if ((epilogue == 1 || epilogue == 2) && !s) return fail(PSD_ERR_INVALID_PARAMS, "epilogue needs S");
  if (epilogue == 3 && (m != n || a_layout != 0 || b_layout != 1))
    return fail(PSD_ERR_INVALID_PARAMS, "mirrored store needs M == N, A row-major, B^T stored");
  psd::GemmOp op;
  op.a_layout = a_layout;
  op.b_layout = b_layout;
  op.A = a;
  op.lda = lda;
  op.B = b;
  op.ldb = ldb;
  op.C = c;
  op.ldc = ldc;
  op.M = m;
  op.N = n;
  op.K = k;
  op.epi = epilogue;
  op.alpha = alpha;
  op.S = s;
  op.lds = lds;
  op.max_splits = (ws && ws_elems > 0 && epilogue <= 1) ? 256 : 1;
  const int r = psd::gemm_f64(op, ws, ws ? (size_t)ws_elems : 0, static_cast<cudaStream_t>(stream));
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "unsupported layout pair (%d, %d)", a_layout, b_layout);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "gemm");
  return PSD_OK;
}

int psd_chol_inv(const double* g, int32_t m, int64_t ldg, double shift, double* l, int64_t ldl,
                 double* rinv, int64_t ldr, double* scratch, double* status, void* stream) {
  if (!g || !l || !rinv || !scratch || !status || m < 1)
    return fail(PSD_ERR_INVALID_PARAMS, "bad chol_inv arguments");
  if (psd::chol_inv(g, ldg, m, shift, l, ldl, rinv, ldr, scratch, status,
                    static_cast<cudaStream_t>(stream)) != 0)
    return fail(PSD_ERR_INVALID_PARAMS, "size %d too large for the CholeskyQR kernel", m);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "chol_inv");
  return PSD_OK;
}

int psd_scale_columns(const double* w, int64_t ldw, const double* d, double* out, int64_t ldo,
                      int64_t rows, int32_t cols, void* stream) {
  if (!w || !d || !out || rows < 0 || cols < 0) return fail(PSD_ERR_INVALID_PARAMS, "bad scale_columns");
  psd::scale_columns(w, ldw, d, out, ldo, rows, cols, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "scale_columns");
  return PSD_OK;
}

int psd_max_abs(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                void* stream) {
  if (!x || !out || rows < 0 || cols < 0) return fail(PSD_ERR_INVALID_PARAMS, "bad max_abs");
  psd::max_abs(x, rows, cols, ldx, out, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "max_abs");
  return PSD_OK;
}

int psd_syrk_window(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t n,
                    int32_t k, int64_t r0, int64_t r1, double* out, int64_t ldo, void* stream) {
  if (!a || !b || !out || n < 1 || k < 1 || r0 < 0 || r1 > n || r0 >= r1)
    return fail(PSD_ERR_INVALID_PARAMS, "bad syrk_window arguments");
  psd::GemmOp op;
  op.a_layout = psd::A_MK;
  op.b_layout = psd::B_NK;
  op.A = a;
  op.lda = lda;
  op.B = b;
  op.ldb = ldb;
  op.C = out;
  op.ldc = ldo;
  op.M = (int)n;
  op.N = (int)n;
  op.K = k;
  op.epi = psd::EPI_MIRROR;
  op.max_splits = 1;
  op.win0 = (int)r0;
  op.win1 = (int)r1;
  const int r = psd::gemm_f64(op, nullptr, 0, static_cast<cudaStream_t>(stream));
  if (r < 0) return fail(PSD_ERR_INVALID_PARAMS, "syrk_window needs 16-byte aligned operands");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "syrk_window");
  return PSD_OK;
}

int psd_fill_sym_gaussian(double* out, int64_t ldo, int64_t r0, int64_t rows, int64_t n,
                          uint64_t seed, double scale, double beta, void* stream) {
  if (!out || rows < 0 || n < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad sym gaussian fill");
  psd::sym_gaussian_rows(out, ldo, r0, rows, n, seed, scale, beta, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sym gaussian");
  return PSD_OK;
}

int psd_pair_defect(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t rows,
                    int64_t cols, double* stats, int32_t reset, void* stream) {
  if (!a || !b || !stats || rows < 0 || cols < 0 || lda < cols || ldb < rows)
    return fail(PSD_ERR_INVALID_PARAMS, "bad pair_defect arguments");
  psd::pair_defect(a, lda, b, ldb, rows, cols, stats, reset != 0, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "pair_defect");
  return PSD_OK;
}

int psd_sdls_assemble(const double* cr, int64_t n, const int64_t* pos, const int32_t* ptr,
                      const int32_t* econ, const double* evals, const double* y, int32_t npos,
                      double* x, void* stream) {
  if (!cr || !x || n < 1 || npos < 0) return fail(PSD_ERR_INVALID_PARAMS, "bad sdls_assemble");
  psd::sdls_assemble(cr, n, reinterpret_cast<const long long*>(pos), ptr, econ, evals, y, npos, x,
                     static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sdls_assemble");
  return PSD_OK;
}

int psd_sdls_traces(const double* wd, const double* w, int64_t ldw, int32_t r, const int32_t* rows,
                    const int32_t* cols, const double* vals, const int32_t* cptr, int32_t m,
                    double* t, void* stream) {
  if (!t || m < 0 || r < 0) return fail(PSD_ERR_INVALID_PARAMS, "bad sdls_traces");
  if (r == 0) {
    cudaMemsetAsync(t, 0, (size_t)m * sizeof(double), static_cast<cudaStream_t>(stream));
    return PSD_OK;
  }
  psd::sdls_traces(wd, w, ldw, r, rows, cols, vals, cptr, m, t, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sdls_traces");
  return PSD_OK;
}

int psd_sdls_traces_dense(const double* x, int64_t ldx, const int32_t* rows, const int32_t* cols,
                          const double* vals, const int32_t* cptr, int32_t m, double* t,
                          void* stream) {
  if (!x || !t || m < 0 || ldx < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad sdls_traces_dense");
  psd::sdls_traces_dense(x, ldx, rows, cols, vals, cptr, m, t, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sdls_traces_dense");
  return PSD_OK;
}

int psd_sdls_step(const double* b, const double* t, double* y, double* grad, int32_t m,
                  double beta, double eps, double* out, void* stream) {
  if (!b || !t || !y || !grad || !out || m < 0) return fail(PSD_ERR_INVALID_PARAMS, "bad sdls_step");
  psd::sdls_step(b, t, y, grad, m, beta, eps, out, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "sdls_step");
  return PSD_OK;
}

int psd_fill_gaussian(double* out, int64_t rows, int32_t cols, int64_t ld, uint64_t seed,
                      uint64_t offset, void* stream) {
  if (!out || rows < 1 || cols < 1) return fail(PSD_ERR_INVALID_PARAMS, "bad gaussian fill");
  psd::philox_normal(out, rows, cols, ld, seed, offset, static_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "philox");
  return PSD_OK;
}

}  // extern "C"
