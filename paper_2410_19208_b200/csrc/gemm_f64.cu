// Instantiations and the split-K / tiling policy for the DMMA GEMM.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "launch.h"

namespace psd {

// X·P (sketch / power scheme / compression), Y·R⁻¹, Q·U:   A row-major, B row-major.
using CfgPanelNN = GemmCfg<64, 2, 4, 9, 16, 4, A_MK, B_KN>;
// Xᵀ·P (sketch.py:79 exact semantics), Gram YᵀY, Qᵀ(XQ):    A transposed, B row-major.
using CfgPanelTN = GemmCfg<64, 2, 4, 9, 16, 4, A_KM, B_KN>;
// (W·D)·Wᵀ reconstruction (lower tiles, mirrored), residual, Cholesky trailing update.
using CfgSquareNT = GemmCfg<128, 2, 4, 4, 16, 4, A_MK, B_NK>;

const DeviceInfo& device_info() {
  static DeviceInfo info[16];
  static bool init[16] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!init[dev]) {
    cudaDeviceGetAttribute(&info[dev].sms, cudaDevAttrMultiProcessorCount, dev);
    int smem = 0;
    cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    info[dev].max_smem = smem;
    init[dev] = true;
  }
  return info[dev];
}

template <class Cfg>
static void ensure_attr() {
  static bool done[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!done[dev]) {
    cudaFuncSetAttribute(gemm_f64_kernel<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg::kSmem);
    done[dev] = true;
  }
}

static bool aligned16(const void* p, long long ld) {
  return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0);
}

template <class Cfg>
static void tiling(const GemmOp& op, int& m_tiles, int& n_tiles, int& nb_per_tile) {
  const int N8 = (op.N + 7) / 8;
  constexpr int TN8 = Cfg::BN / 8;
  m_tiles = (op.M + Cfg::BM - 1) / Cfg::BM;
  if (op.epi == EPI_MIRROR) {
    n_tiles = 1;
    nb_per_tile = TN8;
    return;
  }
  n_tiles = std::max(1, (N8 + TN8 - 1) / TN8);
  nb_per_tile = std::max(1, (N8 + n_tiles - 1) / n_tiles);
}

template <class Cfg>
static int launch_cfg(const GemmOp& op, double* ws, size_t ws_elems, cudaStream_t st) {
  ensure_attr<Cfg>();
  int m_tiles, n_tiles, nb;
  tiling<Cfg>(op, m_tiles, n_tiles, nb);
  GemmParams p{};
  p.A = op.A;
  p.lda = op.lda;
  p.B = op.B;
  p.ldb = op.ldb;
  p.C = op.C;
  p.ldc = op.ldc;
  p.M = op.M;
  p.N = op.N;
  p.K = op.K;
  p.nb_per_tile = nb;
  p.epi = op.epi;
  p.a_vec = aligned16(op.A, op.lda);
  p.b_vec = aligned16(op.B, op.ldb);
  p.alpha = op.alpha;
  p.S = op.S;
  p.lds = op.lds;
  p.partials = op.partials;
  p.split_stride = 0;

  constexpr int BK = Cfg::BK;
  const int sms = device_info().sms;
  const long long tiles = (long long)m_tiles * n_tiles;
  int splits = 1;
  const long long ldw = (op.N + 1) / 2 * 2;
  if ((op.epi == EPI_STORE || op.epi == EPI_SHIFT) && op.max_splits > 1 && ws != nullptr) {
    // minimise waves × K-chunk (the critical path), preferring fewer splits
    double best = 1e300;
    const int smax = std::min<long long>(op.max_splits, std::max(1, op.K / (4 * BK)));
    for (int s = 1; s <= smax; ++s) {
      const long long kc = ((op.K + s - 1) / s + BK - 1) / BK * BK;
      const long long s_eff = (op.K + kc - 1) / kc;
      if (s_eff != s) continue;
      if (s > 1 && (size_t)s * op.M * ldw > ws_elems) break;
      const long long waves = (tiles * s + sms - 1) / sms;
      const double cost = (double)waves * (double)kc + (s > 1 ? 96.0 : 0.0);
      if (cost < best * 0.995) {
        best = cost;
        splits = s;
      }
    }
  }
  if (splits > 1) {
    const long long kc = ((op.K + splits - 1) / splits + BK - 1) / BK * BK;
    p.k_chunk = (int)kc;
    p.C = ws;
    p.ldc = ldw;
    p.split_stride = (long long)op.M * ldw;
    p.epi = EPI_STORE;
  } else {
    p.k_chunk = std::max(op.K, 1);
  }
  dim3 grid;
  if (op.epi == EPI_MIRROR) {
    const long long nt = m_tiles;
    grid = dim3((unsigned)(nt * (nt + 1) / 2), 1, 1);
  } else {
    grid = dim3(m_tiles, n_tiles, splits);
  }
  if (grid.x == 0) return 0;
  gemm_f64_kernel<Cfg><<<grid, Cfg::kThreads, Cfg::kSmem, st>>>(p);
  count_launch();
  if (splits > 1) {
    splitk_reduce(ws, splits, p.split_stride, op.M, op.N, ldw, op.C, op.ldc, op.epi, op.alpha,
                  op.S, op.lds, st);
    return 2;
  }
  return 1;
}

static bool legacy_forced() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PSD_GEMM");
    v = (e && e[0] == 'l') ? 1 : 0;  // PSD_GEMM=legacy → cp.async kernel only (A/B testing)
  }
  return v == 1;
}

int gemm_f64(const GemmOp& op, double* ws, size_t ws_elems, cudaStream_t st) {
  if (op.M <= 0 || op.N <= 0) return 0;
  if (!legacy_forced()) {
    const int r = gemm_f64_tma(op, ws, ws_elems, st);
    if (r != -2) return r;
  }
  if (op.epi == EPI_MIRROR && (op.win0 != 0 || (op.win1 != 0 && op.win1 != op.M)))
    return -3;  // row-windowed mirror store needs the TMA path (16-byte aligned operands)
  if (op.a_layout == A_MK && op.b_layout == B_KN) return launch_cfg<CfgPanelNN>(op, ws, ws_elems, st);
  if (op.a_layout == A_KM && op.b_layout == B_KN) return launch_cfg<CfgPanelTN>(op, ws, ws_elems, st);
  if (op.a_layout == A_MK && op.b_layout == B_NK) return launch_cfg<CfgSquareNT>(op, ws, ws_elems, st);
  return -1;
}

long long gemm_resid_ctas(const GemmOp& op) {
  int m_tiles, n_tiles, nb;
  tiling<CfgSquareNT>(op, m_tiles, n_tiles, nb);
  return std::max<long long>((long long)m_tiles * n_tiles, gemm_tma_resid_parts(op));
}

}  // namespace psd
