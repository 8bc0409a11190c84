// FP64 tensor-core (DMMA) GEMM for sm_100a.
//
// tcgen05 has no kind::f64, so the B200 FP64 tensor path is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) with register accumulators.  This
// kernel keeps the DMMA pipe fed with a cp.async (LDGSTS) multi-stage
// shared-memory pipeline whose row strides are ≡ 4 (mod 16) doubles, which
// makes every 64-bit fragment load bank-conflict free for all four operand
// layouts (A: MK / KM, B: KN / NK).
//
// C[M×N] = Σ_k A(m,k)·B(k,n), tiled BM × BN × BK; each warp column owns a
// contiguous run of ≤ MAXN8 n8-blocks, distributed so the four SM
// sub-partitions (warp % 4) carry equal DMMA work even when N/8 is not a
// multiple of the warp-column count (e.g. w = 272 → 34 n8-blocks → 8/9/8/9).
#pragma once
#include "common.cuh"

namespace psd {

enum ALayout { A_MK = 0, A_KM = 1 };
enum BLayout { B_KN = 0, B_NK = 1 };
enum Epilogue {
  EPI_STORE = 0,   // C = acc                                  (split-K: raw partial)
  EPI_SHIFT = 1,   // C = (acc + α·S)/α    — B = (X + αI)/α fused (projection.py:139)
  EPI_SUB = 2,     // C = S − acc          — trailing Cholesky update
  EPI_MIRROR = 3,  // lower-tri tiles, C[m][n] = C[n][m] = acc for m ≥ n (SYRK store)
  EPI_RESID = 4,   // partial Σ (S − acc)² per CTA             (projection.py:110)
};

struct GemmParams {
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;
  long long ldc;
  int M, N, K;
  int k_chunk;             // K per split (multiple of BK)
  long long split_stride;  // elements between split slices of C
  int nb_per_tile;         // n8 blocks per CTA N-tile
  int epi;
  int a_vec, b_vec;        // 16-byte cp.async legal for A / B
  double alpha;
  const double* S;
  long long lds;
  double* partials;
};

template <int BM_, int WARPS_M_, int WARPS_N_, int MAXN8_, int BK_, int STAGES_, int AL_, int BL_>
struct GemmCfg {
  static constexpr int BM = BM_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, MAXN8 = MAXN8_;
  static constexpr int BK = BK_, STAGES = STAGES_, AL = AL_, BL = BL_;
  static constexpr int kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int BN = WARPS_N * MAXN8 * 8;
  static constexpr int WM = BM / WARPS_M;
  static constexpr int M8 = WM / 8;
  static constexpr int SA = (AL == A_MK) ? (BK + 4) : (BM + 4);
  static constexpr int A_ELEMS = (AL == A_MK) ? BM * SA : BK * SA;
  static constexpr int SB = (BL == B_KN) ? (BN + 4) : (BK + 4);
  static constexpr int B_ELEMS = (BL == B_KN) ? BK * SB : BN * SB;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t kSmem = size_t(STAGES) * STAGE_ELEMS * sizeof(double);
  static_assert(WM % 8 == 0, "warp M tile must be a multiple of 8");
  static_assert(SA % 16 == 4 && SB % 16 == 4, "strides must be 4 mod 16 doubles");
  static_assert(STAGE_ELEMS % 2 == 0, "stage must keep 16-byte alignment");
};

template <class Cfg>
PSD_DEVINL double a_at(const double* sA, int m, int k) {
  if constexpr (Cfg::AL == A_MK) return sA[m * Cfg::SA + k];
  else return sA[k * Cfg::SA + m];
}

template <class Cfg>
PSD_DEVINL double b_at(const double* sB, int k, int n) {
  if constexpr (Cfg::BL == B_KN) return sB[k * Cfg::SB + n];
  else return sB[n * Cfg::SB + k];
}

// Copy a R×Ccols tile of a row-major global matrix (row r, col c → g[r*ld + c])
// into shared memory with row stride SS, zero-filling outside [rlim, clim).
template <int R, int CC, int SS, int NT>
PSD_DEVINL void load_tile(double* s, const double* g, long long ld, int r0, int c0, int rlim,
                          int clim, bool vec) {
  if (vec) {
    constexpr int CPR = CC / 2;
#pragma unroll 4
    for (int c = threadIdx.x; c < R * CPR; c += NT) {
      const int r = c / CPR, cc = (c % CPR) * 2;
      const int gr = r0 + r, gc = c0 + cc;
      int valid = 0;
      if (gr < rlim) valid = min(max(clim - gc, 0), 2);
      const double* src = valid ? g + (long long)gr * ld + gc : g;
      cp_async16(s + r * SS + cc, src, valid * 8);
    }
  } else {
#pragma unroll 4
    for (int c = threadIdx.x; c < R * CC; c += NT) {
      const int r = c / CC, cc = c % CC;
      const int gr = r0 + r, gc = c0 + cc;
      const bool valid = gr < rlim && gc < clim;
      const double* src = valid ? g + (long long)gr * ld + gc : g;
      cp_async8(s + r * SS + cc, src, valid ? 8 : 0);
    }
  }
}

template <class Cfg>
PSD_DEVINL void load_stage(double* st, const GemmParams& p, int m0, int n0, int nlim, int k0,
                           int kend) {
  double* sA = st;
  double* sB = st + Cfg::A_ELEMS;
  constexpr int NT = Cfg::kThreads;
  if constexpr (Cfg::AL == A_MK)
    load_tile<Cfg::BM, Cfg::BK, Cfg::SA, NT>(sA, p.A, p.lda, m0, k0, p.M, kend, p.a_vec);
  else
    load_tile<Cfg::BK, Cfg::BM, Cfg::SA, NT>(sA, p.A, p.lda, k0, m0, kend, p.M, p.a_vec);
  if constexpr (Cfg::BL == B_KN)
    load_tile<Cfg::BK, Cfg::BN, Cfg::SB, NT>(sB, p.B, p.ldb, k0, n0, kend, nlim, p.b_vec);
  else
    load_tile<Cfg::BN, Cfg::BK, Cfg::SB, NT>(sB, p.B, p.ldb, n0, k0, nlim, kend, p.b_vec);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kThreads, 1) gemm_f64_kernel(const GemmParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BK = Cfg::BK, STAGES = Cfg::STAGES, M8 = Cfg::M8, MAXN8 = Cfg::MAXN8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  int m0, n0;
  if (p.epi == EPI_MIRROR) {
    // lower-triangular tile pairs (ti ≥ tj), BM == BN
    const long long x = blockIdx.x;
    int ti = (int)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= x) ++ti;
    while ((long long)ti * (ti + 1) / 2 > x) --ti;
    const int tj = (int)(x - (long long)ti * (ti + 1) / 2);
    m0 = ti * Cfg::BM;
    n0 = tj * p.nb_per_tile * 8;
  } else {
    m0 = blockIdx.x * Cfg::BM;
    n0 = blockIdx.y * p.nb_per_tile * 8;
  }
  const int nlim = min(p.N, n0 + p.nb_per_tile * 8);
  const int kbeg = blockIdx.z * p.k_chunk;
  const int kend = min(p.K, kbeg + p.k_chunk);
  const int nk = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  // warp → (M row, N column); column c = (smsp + wm) % WARPS_N balances SMSPs
  const int wm = warp / Cfg::WARPS_N;
  const int wc = ((warp % Cfg::WARPS_N) + wm) % Cfg::WARPS_N;
  const int nb = max(0, (nlim - n0 + 7) / 8);
  const int nstart = wc * nb / Cfg::WARPS_N;
  const int ncnt = (wc + 1) * nb / Cfg::WARPS_N - nstart;

  double acc[M8][MAXN8][2];
#pragma unroll
  for (int i = 0; i < M8; ++i)
#pragma unroll
    for (int j = 0; j < MAXN8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage<Cfg>(smem + s * Cfg::STAGE_ELEMS, p, m0, n0, nlim, kbeg + s * BK, kend);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < nk)
      load_stage<Cfg>(smem + (pf % STAGES) * Cfg::STAGE_ELEMS, p, m0, n0, nlim, kbeg + pf * BK,
                      kend);
    cp_async_commit();
    const double* sA = smem + (kt % STAGES) * Cfg::STAGE_ELEMS;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[M8], bf[MAXN8];
#pragma unroll
      for (int i = 0; i < M8; ++i) af[i] = a_at<Cfg>(sA, wm * Cfg::WM + i * 8 + g, kk * 4 + t);
#pragma unroll
      for (int j = 0; j < MAXN8; ++j) bf[j] = b_at<Cfg>(sB, kk * 4 + t, (nstart + j) * 8 + g);
#pragma unroll
      for (int j = 0; j < MAXN8; ++j) {
        if (j < ncnt) {
#pragma unroll
          for (int i = 0; i < M8; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---------------------------------------------------------------- epilogue
  double* C = p.C + (long long)blockIdx.z * p.split_stride;
  double resid = 0.0;
#pragma unroll
  for (int i = 0; i < M8; ++i) {
    const int m = m0 + wm * Cfg::WM + i * 8 + g;
#pragma unroll
    for (int j = 0; j < MAXN8; ++j) {
      if (j >= ncnt) continue;
      const int n = n0 + (nstart + j) * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int nn = n + e;
        if (m >= p.M || nn >= nlim) continue;
        const double v = acc[i][j][e];
        switch (p.epi) {
          case EPI_STORE: C[(long long)m * p.ldc + nn] = v; break;
          case EPI_SHIFT:
            C[(long long)m * p.ldc + nn] = (v + p.alpha * p.S[(long long)m * p.lds + nn]) / p.alpha;
            break;
          case EPI_SUB: C[(long long)m * p.ldc + nn] = p.S[(long long)m * p.lds + nn] - v; break;
          case EPI_MIRROR:
            if (m >= nn) {
              C[(long long)m * p.ldc + nn] = v;
              C[(long long)nn * p.ldc + m] = v;
            }
            break;
          case EPI_RESID: {
            const double d = p.S[(long long)m * p.lds + nn] - v;
            resid = fma(d, d, resid);
          } break;
        }
      }
    }
  }
  if (p.epi == EPI_RESID) {
    __shared__ double red[32];
    __syncthreads();
    resid = warp_sum(resid);
    if (lane == 0) red[warp] = resid;
    __syncthreads();
    if (warp == 0) {
      double v = lane < Cfg::kThreads / 32 ? red[lane] : 0.0;
      v = warp_sum(v);
      if (lane == 0) {
        const long long b = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        p.partials[b] = v;
      }
    }
  }
}

}  // namespace psd
