// TMA-fed, warp-specialised, persistent FP64 DMMA GEMM for sm_100a.
//
// tcgen05 has no kind::f64, so FP64 tensor work on B200 is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) with register accumulators.  This
// kernel takes every load instruction out of the math warps:
//   * warp kConsumers (the producer) has one elected lane that streams
//     A/B tiles with cp.async.bulk.tensor (TMA, SWIZZLE_128B) into a
//     STAGES-deep shared-memory ring, signalling mbarrier `full[s]` with
//     complete_tx and waiting on `empty[s]` before reusing a slot;
//   * consumer warps only do LDS.64 fragment loads + DMMA, waiting on
//     `full[s]` and releasing `empty[s]` per warp — no __syncthreads, so
//     warps drift apart and cover each other's latency.
// Persistent: gridDim.x ≤ #SMs CTAs walk the (m-tile, n-tile, k-split) work
// list; the producer runs ahead across work units, so a unit's epilogue
// overlaps the next unit's loads.
//
// Conflict-free 64-bit fragment loads from 128B-swizzled tiles: the mma row
// (or column) index of each lane is remapped to a physical row/column such
// that the 16 lanes of each half-warp hit 16 distinct (16B-chunk, half)
// pairs.  For tiles whose K is the contiguous dimension (A row-major, Bᵀ
// stored) lane g reads row π(g) = ((g&3)<<1)|(g>>2); for tiles whose M/N is
// contiguous (Aᵀ stored, B row-major) lane g of n8-block jj in a 16-wide box
// reads column ν(g,jj) = (g&1)|((g>>2&1)<<1)|(jj<<2)|((g>>1&1)<<3).  The
// epilogue applies the same maps to the accumulator coordinates.
#pragma once
#include <cuda.h>

#include "gemm_f64.cuh"

namespace psd {

template <int AL_, int BL_, int BM_, int WARPS_M_, int WARPS_N_, int M8W_, int N8W_, int STAGES_,
          bool STAGED_EPI_ = false>
struct TmaCfg {
  static constexpr int AL = AL_, BL = BL_, BM = BM_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int M8W = M8W_, N8W = N8W_, STAGES = STAGES_;
  // EPI_MIRROR through shared memory: consumers park the tile in smem and the
  // three otherwise idle producer-warpgroup warps store it (both orientations,
  // 256-byte rows) while the consumers run the next tile's MMAs.
  static constexpr bool STAGED_EPI = STAGED_EPI_;
  static constexpr int BK = 16;
  static constexpr int BN = WARPS_N * N8W * 8;
  static constexpr int kConsumers = WARPS_M * WARPS_N;
  // consumer warpgroups + one producer warpgroup (setmaxnreg works per warpgroup)
  static constexpr int kThreads = (kConsumers + 4) * 32;
  static constexpr int kConsumerRegs = 232;  // 2 consumer warps + 1 producer warp per SMSP
  static constexpr int kProducerRegs = 40;   //   (2·232 + 40)·32 ≤ 16384 registers
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int C_LD = BN + 1;  // staged tile row stride (doubles)
  static constexpr size_t C_BYTES = STAGED_EPI ? (size_t)BM * C_LD * 8 : 0;
  static constexpr size_t kSmem = (size_t)STAGES * STAGE_BYTES + C_BYTES + 1024;
  static_assert(BM == WARPS_M * M8W * 8, "BM must equal WARPS_M*M8W*8");
  static_assert(kConsumers % 4 == 0, "consumers form whole warpgroups");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle atoms are 1 KiB");
  static_assert(AL == A_MK ? BM <= 256 : BM % 16 == 0, "A box");
  static_assert(BL == B_NK ? BN <= 256 : BN % 16 == 0, "B box");
};

struct TmaParams {
  double* C;
  long long ldc;
  int M, N, K;
  int k_chunk;
  long long split_stride;
  int m_tiles, n_tiles, splits;
  int units;
  int win0, win1;  // EPI_MIRROR: only rows [win0, win1) of the symmetric result, stored at C + (row − win0)·ldc
  int epi;
  double alpha;
  const double* S;
  long long lds;
  double* partials;
};

// ---- PTX wrappers ------------------------------------------------------------
PSD_DEVINL void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
PSD_DEVINL void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
PSD_DEVINL void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
PSD_DEVINL void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
PSD_DEVINL void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// named CTA barriers between warp roles (id 0 is __syncthreads)
PSD_DEVINL void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
PSD_DEVINL void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
PSD_DEVINL void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

PSD_DEVINL double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// row permutation for K-contiguous tiles, column permutation for M/N-contiguous tiles
PSD_DEVINL int pi_row(int g) { return ((g & 3) << 1) | (g >> 2); }
PSD_DEVINL int nu_col(int g, int jj) {
  return (g & 1) | (((g >> 2) & 1) << 1) | (jj << 2) | (((g >> 1) & 1) << 3);
}

// byte offset of A(m, k) inside an A stage, m ∈ [0,BM), k ∈ [0,16)
template <class Cfg>
PSD_DEVINL uint32_t a_off(int m, int k) {
  if constexpr (Cfg::AL == A_MK) {
    return m * 128 + ((((k >> 1) ^ (m & 7))) << 4) + ((k & 1) << 3);
  } else {
    const int ml = m & 15;
    return (m >> 4) * 2048 + k * 128 + ((((ml >> 1) ^ (k & 7))) << 4) + ((ml & 1) << 3);
  }
}
// byte offset of B(k, n) inside a B stage, n ∈ [0,BN), k ∈ [0,16)
template <class Cfg>
PSD_DEVINL uint32_t b_off(int k, int n) {
  if constexpr (Cfg::BL == B_KN) {
    const int nl = n & 15;
    return (n >> 4) * 2048 + k * 128 + ((((nl >> 1) ^ (k & 7))) << 4) + ((nl & 1) << 3);
  } else {
    return n * 128 + ((((k >> 1) ^ (n & 7))) << 4) + ((k & 1) << 3);
  }
}
// physical row (within the CTA tile) of mma row g of m8 block mb
template <class Cfg>
PSD_DEVINL int a_row(int mb, int g) {
  if constexpr (Cfg::AL == A_MK) return mb * 8 + pi_row(g);
  else return (mb >> 1) * 16 + nu_col(g, mb & 1);
}
// physical column (within the CTA tile) of mma column c of n8 block nb
template <class Cfg>
PSD_DEVINL int b_col(int nb, int c) {
  if constexpr (Cfg::BL == B_KN) return (nb >> 1) * 16 + nu_col(c, nb & 1);
  else return nb * 8 + pi_row(c);
}

// Address of the kk-th k4 step from the kk = 0 address (stage base is
// 1 KiB aligned, so the swizzle XOR acts on bits the base does not use).
//   K-contiguous tile rows (A row-major, Bᵀ stored): chunk ^= 2·kk  → addr ^ (kk << 5)
//   M/N-contiguous tiles (Aᵀ stored, B row-major):  row += 4·kk, chunk ^= 4·(kk&1)
template <bool KContig>
PSD_DEVINL uint32_t frag_off(uint32_t addr0, int kk) {
  if constexpr (KContig) return addr0 ^ (uint32_t)(kk << 5);
  else return (addr0 + (uint32_t)(kk * 512)) ^ (uint32_t)((kk & 1) << 6);
}

struct Unit {
  int m0, n0, kbeg, nk, split;
};

// EPI_MIRROR with a row window: a lower tile contributes iff its rows or its
// (mirrored) columns intersect [win0, win1).
template <class Cfg>
PSD_DEVINL bool unit_active(const TmaParams& p, const Unit& u) {
  if (p.epi != EPI_MIRROR) return true;
  const bool rows = u.m0 < p.win1 && u.m0 + Cfg::BM > p.win0;
  const bool cols = u.n0 < p.win1 && u.n0 + Cfg::BN > p.win0;
  return rows || cols;
}

template <class Cfg>
PSD_DEVINL Unit decode_unit(const TmaParams& p, int u) {
  Unit r;
  int mt, nt;
  if (p.epi == EPI_MIRROR) {
    const long long x = u;
    int ti = (int)((sqrt(8.0 * (double)x + 1.0) - 1.0) * 0.5);
    while ((long long)(ti + 1) * (ti + 2) / 2 <= x) ++ti;
    while ((long long)ti * (ti + 1) / 2 > x) --ti;
    mt = ti;
    nt = (int)(x - (long long)ti * (ti + 1) / 2);
    r.split = 0;
  } else {
    mt = u % p.m_tiles;
    const int rest = u / p.m_tiles;
    nt = rest % p.n_tiles;
    r.split = rest / p.n_tiles;
  }
  r.m0 = mt * Cfg::BM;
  r.n0 = nt * Cfg::BN;
  r.kbeg = r.split * p.k_chunk;
  const int kend = min(p.K, r.kbeg + p.k_chunk);
  r.nk = kend > r.kbeg ? (kend - r.kbeg + Cfg::BK - 1) / Cfg::BK : 0;
  return r;
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kThreads, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const TmaParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[Cfg::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[Cfg::STAGES];
  // staged mirror epilogue handshake: named barrier 1 = tile parked in smem
  // (consumers arrive, store warps sync), 2 = tile stored (the reverse).
  // (An mbarrier arrive/wait pair here lost generic-proxy smem writes under
  // load — measured: ~10% of reconstructions had stale rows.)
  constexpr int kEpiBarCount = (Cfg::kConsumers + 3) * 32;
  constexpr int STAGES = Cfg::STAGES, M8W = Cfg::M8W, N8W = Cfg::N8W;
  constexpr int kStoreWarps = 3;
  const uint32_t smem_base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool staged = Cfg::STAGED_EPI && p.epi == EPI_MIRROR;
  double* Cs = reinterpret_cast<double*>(smem_raw + (smem_base - smem_u32(smem_raw)) +
                                         (size_t)STAGES * Cfg::STAGE_BYTES);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), Cfg::kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= Cfg::kConsumers) {
    // ------------------------------------------------------------- producer
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Cfg::kProducerRegs));
    if (warp == Cfg::kConsumers && lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      int it = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = decode_unit<Cfg>(p, u);
        if (!unit_active<Cfg>(p, un)) continue;
        for (int kt = 0; kt < un.nk; ++kt, ++it) {
          const int s = it % STAGES;
          const int use = it / STAGES;
          if (use > 0) mbar_wait(smem_u32(&empty_bar[s]), (use - 1) & 1);
          const uint32_t fb = smem_u32(&full_bar[s]);
          mbar_expect_tx(fb, Cfg::STAGE_BYTES);
          const uint32_t sa = smem_base + s * Cfg::STAGE_BYTES;
          const uint32_t sb = sa + Cfg::A_BYTES;
          const int k0 = un.kbeg + kt * Cfg::BK;
          if constexpr (Cfg::AL == A_MK) {
            tma_load_2d(sa, &mapA, k0, un.m0, fb);
          } else {
#pragma unroll
            for (int b = 0; b < Cfg::BM / 16; ++b) tma_load_2d(sa + b * 2048, &mapA, un.m0 + 16 * b, k0, fb);
          }
          if constexpr (Cfg::BL == B_NK) {
            tma_load_2d(sb, &mapB, k0, un.n0, fb);
          } else {
#pragma unroll
            for (int b = 0; b < Cfg::BN / 16; ++b) tma_load_2d(sb + b * 2048, &mapB, un.n0 + 16 * b, k0, fb);
          }
        }
      }
    } else if (staged && warp > Cfg::kConsumers) {
      // ------------------------------------------------------ store warps
      const int sw = warp - Cfg::kConsumers - 1;   // 0 .. kStoreWarps-1
      int j = 0;
      for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
        const Unit un = decode_unit<Cfg>(p, u);
        if (!unit_active<Cfg>(p, un)) continue;
        named_sync(1, kEpiBarCount);
        // (m, n) = (m0 + r, n0 + c), m ≥ n: C[m][n] (row m) and C[n][m] (row n)
        for (int r = sw; r < Cfg::BM; r += kStoreWarps) {
          const int m = un.m0 + r;
          if (m >= p.M || m < p.win0 || m >= p.win1) continue;
          double* crow = p.C + (long long)(m - p.win0) * p.ldc;
#pragma unroll
          for (int c = lane; c < Cfg::BN; c += 32) {
            const int n = un.n0 + c;
            if (n < p.N && n <= m) crow[n] = Cs[r * Cfg::C_LD + c];
          }
        }
        for (int c = sw; c < Cfg::BN; c += kStoreWarps) {
          const int n = un.n0 + c;
          if (n >= p.N || n < p.win0 || n >= p.win1) continue;
          double* crow = p.C + (long long)(n - p.win0) * p.ldc;
#pragma unroll
          for (int r = lane; r < Cfg::BM; r += 32) {
            const int m = un.m0 + r;
            if (m < p.M && m > n) crow[m] = Cs[r * Cfg::C_LD + c];
          }
        }
        __threadfence_block();   // the tile's reads are done before the consumers may overwrite it
        named_arrive(2, kEpiBarCount);
        ++j;
      }
    }
    return;
  }

  // ---------------------------------------------------------------- consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Cfg::kConsumerRegs));
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % Cfg::WARPS_M, wn = warp / Cfg::WARPS_M;
  // per-lane fragment byte offsets (stage relative) at kk = 0; the kk-th
  // k4 step is a constant add/xor away (see frag_off)
  uint32_t aoff[M8W], boff[N8W];
#pragma unroll
  for (int i = 0; i < M8W; ++i) aoff[i] = a_off<Cfg>(a_row<Cfg>(wm * M8W + i, g), t);
#pragma unroll
  for (int j = 0; j < N8W; ++j) boff[j] = Cfg::A_BYTES + b_off<Cfg>(t, b_col<Cfg>(wn * N8W + j, g));
  double resid = 0.0;
  int it = 0;
  int stage_j = 0;
  for (int u = blockIdx.x; u < p.units; u += gridDim.x) {
    const Unit un = decode_unit<Cfg>(p, u);
    if (!unit_active<Cfg>(p, un)) continue;
    double acc[M8W][N8W][2];
#pragma unroll
    for (int i = 0; i < M8W; ++i)
#pragma unroll
      for (int j = 0; j < N8W; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < un.nk; ++kt, ++it) {
      const int s = it % STAGES;
      mbar_wait(smem_u32(&full_bar[s]), (it / STAGES) & 1);
      const uint32_t st = smem_base + s * Cfg::STAGE_BYTES;
      double af[2][M8W], bf[N8W];
#pragma unroll
      for (int i = 0; i < M8W; ++i) af[0][i] = lds64(frag_off<Cfg::AL == A_MK>(st + aoff[i], 0));
#pragma unroll
      for (int j = 0; j < N8W; ++j) bf[j] = lds64(frag_off<Cfg::BL == B_NK>(st + boff[j], 0));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int cur = kk & 1;
        if (kk < 3) {
#pragma unroll
          for (int i = 0; i < M8W; ++i)
            af[cur ^ 1][i] = lds64(frag_off<Cfg::AL == A_MK>(st + aoff[i], kk + 1));
        }
#pragma unroll
        for (int j = 0; j < N8W; ++j) {
          const double b = bf[j];
          if (kk < 3) bf[j] = lds64(frag_off<Cfg::BL == B_NK>(st + boff[j], kk + 1));
#pragma unroll
          for (int i = 0; i < M8W; ++i) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i], b);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty_bar[s]));
    }

    // ------------------------------------------------------------- epilogue
    if (staged) {
      if (stage_j > 0) named_sync(2, kEpiBarCount);   // previous tile stored
#pragma unroll
      for (int i = 0; i < M8W; ++i) {
        const int r = a_row<Cfg>(wm * M8W + i, g);
#pragma unroll
        for (int j = 0; j < N8W; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) Cs[r * Cfg::C_LD + b_col<Cfg>(wn * N8W + j, 2 * t + e)] = acc[i][j][e];
      }
      // bar.arrive does not wait for this warp's shared-memory stores: make the parked tile
      // visible to the CTA before signalling the store warps (a rare stale-row race otherwise:
      // 2 of 2080 tiles of the C4-shape reconstruction)
      __threadfence_block();
      named_arrive(1, kEpiBarCount);
      ++stage_j;
      continue;
    }
    double* C = p.C + (long long)un.split * p.split_stride;
#pragma unroll
    for (int i = 0; i < M8W; ++i) {
      const int m = un.m0 + a_row<Cfg>(wm * M8W + i, g);
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < N8W; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = un.n0 + b_col<Cfg>(wn * N8W + j, 2 * t + e);
          if (n >= p.N) continue;
          const double v = acc[i][j][e];
          switch (p.epi) {
            case EPI_STORE: C[(long long)m * p.ldc + n] = v; break;
            case EPI_SHIFT:
              C[(long long)m * p.ldc + n] = (v + p.alpha * p.S[(long long)m * p.lds + n]) / p.alpha;
              break;
            case EPI_SUB: C[(long long)m * p.ldc + n] = p.S[(long long)m * p.lds + n] - v; break;
            case EPI_MIRROR:
              if (m >= n) {
                if (m >= p.win0 && m < p.win1) C[(long long)(m - p.win0) * p.ldc + n] = v;
                if (n >= p.win0 && n < p.win1) C[(long long)(n - p.win0) * p.ldc + m] = v;
              }
              break;
            case EPI_RESID: {
              const double d = p.S[(long long)m * p.lds + n] - v;
              resid = fma(d, d, resid);
            } break;
          }
        }
      }
    }
    if (p.epi == EPI_RESID) {
      const double r = warp_sum(resid);
      if (lane == 0) p.partials[(long long)u * Cfg::kConsumers + warp] = r;
      resid = 0.0;
    }
  }
  // consume the store warps' arrival for the last parked tile
  if (staged && stage_j > 0) named_sync(2, kEpiBarCount);
}

}  // namespace psd
