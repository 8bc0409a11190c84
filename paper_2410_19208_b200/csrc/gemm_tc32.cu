// 3xTF32 tcgen05 GEMM (see gemm_tc32.cuh) + the tf32 hi/lo split kernels and
// the split-K reduction that feeds FP64 panels.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "gemm_tc32.cuh"
#include "launch.h"

namespace psd {
namespace tc32 {

// ---- tcgen05 / TMEM wrappers ----------------------------------------------
template <int SW = SWZ>
PSD_DEVINL uint64_t smem_desc(uint32_t saddr) {
  // K-major swizzled canonical layout: 8-row atoms of SW-byte rows, SBO =
  // stride between atoms, LBO unused for swizzled K-major, version 1 (sm_100).
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((8 * SW) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(SW == 128 ? 2 : (SW == 64 ? 4 : 6)) << 61;
  return d;
}

// MN-major tf32 operand (A read M-contiguous): the 32-bit MN-major canonical
// layout SWIZZLE_128B_BASE32B (layout type 1; TMA CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B):
// 128-byte M rows, swizzled in 32-byte granules over 4-row (512 B) atoms;
// LBO = 4 KB between 32-element M chunks (one TMA box each), SBO = 512 B
// between 4-row K groups.  One tf32 MMA (K = 8) spans two groups: +1 KB per
// K step.  (Plain SWIZZLE_128B MN-major is not a valid tf32 operand layout:
// measured, the MMA returns zeros.)
PSD_DEVINL uint64_t smem_desc_mn(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)(4096 >> 4) << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__host__ __device__ inline uint32_t instr_desc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

PSD_DEVINL void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
PSD_DEVINL uint32_t tmem_cols_for(int n) {
  uint32_t c = 32;
  while ((int)c < n) c <<= 1;
  return c;
}

template <int SW>
__global__ void __launch_bounds__(kThreads, 1)
    tc32_gemm_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                     const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                     const Params p) {
  constexpr int BKk = SW / 4;   // K elements per k-block for this swizzle
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], acc_bar;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bn_tot = p.bn * p.n_mma;
  int u = blockIdx.x;
  const int ng = u % p.n_groups;
  u /= p.n_groups;
  const int split = u % p.splits;
  const int mt = u / p.splits;
  const int m0 = mt * BM, n0 = ng * bn_tot;
  // MIRROR keeps only tiles holding some (i, j) with i ≥ j
  if (p.mode == MIRROR && m0 + BM - 1 < n0) return;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;

  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = BM * SW, b_bytes = (uint32_t)bn_tot * SW;
  const uint32_t st_bytes = 2 * a_bytes + 2 * b_bytes;
  const uint32_t tcols = tmem_cols_for(bn_tot);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&acc_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh);
    tma_prefetch_desc(&mAl);
    tma_prefetch_desc(&mBh);
    tma_prefetch_desc(&mBl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        mbar_wait_t(smem_u32(&empty_bar[s]), ph ^ 1u);
        const uint32_t fb = smem_u32(&full_bar[s]);
        mbar_expect_tx(fb, st_bytes);
        const uint32_t sA = sbase + s * st_bytes;
        const uint32_t sB = sA + 2 * a_bytes;
        const int kc = (kb0 + i) * BKk;
        tma_load_2d(sA, &mAh, kc, m0, fb);
        tma_load_2d(sA + a_bytes, &mAl, kc, m0, fb);
        for (int h = 0; h < p.n_mma; ++h) {
          const uint32_t off = (uint32_t)h * p.bn * SW;
          tma_load_2d(sB + off, &mBh, kc, n0 + h * p.bn, fb);
          tma_load_2d(sB + b_bytes + off, &mBl, kc, n0 + h * p.bn, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = instr_desc(p.bn);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        mbar_wait_t(smem_u32(&full_bar[s]), ph);
        tc_fence_after();
        const uint32_t sA = sbase + s * st_bytes;
        const uint32_t sB = sA + 2 * a_bytes;
#pragma unroll
        for (int kk = 0; kk < BKk / 8; ++kk) {
          const uint64_t ah = smem_desc<SW>(sA + kk * 32), al = smem_desc<SW>(sA + a_bytes + kk * 32);
          for (int h = 0; h < p.n_mma; ++h) {
            const uint32_t off = (uint32_t)h * p.bn * SW + kk * 32;
            const uint64_t bh = smem_desc<SW>(sB + off), bl = smem_desc<SW>(sB + b_bytes + off);
            const uint32_t d = tmem + (uint32_t)(h * p.bn);
            mma_tf32(d, al, bh, idesc, (i | kk) != 0);   // small terms first
            mma_tf32(d, ah, bl, idesc, 1u);
            mma_tf32(d, ah, bh, idesc, 1u);
          }
        }
        mma_commit(smem_u32(&empty_bar[s]));   // slot free once these MMAs retire
      }
      mma_commit(smem_u32(&acc_bar));          // accumulator complete
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32·(w mod 4) …
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int i = m0 + r;
    mbar_wait_t(smem_u32(&acc_bar), 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    if (p.mode == PARTIAL) {
      for (int c0 = 0; c0 < bn_tot; c0 += 16) {
        float v[16];
        tmem_ld16(trow + (uint32_t)c0, v);
        if (i >= p.M) continue;
        float4* dst = reinterpret_cast<float4*>(p.out + (long long)split * p.split_stride +
                                                (long long)i * p.ldo + n0 + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    } else {
      // MIRROR: 32×32 blocks; C[j][i] straight from registers (lanes = consecutive i),
      // C[i][j] through a per-warp smem transpose so each store is one 128-B row.
      float* tile = reinterpret_cast<float*>(smem_raw + (sbase - sraw) + p.stages * st_bytes) +
                    (warp - 2) * 32 * 33;
      const int ib = m0 + quad * 32;
      for (int c0 = 0; c0 < bn_tot; c0 += 32) {
        const int j0 = n0 + c0;
        if (j0 >= p.N || j0 > ib + 31) break;          // block entirely above the diagonal / outside
        float v[32];
        tmem_ld16(trow + (uint32_t)c0, *reinterpret_cast<float(*)[16]>(&v[0]));
        tmem_ld16(trow + (uint32_t)c0 + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int j = j0 + e;
          if (i < p.M && j <= i && j < p.N) p.out[(long long)j * p.ldo + i] = v[e];
          tile[lane * 33 + e] = v[e];
        }
        __syncwarp();
        const int j = j0 + lane;
        for (int rr = 0; rr < 32; ++rr) {
          const int ii = ib + rr;
          if (ii < p.M && j <= ii && j < p.N) p.out[(long long)ii * p.ldo + j] = tile[rr * 33 + lane];
        }
        __syncwarp();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols)
                 : "memory");
  }
}

// ---- persistent mirrored reconstruction ----------------------------------
// C = sym(A·Bᵀ) written from the lower 128×256 tiles only (each element to
// (i,j) and (j,i)).  One CTA per SM walks the lower tiles; the TMEM holds two
// 256-column accumulators so the epilogue of tile t (4 warps, TMEM → 2×
// coalesced stores) overlaps the MMAs of tile t+1, and the producer streams
// operands across tile boundaries.
PSD_DEVINL void lower_tile(int t, int m_tiles, int& mt, int& nt) {
  // tiles of block-column nt: mt ∈ [2·nt, m_tiles)
  nt = 0;
  while (true) {
    const int cnt = m_tiles - 2 * nt;
    if (t < cnt) break;
    t -= cnt;
    ++nt;
  }
  mt = 2 * nt + t;
}

constexpr int kMirrorEpi = 16;                      // epilogue warps (4 per TMEM lane quadrant)
constexpr int kMirrorThreads = (2 + kMirrorEpi) * 32;
template <int SW>
__global__ void __launch_bounds__(kMirrorThreads, 1)
    tc32_mirror_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                       const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                       const Params p, int ntiles) {
  constexpr int BKk = SW / 4;
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], accf_bar[2], acce_bar[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = BM * SW, b_bytes = (uint32_t)BN * SW;
  const uint32_t st_bytes = 2 * a_bytes + 2 * b_bytes;
  const int nkb = p.kblocks;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&accf_bar[b]), 1);
      mbar_init(smem_u32(&acce_bar[b]), kMirrorEpi);   // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh);
    tma_prefetch_desc(&mAl);
    tma_prefetch_desc(&mBh);
    tma_prefetch_desc(&mBl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int it = 0;   // global k-block counter across tiles
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int mt, nt;
        lower_tile(t, p.m_tiles, mt, nt);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % p.stages;
          const uint32_t ph = (uint32_t)(it / p.stages) & 1u;
          mbar_wait_t(smem_u32(&empty_bar[s]), ph ^ 1u);
          const uint32_t fb = smem_u32(&full_bar[s]);
          mbar_expect_tx(fb, st_bytes);
          const uint32_t sA = sbase + s * st_bytes;
          const uint32_t sB = sA + 2 * a_bytes;
          const int kc = kb * BKk;
          tma_load_2d(sA, &mAh, kc, mt * BM, fb);
          tma_load_2d(sA + a_bytes, &mAl, kc, mt * BM, fb);
          tma_load_2d(sB, &mBh, kc, nt * BN, fb);
          tma_load_2d(sB + b_bytes, &mBl, kc, nt * BN, fb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      int it = 0, j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int b = j & 1;
        // wait until the epilogue drained this accumulator (its previous use: tile j−2)
        mbar_wait_t(smem_u32(&acce_bar[b]), (((uint32_t)j >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(b * BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % p.stages;
          const uint32_t ph = (uint32_t)(it / p.stages) & 1u;
          mbar_wait_t(smem_u32(&full_bar[s]), ph);
          tc_fence_after();
          const uint32_t sA = sbase + s * st_bytes;
          const uint32_t sB = sA + 2 * a_bytes;
#pragma unroll
          for (int kk = 0; kk < BKk / 8; ++kk) {
            const uint64_t ah = smem_desc<SW>(sA + kk * 32), al = smem_desc<SW>(sA + a_bytes + kk * 32);
            const uint64_t bh = smem_desc<SW>(sB + kk * 32), bl = smem_desc<SW>(sB + b_bytes + kk * 32);
            mma_tf32(d, al, bh, idesc, (kb | kk) != 0);
            mma_tf32(d, ah, bl, idesc, 1u);
            mma_tf32(d, ah, bh, idesc, 1u);
          }
          mma_commit(smem_u32(&empty_bar[s]));
        }
        mma_commit(smem_u32(&accf_bar[b]));
      }
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;            // column slice of the tile this warp stores
    constexpr int kSlice = BN / (kMirrorEpi / 4);
    float* tile = reinterpret_cast<float*>(smem_raw + (sbase - sraw) + p.stages * st_bytes) +
                  (warp - 2) * 32 * 33;
    const uint32_t tq = (uint32_t)(quad * 32) << 16;
    int j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      int mt, nt;
      lower_tile(t, p.m_tiles, mt, nt);
      const int b = j & 1;
      mbar_wait_t(smem_u32(&accf_bar[b]), ((uint32_t)j >> 1) & 1u);
      tc_fence_after();
      const int ib = mt * BM + quad * 32;
      const int i = ib + lane;
      const int n0 = nt * BN;
      for (int c0 = half * kSlice; c0 < (half + 1) * kSlice; c0 += 32) {
        const int j0 = n0 + c0;
        if (j0 >= p.N || j0 > ib + 31) break;          // block above the diagonal / outside
        float v[32];
        tmem_ld16(tmem + tq + (uint32_t)(b * BN + c0), *reinterpret_cast<float(*)[16]>(&v[0]));
        tmem_ld16(tmem + tq + (uint32_t)(b * BN + c0 + 16), *reinterpret_cast<float(*)[16]>(&v[16]));
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int jj = j0 + e;
          if (i < p.M && jj <= i && jj < p.N) p.out[(long long)jj * p.ldo + i] = v[e];
          tile[lane * 33 + e] = v[e];
        }
        __syncwarp();
        const int jj = j0 + lane;
        for (int rr = 0; rr < 32; ++rr) {
          const int ii = ib + rr;
          if (ii < p.M && jj <= ii && jj < p.N) p.out[(long long)ii * p.ldo + jj] = tile[rr * 33 + lane];
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&acce_bar[b]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---- CTA-pair variant (cta_group::2) for the PARTIAL (panel) mode ----------
// A pair of CTAs on one TPC computes a 256 × n_tot tile: each CTA streams its
// own 128 rows of A and HALF of every B box (bn/2 rows), the leader issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' shared memory, and
// each CTA's TMEM receives its 128 rows.  Per SM this halves the B bytes
// streamed and read per MMA.
PSD_DEVINL void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
PSD_DEVINL void mma_tf32_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}

// AMN: A is read M-contiguous ("MN-major"): A = Sᵀ for a row-major S, so every
// TMA box row is 128 contiguous bytes of S and the four M-chunks of a stage
// give 512-byte runs per row of S (DRAM-friendly); used with symmetric X.
template <bool AMN>
__global__ void __launch_bounds__(kThreads, 1)
    tc32_gemm2_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                      const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                      const __grid_constant__ CUtensorMap mBh2, const __grid_constant__ CUtensorMap mBl2,
                      const Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], acc_bar;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool two = p.n_mma > 1;
  const int bn_tot = p.bn + (two ? p.bn2 : 0);   // e.g. 272 = 144 + 128: no padded columns
  const int hb = p.bn / 2, hb2 = p.bn2 / 2;      // B rows per CTA for the first / second MMA
  int u = blockIdx.x >> 1;
  const int ng = u % p.n_groups;
  u /= p.n_groups;
  const int split = u % p.splits;
  const int mp = u / p.splits;
  const int m0 = mp * 2 * BM + (int)rank * BM, n0 = ng * bn_tot;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;

  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = BM * SWZ, b_bytes = (uint32_t)(hb + (two ? hb2 : 0)) * SWZ;
  const uint32_t st_bytes = 2 * a_bytes + 2 * b_bytes;
  const uint32_t tcols = tmem_cols_for(bn_tot);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&acc_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    tma_prefetch_desc(&mAh);
    tma_prefetch_desc(&mAl);
    tma_prefetch_desc(&mBh);
    tma_prefetch_desc(&mBl);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  // Producer and MMA warps run their loops warp-uniformly and elect one lane
  // to issue: the descriptors then live in uniform registers (no per-MMA
  // R2UR round trips on the single issuing thread).
  if (warp == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
      mbar_wait_t(smem_u32(&empty_bar[s]), ph ^ 1u);
      if (elect_one()) {
        const uint32_t fb_local = smem_u32(&full_bar[s]);
        const uint32_t fb = map_to_rank(fb_local, 0);          // the leader's barrier
        if (rank == 0) mbar_expect_tx(fb_local, 2 * st_bytes);  // both CTAs' bytes
        const uint32_t sA = sbase + s * st_bytes;
        const uint32_t sB = sA + 2 * a_bytes;
        const int kc = (kb0 + i) * BK;
        if constexpr (AMN) {
          // box = 32 M × BK K-rows (4 KB); M-chunk c at +4 KB
#pragma unroll
          for (int c = 0; c < BM / 32; ++c) {
            tma_load_2d_pair(sA + c * 4096, &mAh, m0 + 32 * c, kc, fb);
            tma_load_2d_pair(sA + a_bytes + c * 4096, &mAl, m0 + 32 * c, kc, fb);
          }
        } else {
          tma_load_2d_pair(sA, &mAh, kc, m0, fb);
          tma_load_2d_pair(sA + a_bytes, &mAl, kc, m0, fb);
        }
        {
          const int nrow = n0 + (int)rank * hb;
          tma_load_2d_pair(sB, &mBh, kc, nrow, fb);
          tma_load_2d_pair(sB + b_bytes, &mBl, kc, nrow, fb);
        }
        if (two) {
          const uint32_t off = (uint32_t)hb * SWZ;
          const int nrow = n0 + p.bn + (int)rank * hb2;
          tma_load_2d_pair(sB + off, &mBh2, kc, nrow, fb);
          tma_load_2d_pair(sB + b_bytes + off, &mBl2, kc, nrow, fb);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((AMN ? 1u : 0u) << 15) |
                             ((uint32_t)(p.bn >> 3) << 17) | ((uint32_t)(2 * BM >> 4) << 24);
      // stage-0 descriptors; stage s / step kk / half h only move the 14-bit start-address field
      const uint64_t dah = AMN ? smem_desc_mn(sbase) : smem_desc(sbase);
      const uint64_t dal = AMN ? smem_desc_mn(sbase + a_bytes) : smem_desc(sbase + a_bytes);
      const uint64_t dbh = smem_desc(sbase + 2 * a_bytes);
      const uint64_t dbl = smem_desc(sbase + 2 * a_bytes + b_bytes);
      constexpr uint32_t a_kstep = (AMN ? 1024u : 32u) >> 4, b_kstep = 32u >> 4;
      const uint32_t b_half = (uint32_t)(hb * SWZ) >> 4;
      const uint32_t idesc2 = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(p.bn2 >> 3) << 17);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        mbar_wait_t(smem_u32(&full_bar[s]), ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t so = (uint32_t)(s * st_bytes) >> 4;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ah = dah + so + kk * a_kstep, al = dal + so + kk * a_kstep;
            const uint64_t bh0 = dbh + so + kk * b_kstep, bl0 = dbl + so + kk * b_kstep;
            const uint32_t acc0 = (i | kk) != 0;
            mma_tf32_pair(tmem, al, bh0, idesc, acc0);
            mma_tf32_pair(tmem, ah, bl0, idesc, 1u);
            mma_tf32_pair(tmem, ah, bh0, idesc, 1u);
            if (two) {
              const uint32_t d1 = tmem + (uint32_t)p.bn;
              mma_tf32_pair(d1, al, bh0 + b_half, idesc2, acc0);
              mma_tf32_pair(d1, ah, bl0 + b_half, idesc2, 1u);
              mma_tf32_pair(d1, ah, bh0 + b_half, idesc2, 1u);
            }
          }
          mma_commit_pair(smem_u32(&empty_bar[s]));   // frees slot s in both CTAs
          if (i == nkb - 1) mma_commit_pair(smem_u32(&acc_bar));   // accumulators complete
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int i = m0 + quad * 32 + lane;
    mbar_wait_t(smem_u32(&acc_bar), 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    for (int c0 = 0; c0 < bn_tot; c0 += 16) {
      float v[16];
      tmem_ld16(trow + (uint32_t)c0, v);
      if (i >= p.M) continue;
      float4* dst = reinterpret_cast<float4*>(p.out + (long long)split * p.split_stride +
                                              (long long)i * p.ldo + n0 + c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols)
                 : "memory");
  }
}

// ---- CTA-pair variant with A staged in TMEM (tcgen05.cp + MMA "TS") -------
// Experiment (opt-in, PSD_TC32_TS=1): in the SS kernel A is read from shared
// memory by 6 MMAs per K step.  Here each stage's A hi/lo (128 rows × 32 K per CTA)
// is copied once into TMEM with tcgen05.cp and every MMA takes A from TMEM;
// shared memory only feeds B.  The N range is split 256 + n1 (n1 a multiple
// of 32: TS MMAs need N % 32 == 0), e.g. w = 272 → 256 + 32.
PSD_DEVINL void tmem_cp_pair(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::2.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc) : "memory");
}
PSD_DEVINL void mma_tf32_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                 uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum));
}

struct Ts2Maps {
  CUtensorMap ah, al, bh0, bl0, bh1, bl1;
};

__global__ void __launch_bounds__(kThreads, 1)
    tc32_gemm2ts_kernel(const __grid_constant__ Ts2Maps mp, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], acc_bar;
  __shared__ uint32_t tmem_slot;
  constexpr int kAcol = 320;                     // TMEM column of the two A buffers (64 cols each)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int bn1 = p.bn;                          // second N piece (first is 256)
  const int hb0 = 128, hb1 = bn1 / 2;            // B rows per CTA per piece
  const int bn_tot = 256 + bn1;
  int u = blockIdx.x >> 1;
  const int ng = u % p.n_groups;
  u /= p.n_groups;
  const int split = u % p.splits;
  const int mpair = u / p.splits;
  const int m0 = mpair * 2 * BM + (int)rank * BM, n0 = ng * bn_tot;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;

  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = BM * SWZ, b_bytes = (uint32_t)(hb0 + hb1) * SWZ;
  const uint32_t st_bytes = 2 * a_bytes + 2 * b_bytes;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    mbar_init(smem_u32(&acc_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
      mbar_wait_t(smem_u32(&empty_bar[s]), ph ^ 1u);
      if (elect_one()) {
        const uint32_t fb_local = smem_u32(&full_bar[s]);
        const uint32_t fb = map_to_rank(fb_local, 0);
        if (rank == 0) mbar_expect_tx(fb_local, 2 * st_bytes);
        const uint32_t sA = sbase + s * st_bytes;
        const uint32_t sB = sA + 2 * a_bytes;
        const int kc = (kb0 + i) * BK;
        tma_load_2d_pair(sA, &mp.ah, kc, m0, fb);
        tma_load_2d_pair(sA + a_bytes, &mp.al, kc, m0, fb);
        tma_load_2d_pair(sB, &mp.bh0, kc, n0 + (int)rank * hb0, fb);
        tma_load_2d_pair(sB + hb0 * SWZ, &mp.bh1, kc, n0 + 256 + (int)rank * hb1, fb);
        tma_load_2d_pair(sB + b_bytes, &mp.bl0, kc, n0 + (int)rank * hb0, fb);
        tma_load_2d_pair(sB + b_bytes + hb0 * SWZ, &mp.bl1, kc, n0 + 256 + (int)rank * hb1, fb);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (rank == 0) {
      const uint32_t id0 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                           ((uint32_t)(2 * BM >> 4) << 24);
      const uint32_t id1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bn1 >> 3) << 17) |
                           ((uint32_t)(2 * BM >> 4) << 24);
      const uint64_t dah = smem_desc(sbase), dal = smem_desc(sbase + a_bytes);
      const uint64_t dbh = smem_desc(sbase + 2 * a_bytes), dbl = smem_desc(sbase + 2 * a_bytes + b_bytes);
      const uint32_t b1off = (uint32_t)(hb0 * SWZ) >> 4;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        mbar_wait_t(smem_u32(&full_bar[s]), ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t so = (uint32_t)(s * st_bytes) >> 4;
          const uint32_t abuf = tmem + (uint32_t)(kAcol + (i & 1) * 64);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {   // A hi → cols [0,32), A lo → [32,64) of the buffer
            tmem_cp_pair(abuf + kk * 8, dah + so + kk * 2);
            tmem_cp_pair(abuf + 32 + kk * 8, dal + so + kk * 2);
          }
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t ah = abuf + kk * 8, al = abuf + 32 + kk * 8;
            const uint64_t bh = dbh + so + kk * 2, bl = dbl + so + kk * 2;
            const uint32_t acc0 = (i | kk) != 0;
            mma_tf32_pair_ts(tmem, al, bh, id0, acc0);
            mma_tf32_pair_ts(tmem, ah, bl, id0, 1u);
            mma_tf32_pair_ts(tmem, ah, bh, id0, 1u);
            const uint32_t d1 = tmem + 256u;
            mma_tf32_pair_ts(d1, al, bh + b1off, id1, acc0);
            mma_tf32_pair_ts(d1, ah, bl + b1off, id1, 1u);
            mma_tf32_pair_ts(d1, ah, bh + b1off, id1, 1u);
          }
          mma_commit_pair(smem_u32(&empty_bar[s]));
          if (i == nkb - 1) mma_commit_pair(smem_u32(&acc_bar));
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int i = m0 + quad * 32 + lane;
    mbar_wait_t(smem_u32(&acc_bar), 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    for (int c0 = 0; c0 < bn_tot; c0 += 16) {
      float v[16];
      tmem_ld16(trow + (uint32_t)c0, v);
      if (i >= p.M) continue;
      float4* dst = reinterpret_cast<float4*>(p.out + (long long)split * p.split_stride +
                                              (long long)i * p.ldo + n0 + c0);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512) : "memory");
  }
}

// ---- split / convert kernels ----------------------------------------------
PSD_DEVINL float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r & 0xFFFFE000u);
}
// raw mode: hi = x itself — kind::tf32 ignores the low 13 mantissa bits, i.e.
// reads trunc(x) (verified on B200: tools/probe_rawhi.py) — and lo = x − trunc(x),
// exact in fp32; the hi array then never has to be written.
PSD_DEVINL void split_f32(float x, bool raw, float& hi, float& lo) {
  if (raw) {
    hi = x;
    lo = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  } else {
    hi = tf32_rna(x);
    lo = tf32_rna(x - hi);
  }
}
PSD_DEVINL void split2(double x, float& hi, float& lo) {
  hi = tf32_rna((float)x);
  lo = tf32_rna((float)(x - (double)hi));
}

// hi/lo (rows × cols_pad, ld ldh) of a row-major fp32 matrix; columns ≥ cols zero.
__global__ void split_rows_f32_kernel(const float* __restrict__ x, long long rows, long long cols,
                                      long long ldx, float* __restrict__ hi, float* __restrict__ lo,
                                      long long ldh, long long cols_pad, bool raw) {
  const long long total = rows * cols_pad;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols_pad, c = e % cols_pad;
    const float v = c < cols ? x[r * ldx + c] : 0.f;
    float h, l;
    split_f32(v, raw, h, l);
    if (!raw) hi[r * ldh + c] = h;
    lo[r * ldh + c] = l;
  }
}
// vectorised variant: cols % 4 == 0 == ldx % 4 == ldh % 4, 16-B aligned
__global__ void split_rows_f32x4_kernel(const float4* __restrict__ x, long long rows, long long cols4,
                                        long long ldx4, float4* __restrict__ hi,
                                        float4* __restrict__ lo, long long ldh4, bool raw) {
  const long long total = rows * cols4;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols4, c = e % cols4;
    const float4 v = x[r * ldx4 + c];
    float4 h, l;
    split_f32(v.x, raw, h.x, l.x);
    split_f32(v.y, raw, h.y, l.y);
    split_f32(v.z, raw, h.z, l.z);
    split_f32(v.w, raw, h.w, l.w);
    if (!raw) hi[r * ldh4 + c] = h;
    lo[r * ldh4 + c] = l;
  }
}

// hi/lo of (x · diag(scale)) for a row-major fp64 rows × cols matrix, padded to cols_pad.
__global__ void split_rows_f64_kernel(const double* __restrict__ x, long long rows, int cols,
                                      long long ldx, const double* __restrict__ scale,
                                      float* __restrict__ hi, float* __restrict__ lo, long long ldh,
                                      int cols_pad) {
  const long long total = rows * cols_pad;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols_pad;
    const int c = (int)(e % cols_pad);
    double v = 0.0;
    if (c < cols) v = x[r * ldx + c] * (scale ? scale[c] : 1.0);
    float h, l;
    split2(v, h, l);
    hi[r * ldh + c] = h;
    lo[r * ldh + c] = l;
  }
}

// Transposed split of an n × w fp64 panel: out[j][i] (j < w_rows; zero rows j ≥ w).
__global__ void split_transpose_kernel(const double* __restrict__ P, long long n, int w, long long ldp,
                                       float* __restrict__ hi, float* __restrict__ lo, long long ldt,
                                       int w_rows) {
  __shared__ double tile[32][33];
  const long long i0 = (long long)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 × 8
  for (int yy = ty; yy < 32; yy += 8) {
    const long long i = i0 + yy;
    const int j = j0 + tx;
    tile[yy][tx] = (i < n && j < w) ? P[i * ldp + j] : 0.0;
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int j = j0 + yy;
    const long long i = i0 + tx;
    if (j < w_rows && i < n) {
      float h, l;
      split2(tile[tx][yy], h, l);
      hi[(long long)j * ldt + i] = h;
      lo[(long long)j * ldt + i] = l;
    }
  }
}

// require_symmetric statistics (symmetric.py:39-57) fused with the tf32 hi/lo
// split of a square fp32 X: one 64×64 tile pair (I ≥ J) per iteration, tile
// (J, I) staged through shared memory, so X is read from HBM exactly once.
// stats[0] = max|x|, stats[1] = max|x − xᵀ|, ((int*)(stats+2))[0] bit0: not
// bitwise symmetric, bit1: non-finite entry.
constexpr int kSST = 64;
__global__ void __launch_bounds__(256, 4) symsplit_kernel(const float* __restrict__ x, long long n,
                                                       long long ldx, long long npairs,
                                                       double* stats, float* __restrict__ hi,
                                                       float* __restrict__ lo, long long ldh, bool raw) {
  __shared__ float tb[kSST][kSST + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float mabs = 0.f;
  double mdef = 0.0;
  int flags = 0;
  for (long long b = blockIdx.x; b < npairs; b += gridDim.x) {
    long long ti = (long long)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= b) ++ti;
    while (ti * (ti + 1) / 2 > b) --ti;
    const long long tj = b - ti * (ti + 1) / 2;
    const long long r0 = ti * kSST, c0 = tj * kSST;
    float a[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        const long long ar = r0 + r, ac = c0 + c;   // tile (I, J) → registers
        a[q][h] = (ar < n && ac < n) ? __ldcs(x + ar * ldx + ac) : 0.f;
        const long long br = c0 + r, bc = r0 + c;   // tile (J, I) → smem, as stored
        tb[r][c] = (br < n && bc < n) ? __ldcs(x + br * ldx + bc) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        const float av = a[q][h], bt = tb[c][r];    // x[i][j] and x[j][i]
        if (!isfinite(av) || !isfinite(bt)) flags |= 2;
        mabs = fmaxf(mabs, fmaxf(fabsf(av), fabsf(bt)));
        mdef = fmax(mdef, fabs((double)av - (double)bt));   // exact, as after the f64 cast
        if (av != bt) flags |= 1;
        const long long ar = r0 + r, ac = c0 + c;
        if (ar < n && ac < n) {
          float h1, l1;
          split_f32(av, raw, h1, l1);
          if (!raw) __stcs(hi + ar * ldh + ac, h1);
          __stcs(lo + ar * ldh + ac, l1);
        }
        const long long br = c0 + r, bc = r0 + c;
        if (ti != tj && br < n && bc < n) {
          float h2, l2;
          split_f32(tb[r][c], raw, h2, l2);
          if (!raw) __stcs(hi + br * ldh + bc, h2);
          __stcs(lo + br * ldh + bc, l2);
        }
      }
    }
    __syncthreads();
  }
  __shared__ float rmax[8];
  __shared__ double rdef[8];
  __shared__ int rfl[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mabs = fmaxf(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
    mdef = fmax(mdef, __shfl_xor_sync(0xffffffffu, mdef, o));
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (tx == 0) {
    rmax[ty] = mabs;
    rdef[ty] = mdef;
    rfl[ty] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m1 = 0.f;
    double m2 = 0.0;
    int f = 0;
    for (int w = 0; w < 8; ++w) {
      m1 = fmaxf(m1, rmax[w]);
      m2 = fmax(m2, rdef[w]);
      f |= rfl[w];
    }
    if (m1 > 0.f) atomic_max_nonneg(&stats[0], (double)m1);
    if (m2 > 0.0) atomic_max_nonneg(&stats[1], m2);
    if (f) atomicOr(reinterpret_cast<int*>(stats + 2), f);
  }
}

// 128-bit variant of symsplit_kernel (raw mode: only lo is written) for
// n, ldx, ldh multiples of 4 and 16-byte aligned arrays: 4 float4 loads and
// 4 float4 stores per thread per tile instead of 16 scalar ones.
__global__ void __launch_bounds__(256, 4) symsplit4_kernel(const float* __restrict__ x, long long n,
                                                           long long ldx, long long npairs,
                                                           double* stats, float* __restrict__ lo,
                                                           long long ldh) {
  __shared__ float tb[kSST][kSST + 1];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float mabs = 0.f;
  double mdef = 0.0;
  int flags = 0;
  for (long long b = blockIdx.x; b < npairs; b += gridDim.x) {
    long long ti = (long long)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= b) ++ti;
    while (ti * (ti + 1) / 2 > b) --ti;
    const long long tj = b - ti * (ti + 1) / 2;
    const long long r0 = ti * kSST, c0 = tj * kSST;
    float4 a[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int f = tid + 256 * q, row = f >> 4, col = (f & 15) * 4;
      const long long ar = r0 + row, ac = c0 + col;          // tile (I, J) → registers
      a[q] = (ar < n && ac < n) ? __ldcs(reinterpret_cast<const float4*>(x + ar * ldx + ac))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      const long long br = c0 + row, bc = r0 + col;          // tile (J, I) → smem, as stored
      const float4 v = (br < n && bc < n) ? __ldcs(reinterpret_cast<const float4*>(x + br * ldx + bc))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
      tb[row][col] = v.x;
      tb[row][col + 1] = v.y;
      tb[row][col + 2] = v.z;
      tb[row][col + 3] = v.w;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int f = tid + 256 * q, row = f >> 4, col = (f & 15) * 4;
      const float av[4] = {a[q].x, a[q].y, a[q].z, a[q].w};
      float lo4[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float bt = tb[col + e][row];                   // x[j][i]
        if (!isfinite(av[e]) || !isfinite(bt)) flags |= 2;
        mabs = fmaxf(mabs, fmaxf(fabsf(av[e]), fabsf(bt)));
        mdef = fmax(mdef, fabs((double)av[e] - (double)bt));
        if (av[e] != bt) flags |= 1;
        lo4[e] = av[e] - __uint_as_float(__float_as_uint(av[e]) & 0xFFFFE000u);
      }
      const long long ar = r0 + row, ac = c0 + col;
      if (ar < n && ac < n)
        __stcs(reinterpret_cast<float4*>(lo + ar * ldh + ac), make_float4(lo4[0], lo4[1], lo4[2], lo4[3]));
      const long long br = c0 + row, bc = r0 + col;
      if (ti != tj && br < n && bc < n) {
        float l2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float bv = tb[row][col + e];
          l2[e] = bv - __uint_as_float(__float_as_uint(bv) & 0xFFFFE000u);
        }
        __stcs(reinterpret_cast<float4*>(lo + br * ldh + bc), make_float4(l2[0], l2[1], l2[2], l2[3]));
      }
    }
    __syncthreads();
  }
  __shared__ float rmax[8];
  __shared__ double rdef[8];
  __shared__ int rfl[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mabs = fmaxf(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
    mdef = fmax(mdef, __shfl_xor_sync(0xffffffffu, mdef, o));
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0) {
    rmax[wid] = mabs;
    rdef[wid] = mdef;
    rfl[wid] = flags;
  }
  __syncthreads();
  if (tid == 0) {
    float m1 = 0.f;
    double m2 = 0.0;
    int f = 0;
    for (int w = 0; w < 8; ++w) {
      m1 = fmaxf(m1, rmax[w]);
      m2 = fmax(m2, rdef[w]);
      f |= rfl[w];
    }
    if (m1 > 0.f) atomic_max_nonneg(&stats[0], (double)m1);
    if (m2 > 0.0) atomic_max_nonneg(&stats[1], m2);
    if (f) atomicOr(reinterpret_cast<int*>(stats + 2), f);
  }
}

// C (fp64, M × N) = (Σ_s ws[s] + α·S)/α  (α > 0)  or  Σ_s ws[s].
__global__ void reduce_partials_kernel(const float* __restrict__ ws, int splits, long long stride,
                                       long long ldw, int M, int N, double* __restrict__ C,
                                       long long ldc, double alpha, const double* __restrict__ S,
                                       long long lds) {
  const long long total = (long long)M * N;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / N;
    const int j = (int)(e % N);
    double acc = 0.0;
    for (int s = 0; s < splits; ++s) acc += (double)ws[s * stride + i * ldw + j];
    if (alpha > 0.0) acc = (acc + alpha * S[i * lds + j]) / alpha;
    C[i * ldc + j] = acc;
  }
}

}  // namespace tc32

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode32() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool map_f32(CUtensorMap* map, const float* ptr, long long cols, long long rows, long long ld,
             int box_rows, int swz = tc32::SWZ) {
  auto fn = encode32();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)(swz / 4), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D fp32 map for the MN-major operand: box = 32 elements (128 B) × box_rows, 32-byte-atom 128B swizzle
bool map_f32_box(CUtensorMap* map, const float* ptr, long long cols, long long rows, long long ld,
                 int box_cols, int box_rows) {
  auto fn = encode32();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int grid_for(long long total, int threads) {
  const long long b = (total + threads - 1) / threads;
  return (int)std::min<long long>(std::max<long long>(b, 1), (long long)device_info().sms * 16);
}

}  // namespace

long long tc32_ws_elems(long long M, int N, int max_splits) {
  const int bn_tot = (std::min(N, tc32::kMaxN) + 15) / 16 * 16;
  const int groups = (N + bn_tot - 1) / bn_tot;
  return (long long)max_splits * M * groups * bn_tot;
}

int gemm_tf32x3(const Tc32Op& op, cudaStream_t st) {
  using namespace tc32;
  if (op.M < 1 || op.N < 1 || op.K < 1) return 0;
  if ((op.lda % 4) || (op.ldb % 4) || (op.lda_lo % 4) || ((uintptr_t)op.a_hi % 16) || ((uintptr_t)op.a_lo % 16) ||
      ((uintptr_t)op.b_hi % 16) || ((uintptr_t)op.b_lo % 16))
    return -2;
  Params p{};
  p.M = op.M;
  p.N = op.N;
  p.K = op.K;
  // N tiling: one group of up to 512 TMEM columns, as ≤ 2 MMAs of ≤ 256
  int n_tot;
  if (op.mode == MIRROR) {
    n_tot = 256;
  } else {
    const int groups = (op.N + kMaxN - 1) / kMaxN;
    n_tot = ((op.N + groups - 1) / groups + 15) / 16 * 16;
  }
  // A staged in TMEM (TS MMAs, N pieces 256 + n1 with n1 % 32 == 0): correct but measured
  // slower than the SS pair kernel at C3 (2.73 vs 2.50 ms) — opt-in via PSD_TC32_TS=1
  static const bool ts_ok = [] {
    const char* e = getenv("PSD_TC32_TS");
    return e && e[0] == '1';
  }();
  const bool ts = op.mode == PARTIAL && ts_ok && !op.a_mn && n_tot > 256 && n_tot <= 512 &&
                  !(getenv("PSD_TC32_PAIR") && getenv("PSD_TC32_PAIR")[0] == '0');
  if (ts) {
    p.n_mma = 2;
    p.bn = (n_tot - 256 + 31) / 32 * 32;   // second piece
    n_tot = 256 + p.bn;
  } else {
    p.n_mma = n_tot > 256 ? 2 : 1;
    p.bn = (n_tot / p.n_mma + 15) / 16 * 16;
    p.bn2 = p.bn;
    const bool pair_split = op.mode == PARTIAL && p.n_mma == 2 &&
                            !(getenv("PSD_TC32_PAIR") && getenv("PSD_TC32_PAIR")[0] == '0');
    if (pair_split) p.bn2 = n_tot - p.bn;            // unequal halves, no padded columns (272 = 144 + 128)
    n_tot = p.bn + (p.n_mma > 1 ? p.bn2 : 0);
  }
  p.n_groups = (op.N + n_tot - 1) / n_tot;
  p.m_tiles = (op.M + BM - 1) / BM;
  const int sms = device_info().sms;
  // CTA pairs (cta_group::2) for the panel products unless disabled
  static const bool pair_ok = [] {
    const char* e = getenv("PSD_TC32_PAIR");
    return !(e && e[0] == '0');
  }();
  const bool pair = op.mode == PARTIAL && pair_ok;
  // the reconstruction (short K, store-bound) keeps 64-byte rows and 4 stages;
  // the panel products stream 128-byte rows
  const int sw = op.mode == MIRROR ? 64 : 128;
  const int bk = sw / 4;
  p.kblocks = (op.K + bk - 1) / bk;
  int splits = 1;
  if (op.mode == PARTIAL) {
    const long long base = (long long)(pair ? (op.M + 2 * BM - 1) / (2 * BM) : p.m_tiles) * p.n_groups;
    const int slots = pair ? sms / 2 : sms;
    double best = 1e30;
    // TMEM accumulation is FP32: bound the K length of each split (its error
    // grows with it); the fp64 reduction over splits adds the chunks exactly.
    static const int kchunk = [] {
      const char* e = getenv("PSD_TC32_KCHUNK");
      return e ? atoi(e) : 4096;
    }();
    const int smin = kchunk > 0 ? std::max(1, (op.K + kchunk - 1) / kchunk) : 1;
    const int smax = std::max(smin, std::min(std::max(op.max_splits, smin), p.kblocks / 8));
    for (int s = smin; s <= smax; ++s) {
      const long long units = base * s;
      const double t = (double)((units + slots - 1) / slots) / s + 0.01 * s;
      if (t < best - 1e-9) {
        best = t;
        splits = s;
      }
    }
    const long long ldw = (long long)p.n_groups * n_tot;
    while (splits > 1 && (size_t)splits * op.M * ldw > op.ws_elems) --splits;
    if ((size_t)op.M * ldw > op.ws_elems) return -3;
    p.out = op.ws;
    p.ldo = ldw;
    p.split_stride = (long long)op.M * ldw;
  } else {
    if (op.M != op.N) return -2;
    p.out = op.c32;
    p.ldo = op.ldc32;
    p.split_stride = 0;
  }
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;   // every split non-empty
  p.splits = splits;
  p.mode = op.mode;
  {
    const char* e = getenv("PSD_TC32_NPROD");   // experiment knob: tf32 products per k-step
    p.nprod = e ? std::max(1, std::min(3, atoi(e))) : 3;
  }
  const int sb = ts ? 2 * BM * sw + (256 + p.bn) * sw
                    : (pair ? 2 * BM * sw + (p.bn + (p.n_mma > 1 ? p.bn2 : 0)) * sw
                            : 2 * BM * sw + 2 * p.bn * p.n_mma * sw);
  const int epi_bytes = op.mode == MIRROR ? kMirrorEpi * 32 * 33 * 4 : 0;   // epilogue transpose tiles
  const int avail = (int)device_info().max_smem - 1024 - 2048 - epi_bytes;
  p.stages = std::min(8, avail / sb);
  if (p.stages < 2) return -4;
  const size_t smem = std::max<size_t>((size_t)p.stages * sb + epi_bytes + 1024, 120 * 1024);

  CUtensorMap mah, mal, mbh, mbl;
  const long long lda_lo = op.lda_lo ? op.lda_lo : op.lda;
  const int brows = pair ? p.bn / 2 : p.bn;
  const bool amn = pair && op.a_mn && !ts;
  bool ok;
  if (amn) {   // A stored K×M row-major (Aᵀ): box = 32 M-columns × BK K-rows
    ok = map_f32_box(&mah, op.a_hi, op.M, op.K, op.lda, 32, BK) &&
         map_f32_box(&mal, op.a_lo, op.M, op.K, lda_lo, 32, BK);
  } else {
    ok = map_f32(&mah, op.a_hi, op.K, op.M, op.lda, BM, sw) && map_f32(&mal, op.a_lo, op.K, op.M, lda_lo, BM, sw);
  }
  ok = ok && map_f32(&mbh, op.b_hi, op.K, op.N, op.ldb, brows, sw) && map_f32(&mbl, op.b_lo, op.K, op.N, op.ldb, brows, sw);
  CUtensorMap mbh2 = mbh, mbl2 = mbl;
  if (pair && p.n_mma > 1 && p.bn2 != p.bn)
    ok = ok && map_f32(&mbh2, op.b_hi, op.K, op.N, op.ldb, p.bn2 / 2, sw) &&
         map_f32(&mbl2, op.b_lo, op.K, op.N, op.ldb, p.bn2 / 2, sw);
  if (!ok) return -5;
  int dev = 0;
  cudaGetDevice(&dev);
  if (ts) {
    Ts2Maps mp;
    ok = map_f32(&mp.ah, op.a_hi, op.K, op.M, op.lda, BM, sw) && map_f32(&mp.al, op.a_lo, op.K, op.M, lda_lo, BM, sw) &&
         map_f32(&mp.bh0, op.b_hi, op.K, op.N, op.ldb, 128, sw) && map_f32(&mp.bl0, op.b_lo, op.K, op.N, op.ldb, 128, sw) &&
         map_f32(&mp.bh1, op.b_hi, op.K, op.N, op.ldb, p.bn / 2, sw) &&
         map_f32(&mp.bl1, op.b_lo, op.K, op.N, op.ldb, p.bn / 2, sw);
    if (!ok) return -5;
    static size_t attrts[16] = {};
    if (attrts[dev] < smem) {
      cudaFuncSetAttribute(tc32_gemm2ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attrts[dev] = smem;
    }
    const long long units = (long long)((op.M + 2 * BM - 1) / (2 * BM)) * p.n_groups * p.splits;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * units));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc32_gemm2ts_kernel, mp, p) != cudaSuccess) return -6;
  } else if (op.mode == MIRROR) {
    static size_t attrm[16] = {};
    if (attrm[dev] < smem) {
      cudaFuncSetAttribute(tc32_mirror_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attrm[dev] = smem;
    }
    long long ntiles = 0;
    for (int nt = 0; 2 * nt < p.m_tiles; ++nt) ntiles += p.m_tiles - 2 * nt;
    const int grid = (int)std::min<long long>(ntiles, sms);
    tc32_mirror_kernel<64><<<grid, kMirrorThreads, smem, st>>>(mah, mal, mbh, mbl, p, (int)ntiles);
  } else if (pair) {
    static size_t attr2[2][16] = {};
    if (attr2[amn][dev] < smem) {
      cudaFuncSetAttribute(amn ? tc32_gemm2_kernel<true> : tc32_gemm2_kernel<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr2[amn][dev] = smem;
    }
    const long long units = (long long)((op.M + 2 * BM - 1) / (2 * BM)) * p.n_groups * p.splits;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * units));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t le =
        amn ? cudaLaunchKernelEx(&cfg, tc32_gemm2_kernel<true>, mah, mal, mbh, mbl, mbh2, mbl2, p)
            : cudaLaunchKernelEx(&cfg, tc32_gemm2_kernel<false>, mah, mal, mbh, mbl, mbh2, mbl2, p);
    if (le != cudaSuccess) return -6;
  } else {
    static size_t attr64[16] = {}, attr128[16] = {};
    size_t* attr1 = sw == 64 ? attr64 : attr128;
    if (attr1[dev] < smem) {
      cudaFuncSetAttribute(sw == 64 ? tc32_gemm_kernel<64> : tc32_gemm_kernel<128>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr1[dev] = smem;
    }
    const long long units = (long long)p.m_tiles * p.n_groups * p.splits;
    if (sw == 64)
      tc32_gemm_kernel<64><<<(unsigned)units, kThreads, smem, st>>>(mah, mal, mbh, mbl, p);
    else
      tc32_gemm_kernel<128><<<(unsigned)units, kThreads, smem, st>>>(mah, mal, mbh, mbl, p);
  }
  count_launch();
  if (op.mode == PARTIAL) {
    const long long total = (long long)op.M * op.N;
    reduce_partials_kernel<<<grid_for(total, 256), 256, 0, st>>>(
        op.ws, p.splits, p.split_stride, p.ldo, op.M, op.N, op.c64, op.ldc64, op.alpha, op.S, op.lds);
    count_launch();
  }
  return p.splits;
}

void symsplit_f32(const float* x, long long n, long long ldx, double* stats, float* hi, float* lo,
                  long long ldh, cudaStream_t st, long long grid) {
  cudaMemsetAsync(stats, 0, 3 * sizeof(double), st);
  const long long nt = (n + tc32::kSST - 1) / tc32::kSST;
  const long long npairs = nt * (nt + 1) / 2;
  static const int per_sm = [] {
    const char* e = getenv("PSD_SYMSPLIT_BPS");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const long long blocks = std::min<long long>(npairs, grid > 0 ? grid : (long long)device_info().sms * per_sm);
  const bool vec = hi == nullptr && n % 4 == 0 && ldx % 4 == 0 && ldh % 4 == 0 &&
                   (uintptr_t)x % 16 == 0 && (uintptr_t)lo % 16 == 0;
  if (vec)
    tc32::symsplit4_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, n, ldx, npairs, stats, lo, ldh);
  else
    tc32::symsplit_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, n, ldx, npairs, stats, hi, lo, ldh,
                                                            hi == nullptr);
  count_launch();
}

void split_rows_f32(const float* x, long long rows, long long cols, long long ldx, float* hi,
                    float* lo, long long ldh, long long cols_pad, cudaStream_t st) {
  const bool vec = cols == cols_pad && cols % 4 == 0 && ldx % 4 == 0 && ldh % 4 == 0 &&
                   (uintptr_t)x % 16 == 0 && (uintptr_t)hi % 16 == 0 && (uintptr_t)lo % 16 == 0;
  const bool raw = hi == nullptr;
  if (vec) {
    const long long total = rows * (cols / 4);
    tc32::split_rows_f32x4_kernel<<<grid_for(total, 256), 256, 0, st>>>(
        reinterpret_cast<const float4*>(x), rows, cols / 4, ldx / 4, reinterpret_cast<float4*>(hi),
        reinterpret_cast<float4*>(lo), ldh / 4, raw);
  } else {
    tc32::split_rows_f32_kernel<<<grid_for(rows * cols_pad, 256), 256, 0, st>>>(x, rows, cols, ldx, hi,
                                                                                lo, ldh, cols_pad, raw);
  }
  count_launch();
}

void split_rows_f64(const double* x, long long rows, int cols, long long ldx, const double* scale,
                    float* hi, float* lo, long long ldh, int cols_pad, cudaStream_t st) {
  tc32::split_rows_f64_kernel<<<grid_for(rows * cols_pad, 256), 256, 0, st>>>(x, rows, cols, ldx, scale,
                                                                              hi, lo, ldh, cols_pad);
  count_launch();
}

void split_transpose(const double* P, long long n, int w, long long ldp, float* hi, float* lo,
                     long long ldt, int w_rows, cudaStream_t st) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((w_rows + 31) / 32));
  tc32::split_transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(P, n, w, ldp, hi, lo, ldt, w_rows);
  count_launch();
}

}  // namespace psd
