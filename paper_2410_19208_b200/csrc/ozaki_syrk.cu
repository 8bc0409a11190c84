// Reconstruction X̂₊ = W·diag(d)·Wᵀ (projection.py:72-78, _assemble_clipped) on
// the INT8 tensor cores: Ozaki scheme I (exact integer digit slices) for a SYRK.
//
//   V = W·diag(√d)  (d > 0: the kept eigenvalues), so X̂₊ = V·Vᵀ.
//   Row i of V is rounded to an integer a_ik = rint(v_ik·2^(7D−1−e_i)), |a| ≤ 2^(7D−1)
//   (e_i: max_k |v_ik| < 2^e_i), and split into D balanced base-128 digits
//   a = Σ_t d_t·128^(D−1−t), d_t ∈ [−64, 63] for t ≥ 1, |d_0| ≤ 65 (int8).  Then
//     Σ_k a_ik a_jk = Σ_{t,u} 128^(2D−2−t−u) · S_tu,   S_tu = Σ_k d_t(i,k)·d_u(j,k)
//   and the terms of level L = t+u ≤ D−1 are kept:  C = Σ_L 128^(D−1−L)·S_L with
//   S_L = Σ_{t+u=L} S_tu, each exact in s32 TMEM (|S_L| ≤ (L+1)·K·65·64).
//   X̂₊_ij = C · 2^(e_i + e_j − 7D − 5).
//
// Error per entry (D = 7): the rounding of each row to 48 bits (≤ 2^-49 of its max,
// unbiased) and the dropped levels (balanced digits: ≲ 6·2^-49 per term, zero-mean)
// → |Ĉ − VVᵀ|_ij ≤ 2^-45·K·2^(e_i+e_j) (tests/test_gpu_ozaki_syrk.py checks it entry
// by entry); ≈3.5e-14 relative Frobenius at the C3 shape (n = 32768, K = 158).
//
// Kernel: one persistent CTA per SM walks the 128×32 tiles on or below the diagonal
// (contiguous unit ranges, so a CTA mostly stays on one 128-row block).  The digits are
// stored pre-tiled and pre-swizzled (SWIZZLE_32B image of a stage), so per k-step
// (32 K-bytes) two contiguous bulk copies bring the D slices of the 128 A rows (28 KB)
// and of the 32 B rows (7 KB) — 3-D TMA boxes with 32-byte rows ran at a third of this
// rate.  The B slices sit contiguously as one 32·D-row operand, so ONE MMA per A slice
// t (N = 32·(D−t), accumulator columns from 32·t) adds S_t,u for every u ≤ D−1−t into
// level t+u.  Two TMEM buffers (D·32 ≤ 224 columns each); 8 epilogue warps load their
// 16 columns × D levels, hand the buffer back at once, then combine the levels (s32 pair
// + IMAD.WIDE onto a magic-number double, one FMA) and store both (i,j) (256-bit row
// stores) and (j,i) (256-byte warp stores) while the MMAs of the next tiles run.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "gemm_tc32.cuh"
#include "launch.h"

namespace psd {
namespace ozs {

constexpr int BM = 128;        // tile rows (TMEM lanes)
constexpr int BN = 32;         // tile columns per level
constexpr int KB = 32;         // K bytes per stage (one kind::i8 MMA)
#ifndef PSD_SYRK_EPI
#define PSD_SYRK_EPI 8
#endif
// epilogue warps: kEpi/4 per TMEM lane quadrant, each owning kGroups groups of 8 columns of
// the 32-column tile.  8 warps × 2 groups (168 registers) measured 2.46 ms at C3; 16 warps ×
// 1 group is capped at 96 registers by the 576-thread block and spills: 2.73 ms.
constexpr int kEpi = PSD_SYRK_EPI;
constexpr int kGroups = 32 / (kEpi / 4) / 8;
static_assert(kGroups >= 1 && (kEpi / 4) * kGroups * 8 == 32, "epilogue warps must tile 32 columns");
constexpr int kThreads = (2 + kEpi) * 32;
constexpr int kBufCols = 256;  // TMEM column offset of the second accumulator

// SWIZZLE_32B position of byte k (0..31) of row r inside an 8-row × 32-byte atom
// (the 16-byte halves of rows 4–7 swap: address bit 4 ^= bit 7)
PSD_DEVINL int sw32(int r, int k) { return r * 32 + (k ^ (((r >> 2) & 1) << 4)); }

// Rows of V = W·diag(√d) → balanced base-128 digits, written twice, pre-tiled and
// pre-swizzled exactly as the MMA reads them from shared memory, so one contiguous
// bulk copy fills a stage:
//   A tiles [I][kb][t][128 rows][32 B]  (row blocks of 128),
//   B tiles [J][kb][t][32 rows][32 B]   (row blocks of 32).
// Rows ≥ n (up to the 128-row padding) are zero.  rs / cs: row / column scales.
template <int D>
__global__ void __launch_bounds__(256) syrk_slices_kernel(const double* __restrict__ w, long long n, int r,
                                                         long long ldw, const double* __restrict__ d,
                                                         int8_t* __restrict__ ta, int8_t* __restrict__ tb,
                                                         int nkb, long long rows_a, long long rows_b,
                                                         double* __restrict__ rs, double* __restrict__ cs) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= rows_a) return;
  int ei = 0;
  if (i < n) {
    const double* row = w + i * ldw;
    double mx = 0.0;
    for (int k = lane; k < r; k += 32) mx = fmax(mx, fabs(row[k] * sqrt(d[k])));
    mx = warp_max(mx);
    ei = mx > 0.0 ? ilogb(mx) + 1 : 0;
  }
  // X̂_ij = C·2^(e_i + e_j − 7D − 5), split as 2^(e_i − 32) · 2^(e_j − 7D + 27)
  if (lane == 0) {   // padded to the 128-row (rs) / 32-row (cs) tiles
    rs[i] = i < n ? ldexp(1.0, ei - 32) : 0.0;
    if (i < rows_b) cs[i] = i < n ? ldexp(1.0, ei - 7 * D + 27) : 0.0;
  }
  const double sc = ldexp(1.0, 7 * D - 1 - ei);
  const long long ia = i >> 7, ib = i >> 5;
  const int ra = (int)(i & 127), rb = (int)(i & 31);
  for (int kb = 0; kb < nkb; ++kb) {
    const int k = kb * 32 + lane;
    long long a = 0;
    if (i < n && k < r) a = __double2ll_rn(w[i * ldw + k] * sqrt(d[k]) * sc);   // |a| ≤ 2^(7D−1)
    int8_t dg[D];
    // balanced digits: d_t ∈ [−64, 63] for t ≥ 1, top digit |d_0| ≤ 65
#pragma unroll
    for (int t = D - 1; t >= 1; --t) {
      const long long v = ((a + 64) & 127) - 64;
      dg[t] = (int8_t)v;
      a = (a - v) >> 7;
    }
    dg[0] = (int8_t)a;
    int8_t* oa = ta + ((ia * nkb + kb) * D) * (128 * 32) + sw32(ra, lane);
#pragma unroll
    for (int t = 0; t < D; ++t) oa[t * 128 * 32] = dg[t];
    if (i < rows_b) {
      int8_t* ob = tb + ((ib * nkb + kb) * D) * (32 * 32) + sw32(rb, lane);
#pragma unroll
      for (int t = 0; t < D; ++t) ob[t * 32 * 32] = dg[t];
    }
  }
}

struct SyrkParams {
  int n, kblocks, mt, nt;
  long long units;
  const int8_t* ta;   // pre-swizzled A tiles [I][kb][t][128][32]
  const int8_t* tb;   // pre-swizzled B tiles [J][kb][t][32][32]
  double* c;
  long long ldc;
  const double* rs;   // 2^(e_i − 32)      (row scale), padded to the 128-row tiles
  const double* cs;   // 2^(e_j − 7D + 27) (column scale), padded to the 32-row tiles
  int stages;
  int vec;   // 1: C and ldc allow 32-byte row stores
};

PSD_DEVINL void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
PSD_DEVINL void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// K-major SWIZZLE_32B operand: 8-row atoms of 32-byte rows, SBO = 256 B, layout type 6
PSD_DEVINL uint64_t desc_sw32(uint32_t saddr) {
  uint64_t dsc = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  dsc |= (uint64_t)1 << 16;
  dsc |= (uint64_t)(256 >> 4) << 32;
  dsc |= (uint64_t)1 << 46;
  dsc |= (uint64_t)6 << 61;
  return dsc;
}
PSD_DEVINL void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
PSD_DEVINL void tmem_ld16(uint32_t taddr, uint32_t (&r)[8], uint32_t (&q)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
      : "r"(taddr));
}
PSD_DEVINL void st_v4_f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}
// exact s32 → f64 (|s| < 2^31): 1.5·2^52 + 2^31 + s has s + 2^31 in its low word
PSD_DEVINL double s32_to_f64(uint32_t s) {
  return __hiloint2double(0x43380000, (int)(s ^ 0x80000000u)) - 6755401588539392.0;
}
// unit u → tile (I, J): row block I holds min(4(I+1), nt) column tiles, prefix 2I(I+1)
PSD_DEVINL void unit_tile(long long u, int& I, int& J) {
  int i = (int)((sqrt(2.0 * (double)u + 1.0) - 1.0) * 0.5);
  while (2LL * (i + 1) * (i + 2) <= u) ++i;
  while (2LL * i * (i + 1) > u) --i;
  I = i;
  J = (int)(u - 2LL * i * (i + 1));
}

// AR (A resident): the D digit slices of the current 128-row block for ALL k-steps stay
// in shared memory (nkb·28 KB) while the CTA walks that block's column tiles; only the
// 7 KB B slices stream per k-step.  Otherwise A and B stream together per k-step.
template <int D, bool AR>
__global__ void __launch_bounds__(kThreads, 1) i8_syrk_kernel(const SyrkParams p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], accf_bar[2], acce_bar[2], afull_bar, aempty_bar;
  // per-unit row / column scales, 4 slots filled by the producer with the unit's bulk copies
  __shared__ __align__(8) uint64_t sfull_bar[4], sempty_bar[4];
  __shared__ __align__(16) double s_rs[4][BM], s_cs[4][BN];
  __shared__ uint32_t tmem_slot;
  constexpr uint32_t a_bytes = D * BM * KB, b_bytes = D * BN * KB;
  constexpr uint32_t st_bytes = AR ? b_bytes : a_bytes + b_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const long long u0 = p.units * blockIdx.x / gridDim.x, u1 = p.units * (blockIdx.x + 1) / gridDim.x;
  const int nkb = p.kblocks;
  const uint32_t sring = AR ? sbase + (uint32_t)nkb * a_bytes : sbase;   // AR: A block first, then the B ring

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&accf_bar[b]), 1);
      mbar_init(smem_u32(&acce_bar[b]), kEpi);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(smem_u32(&sfull_bar[b]), 1);
      mbar_init(smem_u32(&sempty_bar[b]), kEpi);
    }
    mbar_init(smem_u32(&afull_bar), 1);
    mbar_init(smem_u32(&aempty_bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc32::tc_fence_before();
  __syncthreads();
  tc32::tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    int aload = 0, curI = -1, j = 0, rs = 0;
    uint32_t rph = 0;
    int I, J;
    unit_tile(u0, I, J);
    for (long long u = u0; u < u1; ++u, ++j) {
      {   // this unit's 128 row scales and 32 column scales → slot j mod 4
        const int sb = j & 3;
        tc32::mbar_wait_t(smem_u32(&sempty_bar[sb]), (((uint32_t)j >> 2) & 1u) ^ 1u);
        if (tc32::elect_one()) {
          const uint32_t sf = smem_u32(&sfull_bar[sb]);
          mbar_expect_tx(sf, (BM + BN) * sizeof(double));
          bulk_load(smem_u32(&s_rs[sb][0]), p.rs + (long long)I * BM, BM * sizeof(double), sf);
          bulk_load(smem_u32(&s_cs[sb][0]), p.cs + (long long)J * BN, BN * sizeof(double), sf);
        }
        __syncwarp();
      }
      if (AR && I != curI) {
        // the previous block's MMAs have all retired (aempty) → load this block's A slices
        tc32::mbar_wait_t(smem_u32(&aempty_bar), ((uint32_t)aload & 1u) ^ 1u);
        if (tc32::elect_one()) {
          const uint32_t ab = smem_u32(&afull_bar);
          mbar_expect_tx(ab, (uint32_t)nkb * a_bytes);
          for (int kb = 0; kb < nkb; ++kb)
            bulk_load(sbase + (uint32_t)kb * a_bytes, p.ta + ((long long)I * nkb + kb) * a_bytes, a_bytes, ab);
        }
        __syncwarp();
        ++aload;
        curI = I;
      }
      for (int kb = 0; kb < nkb; ++kb) {
        tc32::mbar_wait_t(smem_u32(&empty_bar[rs]), rph ^ 1u);
        if (tc32::elect_one()) {
          const uint32_t fb = smem_u32(&full_bar[rs]);
          mbar_expect_tx(fb, st_bytes);
          const uint32_t sS = sring + rs * st_bytes;
          if (AR) {
            bulk_load(sS, p.tb + ((long long)J * nkb + kb) * b_bytes, b_bytes, fb);
          } else {
            bulk_load(sS, p.ta + ((long long)I * nkb + kb) * a_bytes, a_bytes, fb);
            bulk_load(sS + a_bytes, p.tb + ((long long)J * nkb + kb) * b_bytes, b_bytes, fb);
          }
        }
        __syncwarp();
        if (++rs == p.stages) {   // ring position kept incrementally (no division per k-step)
          rs = 0;
          rph ^= 1u;
        }
      }
      if (++J >= min(4 * (I + 1), p.nt)) {
        ++I;
        J = 0;
      }
    }
  } else if (warp == 1) {
    int j = 0, aload = 0, curI = -1, rs = 0;
    uint32_t rph = 0;
    int I, J;
    unit_tile(u0, I, J);
    // descriptors built once; per MMA only the start-address field moves (byte offset >> 4,
    // smem addresses < 2^18 so the 14-bit field never carries)
    const uint64_t a_desc0 = desc_sw32(AR ? sbase : sring);
    const uint64_t b_desc0 = desc_sw32(AR ? sring : sring + a_bytes);
    for (long long u = u0; u < u1; ++u, ++j) {
      const int b = j & 1;
      if (AR && I != curI) {
        if (curI >= 0) {   // release the old A block once its MMAs retire
          if (tc32::elect_one()) tc32::mma_commit(smem_u32(&aempty_bar));
          __syncwarp();
        }
        tc32::mbar_wait_t(smem_u32(&afull_bar), (uint32_t)aload & 1u);
        ++aload;
        curI = I;
      }
      tc32::mbar_wait_t(smem_u32(&acce_bar[b]), (((uint32_t)j >> 1) & 1u) ^ 1u);
      tc32::tc_fence_after();
      const uint32_t dbuf = tmem + (uint32_t)(b * kBufCols);
      for (int kb = 0; kb < nkb; ++kb) {
        tc32::mbar_wait_t(smem_u32(&full_bar[rs]), rph);
        tc32::tc_fence_after();
        if (tc32::elect_one()) {
          const uint32_t soff = (uint32_t)rs * st_bytes;
          const uint64_t ad = a_desc0 + ((AR ? (uint32_t)kb * a_bytes : soff) >> 4);
          const uint64_t db = b_desc0 + (soff >> 4);
#pragma unroll
          for (int t = 0; t < D; ++t) {
            // kind::i8: D s32, A/B signed, K-major, M = 128, N = 32·(D − t)
            constexpr uint32_t base = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BM >> 4) << 24);
            const uint32_t idesc = base | ((uint32_t)((BN * (D - t)) >> 3) << 17);
            mma_i8(dbuf + (uint32_t)(t * BN), ad + (uint64_t)((t * BM * KB) >> 4), db, idesc, (kb | t) != 0);
          }
          tc32::mma_commit(smem_u32(&empty_bar[rs]));
          if (kb == nkb - 1) tc32::mma_commit(smem_u32(&accf_bar[b]));
        }
        __syncwarp();
        if (++rs == p.stages) {
          rs = 0;
          rph ^= 1u;
        }
      }
      if (++J >= min(4 * (I + 1), p.nt)) {
        ++I;
        J = 0;
      }
    }
  } else {
    const int quad = warp & 3;
    const int slice = (warp - 2) >> 2;          // columns 8·kGroups·slice … of each level
    const uint32_t tq = (uint32_t)(quad * 32) << 16;
    // barrier addresses hoisted (each smem_u32 of a __shared__ object costs an S2R)
    const uint32_t accf0 = smem_u32(&accf_bar[0]), acce0 = smem_u32(&acce_bar[0]);
    const uint32_t sfull0 = smem_u32(&sfull_bar[0]), sempty0 = smem_u32(&sempty_bar[0]);
    int I, J;
    unit_tile(u0, I, J);
    int j = 0;
    for (long long u = u0; u < u1; ++u, ++j) {
      const int b = j & 1, sb = j & 3;
      tc32::mbar_wait_t(accf0 + 8u * (uint32_t)b, ((uint32_t)j >> 1) & 1u);
      tc32::tc_fence_after();
      tc32::mbar_wait_t(sfull0 + 8u * (uint32_t)sb, ((uint32_t)j >> 2) & 1u);
      const int ib = I * BM + quad * 32;
      const int i = ib + lane;
      const int jb = J * BN + slice * 8 * kGroups;
      // warp-uniform: the 8-column group g holds some (i, j) with j ≤ i
      bool active[kGroups];
      uint32_t v[kGroups][D][8];
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const int j0 = jb + 8 * g;
        active[g] = j0 <= ib + 31 && j0 < p.n && ib < p.n;
      }
      if constexpr (kGroups == 2) {   // both groups of a level in one 16-column load
        if (active[0]) {
#pragma unroll
          for (int L = 0; L < D; ++L)
            tmem_ld16(tmem + tq + (uint32_t)(b * kBufCols + L * BN + slice * 16), v[0][L], v[1][L]);
        }
      } else {
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
          if (active[g]) {
#pragma unroll
            for (int L = 0; L < D; ++L)
              tmem_ld8(tmem + tq + (uint32_t)(b * kBufCols + L * BN + slice * 8 * kGroups + 8 * g), v[g][L]);
          }
        }
      }
      const double si = s_rs[sb][quad * 32 + lane];
      if (active[0]) asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      // the accumulator is in registers: hand the TMEM buffer back before the math and stores
      tc32::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acce0 + 8u * (uint32_t)b);
      const bool row_ok = i < p.n;
      const long long ldc = p.ldc;
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        if (!active[g]) continue;
        const int j0 = jb + 8 * g;
        const double* sj = &s_cs[sb][slice * 8 * kGroups + 8 * g];   // broadcast smem reads
        double val[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          // C = (S_0·128 + S_1)·2^(7(D−2)) + Σ_{L≥2} S_L·2^(7(D−1−L)): the high pair in s32
          // (|S_0·128 + S_1| < 2^31 for K ≤ 3900), the rest accumulated by IMAD.WIDE onto the
          // bit pattern of 1.5·2^52 (|Σ| < 2^51 for K ≤ 640), so one DADD yields it exactly
          const int top = (int)v[g][0][q] * 128 + (int)v[g][1][q];
          long long lo = 0x4338000000000000LL;
#pragma unroll
          for (int L = 2; L < D; ++L) lo += (long long)(int)v[g][L][q] * (long long)(1 << (7 * (D - 1 - L)));
          const double low = __longlong_as_double(lo) - 6755399441055744.0;
          const double acc = fma(s32_to_f64((uint32_t)top), (double)(1LL << (7 * (D - 2))), low);
          val[q] = acc * si * sj[q];
        }
        // (j, i): for each column, the warp's 32 consecutive rows — one 256-byte store
        double* colp = p.c + (long long)j0 * ldc + i;
        const int jlim = row_ok ? i : 0;   // store (j, i) for j < i (i < n, so j < n)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (j0 + q < jlim) *colp = val[q];
          colp += ldc;
        }
        // (i, j): this thread's 8 consecutive columns
        double* dst = p.c + (long long)i * ldc + j0;
        if (row_ok && p.vec && j0 + 7 <= i && j0 + 7 < p.n) {
          st_v4_f64(dst, val[0], val[1], val[2], val[3]);
          st_v4_f64(dst + 4, val[4], val[5], val[6], val[7]);
        } else if (row_ok) {
          const int jl2 = min(i + 1, p.n);
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (j0 + q < jl2) dst[q] = val[q];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty0 + 8u * (uint32_t)sb);   // scale slot read
      if (++J >= min(4 * (I + 1), p.nt)) {
        ++I;
        J = 0;
      }
    }
  }
  tc32::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc32::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace ozs

namespace {

int syrk_digits() {
  static const int dg = [] {
    const char* s = getenv("PSD_OZ_SYRK_DIGITS");
    const int v = s ? atoi(s) : 7;
    return (v == 6) ? 6 : 7;
  }();
  return dg;
}

template <int D>
int launch_syrk(const double* w, long long n, int r, long long ldw, const double* d, double* c, long long ldc,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace ozs;
  SyrkParams p{};
  p.n = (int)n;
  p.kblocks = (r + KB - 1) / KB;
  p.mt = (int)((n + BM - 1) / BM);
  p.nt = (int)((n + BN - 1) / BN);
  const size_t ta_bytes = (size_t)p.mt * p.kblocks * D * BM * KB, tb_bytes = (size_t)p.nt * p.kblocks * D * BN * KB;
  const long long rows_a = (long long)p.mt * BM, rows_b = (long long)p.nt * BN;
  if (ws_bytes < ta_bytes + tb_bytes + (size_t)(rows_a + rows_b) * sizeof(double) || (uintptr_t)ws % 256) return -3;
  int8_t* ta = static_cast<int8_t*>(ws);
  int8_t* tb = ta + ta_bytes;
  double* rs = reinterpret_cast<double*>(tb + tb_bytes);
  double* cs = rs + rows_a;
  syrk_slices_kernel<D><<<(unsigned)((rows_a + 7) / 8), 256, 0, st>>>(w, n, r, ldw, d, ta, tb, p.kblocks, rows_a,
                                                                       rows_b, rs, cs);
  count_launch();
  p.units = 2LL * (p.mt - 1) * p.mt + std::min(4 * p.mt, p.nt);
  p.ta = ta;
  p.tb = tb;
  p.c = c;
  p.ldc = ldc;
  p.rs = rs;
  p.cs = cs;
  p.vec = ((uintptr_t)c % 32 == 0 && ldc % 4 == 0) ? 1 : 0;
  // A resident when the block's slices leave room for a ≥ 4-deep B ring
  // dynamic budget: opt-in maximum minus the kernel's static shared memory (barriers, scale
  // slots ≈ 5.4 KB) and the 1 KB alignment slack
  const int budget = (int)device_info().max_smem - 8192;
  const int a_blk = p.kblocks * D * BM * KB, b_st = D * BN * KB;
  static const bool ar_on = [] { const char* e = getenv("PSD_OZ_SYRK_AR"); return !(e && e[0] == '0'); }();
  const bool ar = ar_on && a_blk + 4 * b_st <= budget;
  const int st_bytes = ar ? b_st : D * (BM + BN) * KB;
  p.stages = std::min(8, (budget - (ar ? a_blk : 0)) / st_bytes);
  const size_t smem = (size_t)(ar ? a_blk : 0) + (size_t)p.stages * st_bytes + 1024;
  auto kern = ar ? i8_syrk_kernel<D, true> : i8_syrk_kernel<D, false>;
  static size_t attr[2][16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr[ar][dev] < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[ar][dev] = smem;
  }
  const int grid = (int)std::min<long long>(device_info().sms, p.units);
  kern<<<grid, kThreads, smem, st>>>(p);
  count_launch();
  if (cudaPeekAtLastError() != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "i8_syrk launch failed: %s (regs %d, maxThreadsPerBlock %d, static smem %zu, dyn smem %zu, "
            "threads %d)\n", cudaGetErrorString(cudaPeekAtLastError()), fa.numRegs, fa.maxThreadsPerBlock,
            fa.sharedSizeBytes, smem, kThreads);
    return -6;
  }
  return 0;
}

}  // namespace

size_t oz_syrk_ws_bytes(long long n, int r) {
  const size_t kb = (size_t)(r + 31) / 32;
  const size_t rows_a = (size_t)(n + 127) / 128 * 128, rows_b = (size_t)(n + 31) / 32 * 32;
  return 7 * kb * 32 * (rows_a + rows_b) + (rows_a + rows_b) * sizeof(double);
}

// C (n×n) = W·diag(d)·Wᵀ, all d > 0, written as a bitwise-symmetric matrix.
int oz_syrk(const double* w, long long n, int r, long long ldw, const double* d, double* c, long long ldc,
            void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n < 1 || r < 1) return 0;
  if (r > 640) return -2;   // exact level combination in the epilogue needs K ≤ 640
  return syrk_digits() == 6 ? launch_syrk<6>(w, n, r, ldw, d, c, ldc, ws, ws_bytes, st)
                            : launch_syrk<7>(w, n, r, ldw, d, c, ldc, ws, ws_bytes, st);
}

}  // namespace psd
