// 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05, TMEM) for the
// FP32 path of the projection (BASELINE config 3, fp32).
//
//   C (M×N) = A (M×K) · Bᵀ   with A, B both K-contiguous ("K-major") fp32,
//   each operand pre-split into tf32 hi/lo parts (hi = rna_tf32(x),
//   lo = rna_tf32(x − hi)), accumulated in FP32 in TMEM as
//   A_lo·B_hi + A_hi·B_lo + A_hi·B_hi  (the lo·lo term, 2⁻²² relative, dropped).
//
// Warp roles (192 threads, one CTA per SM):
//   warp 0  — one lane streams the four operand tiles per k-block with TMA
//             (SWIZZLE_64B, 64-byte rows = 16 fp32 of K) into a STAGES ring;
//   warp 1  — allocates TMEM; one lane issues tcgen05.mma.kind::tf32
//             (M = 128, N = bn ≤ 256, up to two N halves) and releases each
//             ring slot with tcgen05.commit → mbarrier;
//   warps 2–5 — epilogue: tcgen05.ld (32 lanes × 16 columns per load) of
//             their TMEM lane quadrant, then the output mode's stores.
// Grid = (m-tile, n-group, k-split) units, one per CTA.
#pragma once
#include <cuda.h>

#include "gemm_tma.cuh"

namespace psd {
namespace tc32 {

constexpr int BM = 128;
constexpr int SWZ = 128;         // smem row bytes (TMA/UMMA swizzle span) of the pair kernel
constexpr int BK = SWZ / 4;      // fp32 K elements per k-block of the pair kernel
constexpr int kThreads = 192;
constexpr int kMaxN = 512;       // TMEM columns

enum Mode { PARTIAL = 0, MIRROR = 1 };

struct Params {
  int M, N, K;
  int bn, n_mma;        // N per MMA (multiple of 16, ≤ 256), MMAs per k-step along N (1–2)
  int bn2;              // CTA-pair kernel: N of the second MMA (n_mma = 2), may differ from bn
  int kblocks, kb_per_split;
  int m_tiles, n_groups, splits;
  int stages;
  int mode;
  int nprod;            // tf32 products per k-step (3 = 3xTF32; fewer only for experiments)
  float* out;           // PARTIAL: out[split·split_stride + row·ldo + col]; MIRROR: C
  long long ldo, split_stride;
};



// ---- device helpers shared by the tcgen05 kernels (gemm_tc32.cu, ozaki.cu) ----
PSD_DEVINL void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
PSD_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
PSD_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

PSD_DEVINL void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// mbarrier wait that traps instead of hanging if a phase never completes
// (a mis-programmed pipeline fails loudly rather than wedging the GPU).
PSD_DEVINL void mbar_wait_t(uint32_t bar, uint32_t parity) {
  uint32_t done = 0, spins = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) return;
    if (++spins > (1u << 24)) __trap();
  }
}

PSD_DEVINL bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}
PSD_DEVINL uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
PSD_DEVINL uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
PSD_DEVINL void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

PSD_DEVINL void mma_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(bar)
      : "memory");
}

}  // namespace tc32
}  // namespace psd
