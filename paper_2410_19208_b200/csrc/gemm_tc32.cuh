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
  int kblocks, kb_per_split;
  int m_tiles, n_groups, splits;
  int stages;
  int mode;
  int nprod;            // tf32 products per k-step (3 = 3xTF32; fewer only for experiments)
  float* out;           // PARTIAL: out[split·split_stride + row·ldo + col]; MIRROR: C
  long long ldo, split_stride;
};


}  // namespace tc32
}  // namespace psd
