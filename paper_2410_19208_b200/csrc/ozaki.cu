// FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme II: integer
// scaling + Chinese-remainder reconstruction), for the n×n · n×w products of
// the projection.
//
//   A (M×K, fp64) is scaled per row to 53-bit integers a = rint(x·2^(53−e_i)),
//   B (K×N, fp64) per column to b = rint(p·2^(53−f_j));
//   for 16 pairwise-coprime moduli m_ℓ ≤ 256 the symmetric residues a mod m_ℓ,
//   b mod m_ℓ are int8; each (A mod m_ℓ)·(B mod m_ℓ) runs as an exact INT8
//   GEMM with INT32 TMEM accumulation (|Σ| ≤ K·2^14 < 2^31 per K split of
//   ≤ 32768), reduced mod m_ℓ; a direct CRT (Σ_ℓ y_ℓ·M/m_ℓ, quotient by a
//   float estimate, 128-bit wrap) recovers the exact integer product
//   C' = Σ_k a_ik b_kj and C = C'·2^(e_i + f_j − 106).  Exactness needs
//   |C'| ≤ K·2^106 < M/2 (M = Π m_ℓ ≈ 2^125.4), i.e. K < 2^18.4: every entry
//   point rejects K > kMaxK = 2^18 (|C'|/M ≤ 2^-1.4) and the callers keep such
//   products on the FP64 DMMA kernel.
//
// The only rounding is the 53-bit fixed-point truncation of each row / column
// (≤ 2^-54 of its largest entry) and the final conversion of C' to double —
// the result is as accurate as an FP64 GEMM.  Cost: 16 INT8 GEMMs (≈ 4.5
// POPS dense) and one n²-byte residue stream per modulus instead of an FP64
// DMMA GEMM (≈ 37 TFLOP/s).
#include <cudaTypedefs.h>

#include <algorithm>
#include <utility>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "gemm_tc32.cuh"
#include "launch.h"

namespace psd {
namespace oz {

constexpr int kNumMod = 16;
constexpr long long kMaxK = 1LL << 18;   // CRT exactness: K·2^106 < M/2 (see the header)
constexpr int kMods[kNumMod] = {256, 255, 253, 251, 247, 241, 239, 233,
                                229, 227, 223, 217, 211, 199, 197, 193};
// compile-time modulus tables: inside the residue loops l is a template constant, so
// the limb weights, 1/m and −m become instruction immediates (FFMA immediate form
// issues at twice the rate of the constant-bank form on the fma pipe)
__host__ __device__ constexpr int mod_at(int l) {
  return l == 0 ? 256 : l == 1 ? 255 : l == 2 ? 253 : l == 3 ? 251 : l == 4 ? 247 : l == 5 ? 241 :
         l == 6 ? 239 : l == 7 ? 233 : l == 8 ? 229 : l == 9 ? 227 : l == 10 ? 223 : l == 11 ? 217 :
         l == 12 ? 211 : l == 13 ? 199 : l == 14 ? 197 : 193;
}
__host__ __device__ constexpr float pow13_sym(int l, int t) {   // 2^(13t) mod m in (−m/2, m/2]
  long long v = 1;
  for (int i = 0; i < t; ++i) v = (v * 8192) % mod_at(l);
  return (float)(v > mod_at(l) / 2 ? v - mod_at(l) : v);
}
static_assert(mod_at(15) == 193, "modulus table");

__constant__ int c_mod[kNumMod];
__constant__ double c_rmod[kNumMod];        // 1 / m
__constant__ float c_rmodf[kNumMod];        // 1 / m (fp32) for small non-negative operands
__constant__ int c_inv[kNumMod][kNumMod];   // (m_i)^{-1} mod m_j, i < j
__constant__ unsigned long long c_M[2];     // M = Π m_ℓ as (lo, hi)
__constant__ float c_modf[kNumMod];         // m_ℓ
__constant__ uint32_t c_nmod[kNumMod];      // −m_ℓ mod 2^32
__constant__ float c_pow13f[4][kNumMod];    // 2^(13t) mod m_ℓ in (−m/2, m/2]
__constant__ float c_wInvf[kNumMod];        // (M/m_ℓ)^{-1} mod m_ℓ
__constant__ unsigned long long c_W[kNumMod][2];   // M/m_ℓ as (lo, hi)
// y-table of the single-split CRT: g_ytab[ℓ][b] = (r·(M/m_ℓ)^{-1} mod m_ℓ) ∈ [0, m_ℓ) for the
// stored residue byte b (r = (int8)b), four entries per word
__device__ uint32_t g_ytab[kNumMod * 64];

// fp32 integer tricks.  kMagic = 1.5·2^23: fmaf(s, 1/m, kMagic) − kMagic = rint(s/m)
// for |s| < 2^22·m; the bits of (r + kMagic) hold the integer r in their low bytes.
constexpr float kMagic = 12582912.0f;
PSD_DEVINL float sym_mod_f(float s, float m, float rm) {   // s − m·rint(s/m), |s| < 2^24 exact
  const float q = fmaf(s, rm, kMagic) - kMagic;
  return fmaf(-m, q, s);
}
PSD_DEVINL uint32_t low_bits(float r) { return __float_as_uint(r + kMagic); }
PSD_DEVINL float u2f_small(uint32_t u) { return __uint_as_float(u | 0x4B000000u) - 8388608.0f; }   // u < 2^23
PSD_DEVINL uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {   // low bytes → one word
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

constexpr int BM = 128;
constexpr int BKB = 128;                    // K bytes (= int8 elements) per stage row (SWIZZLE_128B)
constexpr int kThreads = 192;

// r = v mod m ∈ [0, m) for |v| < 2^53 (exact: fma residual, one fix-up)
PSD_DEVINL int mod_pos(double v, int l) {
  const double m = (double)c_mod[l];
  const double q = floor(v * c_rmod[l]);
  double r = fma(-m, q, v);
  if (r < 0.0) r += m;
  if (r >= m) r -= m;
  return (int)r;
}
// x mod m for 0 ≤ x < 2^22 (fp32 reciprocal, one fix-up each way)
PSD_DEVINL int mod_small(int x, int l) {
  const int m = c_mod[l];
  int q = (int)((float)x * c_rmodf[l]);
  int r = x - q * m;
  if (r < 0) r += m;
  if (r >= m) r -= m;
  return r;
}
// symmetric residue as int8: [−128, 127] for m = 256, [−(m−1)/2, (m−1)/2] for odd m
PSD_DEVINL int8_t sym_res(int r, int l) {
  const int m = c_mod[l];
  return (int8_t)(r > (m - 1) / 2 ? r - m : r);
}

// ---- exponents: e[i] with max_k |x_ik| < 2^e[i] (0 for an all-zero row) ----------
__global__ void row_exp_kernel(const double* __restrict__ x, long long rows, long long cols,
                               long long ldx, int* __restrict__ e) {
  const long long i = blockIdx.x;
  if (i >= rows) return;
  double m = 0.0;
  const double* row = x + i * ldx;
  for (long long k = threadIdx.x; k < cols; k += blockDim.x) m = fmax(m, fabs(__ldcs(row + k)));
  m = warp_max(m);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    e[i] = t > 0.0 ? ilogb(t) + 1 : 0;
  }
}
// column exponents of a K×N row-major panel: atomicMax over per-element exponents
__global__ void col_exp_kernel(const double* __restrict__ p, long long rows, int cols, long long ldp,
                               int* __restrict__ f) {
  // max over the block's rows in registers (doubles: the exponent is taken once per column),
  // the 8 warps combined in shared memory, then ONE atomic per column per block
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.y * 32 + lane;
  double mx = 0.0;
  if (j < cols)
    for (long long k = blockIdx.x * 8 + warp; k < rows; k += (long long)gridDim.x * 8)
      mx = fmax(mx, fabs(p[k * ldp + j]));
  red[warp][lane] = mx;
  __syncthreads();
  if (warp == 0 && j < cols) {
#pragma unroll
    for (int w = 1; w < 8; ++w) mx = fmax(mx, red[w][lane]);
    if (mx > 0.0) atomicMax(&f[j], ilogb(mx) + 1);
  }
}

// ---- residues of a row-scaled matrix: R[ℓ][i][k] (int8), ld ldr bytes ---------------
template <int L>
PSD_DEVINL void res_limb_store8(const float (&f)[8][4], int8_t* out, long long plane) {
  constexpr float m = (float)mod_at(L), rm = 1.0f / (float)mod_at(L);
  constexpr float p1 = pow13_sym(L, 1), p2 = pow13_sym(L, 2), p3 = pow13_sym(L, 3);
  constexpr uint32_t nmi = 0u - (uint32_t)mod_at(L);
  uint32_t b[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float sacc = fmaf(f[q][3], p3, fmaf(f[q][2], p2, fmaf(f[q][1], p1, f[q][0])));
    if constexpr (L == 1) {   // m = 255: |r| can reach 128 — fold into int8 range
      float rr = sym_mod_f(sacc, m, rm);
      rr = rr > 127.5f ? rr - m : rr;
      b[q] = low_bits(rr);
    } else {                  // |r| ≤ 0.503·m ≤ 127
      b[q] = __float_as_uint(fmaf(sacc, rm, kMagic)) * nmi + __float_as_uint(sacc + kMagic);
    }
  }
  *reinterpret_cast<uint2*>(out + L * plane) =
      make_uint2(pack4(b[0], b[1], b[2], b[3]), pack4(b[4], b[5], b[6], b[7]));
}
template <int L>
PSD_DEVINL void res_limb_all(const float (&f)[8][4], int8_t* out, long long plane) {
  if constexpr (L < kNumMod) {
    res_limb_store8<L>(f, out, plane);
    res_limb_all<L + 1>(f, out, plane);
  }
}

// 4 consecutive k (one 32-bit word per modulus), compile-time modulus constants
template <int L>
PSD_DEVINL void res_limb_store4(const float (&f)[4][4], int8_t* out, long long plane) {
  constexpr float m = (float)mod_at(L), rm = 1.0f / (float)mod_at(L);
  constexpr float p1 = pow13_sym(L, 1), p2 = pow13_sym(L, 2), p3 = pow13_sym(L, 3);
  constexpr uint32_t nmi = 0u - (uint32_t)mod_at(L);
  uint32_t b[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float sacc = fmaf(f[q][3], p3, fmaf(f[q][2], p2, fmaf(f[q][1], p1, f[q][0])));
    if constexpr (L == 1) {
      float rr = sym_mod_f(sacc, m, rm);
      rr = rr > 127.5f ? rr - m : rr;
      b[q] = low_bits(rr);
    } else {
      b[q] = __float_as_uint(fmaf(sacc, rm, kMagic)) * nmi + __float_as_uint(sacc + kMagic);
    }
  }
  *reinterpret_cast<uint32_t*>(out + L * plane) = pack4(b[0], b[1], b[2], b[3]);
}
template <int L>
PSD_DEVINL void res_limb_all4(const float (&f)[4][4], int8_t* out, long long plane) {
  if constexpr (L < kNumMod) {
    res_limb_store4<L>(f, out, plane);
    res_limb_all4<L + 1>(f, out, plane);
  }
}

// ---- residues via paired moduli on the FP64 pipe ------------------------------------
// The 16 moduli form 8 pairs (m_P, m_{15−P}) with M_P = m_P·m_{15−P} < 2^16.  For the
// 53-bit integer a (exact in a double): r = a − M_P·rint(a/M_P) by two DFMA and a DADD
// (|r| < M_P/2 + 1 < 2^15), its low word comes out of one more DADD onto 1.5·2^52, and
// the two residues are r mod m_P and r mod m_{15−P} with the fp32 trick of
// res_limb_store8 (one FFMA + one IMAD each, r exact in fp32).  m = 256 (pair 0) is the
// low byte of r.  Per (element, modulus) ≈ 5 issue slots instead of ≈ 9 for the
// 13-bit-limb form, spread over the FP64 and FP32 pipes.
constexpr double kMagicD = 6755399441055744.0;   // 1.5·2^52
template <int P>
PSD_DEVINL void res_pair_store8(const double (&a)[8], int8_t* out, long long plane) {
  constexpr int lo = P, hi = kNumMod - 1 - P;
  constexpr int m1 = mod_at(lo), m2 = mod_at(hi);
  constexpr double M = (double)(m1 * m2);
  constexpr double rM = 1.0 / M;
  constexpr float rm1 = 1.0f / (float)m1, rm2 = 1.0f / (float)m2;
  constexpr uint32_t n1 = 0u - (uint32_t)m1, n2 = 0u - (uint32_t)m2;
  uint32_t b1[8], b2[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double qd = fma(a[q], rM, kMagicD) - kMagicD;     // rint(a/M) (±1: |r| < M/2 + 1)
    const double r = fma(-qd, M, a[q]);                      // exact
    const uint32_t ri = (uint32_t)__double2loint(r + kMagicD);   // r in the low word
    const uint32_t sb = ri + 0x4B400000u;                    // bits of (float)r + kMagic
    const float rf = __uint_as_float(sb) - kMagic;
    if constexpr (m1 == 256) b1[q] = ri;
    else b1[q] = __float_as_uint(fmaf(rf, rm1, kMagic)) * n1 + sb;
    b2[q] = __float_as_uint(fmaf(rf, rm2, kMagic)) * n2 + sb;
  }
  *reinterpret_cast<uint2*>(out + lo * plane) =
      make_uint2(pack4(b1[0], b1[1], b1[2], b1[3]), pack4(b1[4], b1[5], b1[6], b1[7]));
  *reinterpret_cast<uint2*>(out + hi * plane) =
      make_uint2(pack4(b2[0], b2[1], b2[2], b2[3]), pack4(b2[4], b2[5], b2[6], b2[7]));
}
template <int P>
PSD_DEVINL void res_pair_all(const double (&a)[8], int8_t* out, long long plane) {
  if constexpr (P < kNumMod / 2) {
    res_pair_store8<P>(a, out, plane);
    res_pair_all<P + 1>(a, out, plane);
  }
}
static_assert(mod_at(0) == 256 && 256 * mod_at(15) < 65536 && mod_at(1) * mod_at(14) < 65536 &&
                  mod_at(7) * mod_at(8) < 65536, "moduli pairs must multiply below 2^16");

__global__ void __launch_bounds__(256) residues_rows_dp_kernel(const double* __restrict__ x, long long rows,
                                                             long long cols, long long ldx, int* __restrict__ e,
                                                             int8_t* __restrict__ r, long long ldr,
                                                             long long plane) {
  // as residues_rows_kernel (one block per row, pass 1 = row exponent, pass 2 from L2),
  // residues by res_pair_store8
  __shared__ double red[8];
  const long long c4 = cols / 4;
  for (long long i = blockIdx.x; i < rows; i += gridDim.x) {
    const double* row = x + i * ldx;
    double mx = 0.0;
    for (long long k4 = threadIdx.x; k4 < c4; k4 += blockDim.x) {
      const double2 v01 = reinterpret_cast<const double2*>(row)[2 * k4];
      const double2 v23 = reinterpret_cast<const double2*>(row)[2 * k4 + 1];
      mx = fmax(mx, fmax(fmax(fabs(v01.x), fabs(v01.y)), fmax(fabs(v23.x), fabs(v23.y))));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    double t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    __syncthreads();
    const int ei = t > 0.0 ? ilogb(t) + 1 : 0;
    if (threadIdx.x == 0) e[i] = ei;
    const int sh = 53 - ei;
    const double s1 = ldexp(1.0, sh / 2), s2 = ldexp(1.0, sh - sh / 2);
    int8_t* orow = r + i * ldr;
    for (long long k8 = threadIdx.x; k8 < c4 / 2; k8 += blockDim.x) {
      const double2* src = reinterpret_cast<const double2*>(row) + 4 * k8;
      double a[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = __ldcs(src + h);
        a[2 * h] = rint(v.x * s1 * s2);        // |a| < 2^53, exact integer
        a[2 * h + 1] = rint(v.y * s1 * s2);
      }
      res_pair_all<0>(a, orow + 8 * k8, plane);
    }
  }
}

// Single pass: the row maxima come from the symmetry check (sym_stats, kernels_misc.cu),
// so X is read once here (25.8 GB moved at C3 instead of 8.6 + 16.5 read + 17.2 written:
// pass 2 of the two-pass kernels re-reads the row from DRAM — 1184 rows of 256 KB in
// flight exceed L2).
// rowmax_hi[i] = high word of max_j |x_ij|: the exponent is all the row scale needs (a row
// whose maximum is below 2^-1042, i.e. high word 0, is treated as zero, as its entries
// are far below FP64 resolution of any product).
__global__ void __launch_bounds__(256) residues_rows_max_kernel(const double* __restrict__ x, long long rows,
                                                              long long cols, long long ldx,
                                                              const unsigned* __restrict__ rowmax_hi,
                                                              int* __restrict__ e, int8_t* __restrict__ r,
                                                              long long ldr, long long plane) {
  const long long c8 = cols / 8;
  for (long long i = blockIdx.x; i < rows; i += gridDim.x) {
    const unsigned hi = rowmax_hi[i];
    const int ei = hi ? ilogb(__hiloint2double((int)hi, 0)) + 1 : 0;
    if (threadIdx.x == 0) e[i] = ei;
    const int sh = 53 - ei;
    const double s1 = ldexp(1.0, sh / 2), s2 = ldexp(1.0, sh - sh / 2);
    const double* row = x + i * ldx;
    int8_t* orow = r + i * ldr;
    for (long long k8 = threadIdx.x; k8 < c8; k8 += blockDim.x) {
      const double2* src = reinterpret_cast<const double2*>(row) + 4 * k8;
      double a[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = __ldcs(src + h);
        a[2 * h] = rint(v.x * s1 * s2);
        a[2 * h + 1] = rint(v.y * s1 * s2);
      }
      res_pair_all<0>(a, orow + 8 * k8, plane);
    }
  }
}

__global__ void __launch_bounds__(256) residues_rows_kernel(const double* __restrict__ x, long long rows,
                                                          long long cols, long long ldx, int* __restrict__ e,
                                                          int8_t* __restrict__ r, long long ldr,
                                                          long long plane) {
  // One block per row (grid-stride): pass 1 takes the row's max exponent (the row
  // then sits in L2 for pass 2), pass 2 writes the 16 residues of 8 consecutive k
  // per thread, one 64-bit store per modulus (cols % 8 == 0 path).
  // a (signed, |a| < 2^53) = d0 + d1·2^13 + d2·2^26 + d3·2^39 with 13-bit limbs d0..d2 ≥ 0 and
  // signed d3 (|d3| ≤ 2^14); a ≡ s = Σ d_t·p_t, p_t = 2^(13t) mod m taken in (−m/2, m/2], so
  // |s| < 2^22 and s, s + kMagic are exact in fp32.  With q = rint(s/m) from one fma, the
  // residue byte is (bits(s + kMagic) − m·bits(q + kMagic)) mod 256 — one IMAD (the kMagic
  // bit patterns cancel in the low byte).  m = 256 is the low byte of a.
  __shared__ double red[8];
  const long long c4 = cols / 4;
  for (long long i = blockIdx.x; i < rows; i += gridDim.x) {
    const double* row = x + i * ldx;
    double mx = 0.0;
    for (long long k4 = threadIdx.x; k4 < c4; k4 += blockDim.x) {
      const double2 v01 = reinterpret_cast<const double2*>(row)[2 * k4];
      const double2 v23 = reinterpret_cast<const double2*>(row)[2 * k4 + 1];
      mx = fmax(mx, fmax(fmax(fabs(v01.x), fabs(v01.y)), fmax(fabs(v23.x), fabs(v23.y))));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    double t = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
    __syncthreads();
    const int ei = t > 0.0 ? ilogb(t) + 1 : 0;
    if (threadIdx.x == 0) e[i] = ei;
    const int sh = 53 - ei;
    const double s1 = ldexp(1.0, sh / 2), s2 = ldexp(1.0, sh - sh / 2);
    int8_t* orow = r + i * ldr;
    // 8 consecutive k per thread (two 32-bit words per modulus → one 64-bit store)
    for (long long k8 = threadIdx.x; k8 < c4 / 2; k8 += blockDim.x) {
      const double2* src = reinterpret_cast<const double2*>(row) + 4 * k8;
      float f[8][4];
      uint32_t lowb[8];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = __ldcs(src + h);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int q = 2 * h + u;
          const long long a = __double2ll_rn((u ? v.y : v.x) * s1 * s2);
          lowb[q] = (uint32_t)a;
          f[q][0] = u2f_small((uint32_t)a & 8191u);
          f[q][1] = u2f_small((uint32_t)(a >> 13) & 8191u);
          f[q][2] = u2f_small((uint32_t)(a >> 26) & 8191u);
          f[q][3] = u2f_small((uint32_t)((a >> 39) + 16384)) - 16384.0f;
        }
      }
      int8_t* out = orow + 8 * k8;
      *reinterpret_cast<uint2*>(out) =
          make_uint2(pack4(lowb[0], lowb[1], lowb[2], lowb[3]), pack4(lowb[4], lowb[5], lowb[6], lowb[7]));
      res_limb_all<1>(f, out, plane);
    }
  }
}
// scalar fallback (cols % 4 != 0)
__global__ void residues_rows1_kernel(const double* __restrict__ x, long long rows, long long cols,
                                      long long ldx, const int* __restrict__ e, int8_t* __restrict__ r,
                                      long long ldr, long long plane) {
  const long long total = rows * cols;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / cols, k = t % cols;
    const double a = rint(ldexp(__ldcs(x + i * ldx + k), 53 - e[i]));
    int8_t* out = r + i * ldr + k;
#pragma unroll
    for (int l = 0; l < kNumMod; ++l) out[l * plane] = sym_res(mod_pos(a, l), l);
  }
}
// residues of a K×N panel, transposed and column-scaled: R[ℓ][j][k], j < nrows_pad (zero rows j ≥ N)
// Residues of the panel, transposed and column-scaled: R[ℓ][j][k], j < nrows_pad (zero
// rows j ≥ N).  A 32(k) × 32(j) tile is staged through shared memory; thread (j, k4)
// then reduces 4 consecutive k of row j with the 13-bit-limb fp32 arithmetic of
// residues_rows_kernel and stores one 32-bit word per modulus.
__global__ void __launch_bounds__(256) residues_panel_t_kernel(const double* __restrict__ p, long long K, int N,
                                                               long long ldp, const int* __restrict__ f,
                                                               int8_t* __restrict__ r, long long ldr,
                                                               long long plane, int nrows_pad) {
  __shared__ double tile[32][33];
  const long long k0 = (long long)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 × 8
  for (int yy = ty; yy < 32; yy += 8) {
    const long long k = k0 + yy;
    const int j = j0 + tx;
    tile[yy][tx] = (k < K && j < N) ? p[k * ldp + j] : 0.0;
  }
  __syncthreads();
  const int tid = ty * 32 + tx;
  const int jl = tid >> 3, kq = (tid & 7) * 4;        // row j0 + jl, columns k0 + kq .. +3
  const int j = j0 + jl;
  const long long k = k0 + kq;
  if (j >= nrows_pad || k >= K) return;
  const int fj = j < N ? f[j] : 0;
  const int sh = fj > -2000 ? 53 - fj : 0;          // all-zero column: f stays at its fill value
  const double s1 = ldexp(1.0, sh / 2), s2 = ldexp(1.0, sh - sh / 2);
  float fl[4][4];
  uint32_t lowb[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long a = (j < N) ? __double2ll_rn(tile[kq + q][jl] * s1 * s2) : 0;
    lowb[q] = (uint32_t)a;
    fl[q][0] = u2f_small((uint32_t)a & 8191u);
    fl[q][1] = u2f_small((uint32_t)(a >> 13) & 8191u);
    fl[q][2] = u2f_small((uint32_t)(a >> 26) & 8191u);
    fl[q][3] = u2f_small((uint32_t)((a >> 39) + 16384)) - 16384.0f;
  }
  int8_t* out = r + (long long)j * ldr + k;
  const bool full4 = k + 3 < K;
  uint32_t w = pack4(lowb[0], lowb[1], lowb[2], lowb[3]);
  if (full4) {   // common case: immediate-form modulus constants, one 32-bit store per modulus
    *reinterpret_cast<uint32_t*>(out) = w;
    res_limb_all4<1>(fl, out, plane);
    return;
  }
  for (int q = 0; k + q < K; ++q) out[q] = (int8_t)(w >> (8 * q));
#pragma unroll
  for (int l = 1; l < kNumMod; ++l) {
    const float m = c_modf[l], rm = c_rmodf[l];
    const float p1 = c_pow13f[1][l], p2 = c_pow13f[2][l], p3 = c_pow13f[3][l];
    const uint32_t nmi = c_nmod[l];
    uint32_t bq[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float sacc = fmaf(fl[q][3], p3, fmaf(fl[q][2], p2, fmaf(fl[q][1], p1, fl[q][0])));
      if (l == 1) {
        float rr = sym_mod_f(sacc, m, rm);
        rr = rr > 127.5f ? rr - m : rr;
        bq[q] = low_bits(rr);
      } else {
        bq[q] = __float_as_uint(fmaf(sacc, rm, kMagic)) * nmi + __float_as_uint(sacc + kMagic);
      }
    }
    w = pack4(bq[0], bq[1], bq[2], bq[3]);
    for (int q = 0; k + q < K; ++q) out[l * plane + q] = (int8_t)(w >> (8 * q));
  }
}

// ---- INT8 CTA-pair GEMM: residue products mod m_ℓ -------------------------------------
struct I8Params {
  int M, N, K;
  int bn, bn2;              // N of the first MMA (≤ 256) and of the second (0: none); multiples of 16
  int kblocks, kb_per_split, m_pairs, splits;
  int stages;
  uint8_t* out;             // out[((ℓ·splits + split)·M + i)·ldo + col] = (Σ) mod m_ℓ
  long long ldo;
};

PSD_DEVINL void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                 uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
PSD_DEVINL void mma_i8_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
PSD_DEVINL uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1)
    i8_gemm2_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                    const __grid_constant__ CUtensorMap mB2, const I8Params p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full_bar[8], empty_bar[8], acc_bar;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc32::cluster_rank();
  const int bn_tot = p.bn + p.bn2;   // = w rounded to 16: no padded MMA columns
  const int hb = p.bn / 2;
  // modulus slowest: the concurrently running CTAs share one B residue plane (L2-resident)
  int u = blockIdx.x >> 1;
  const int mp = u % p.m_pairs;
  u /= p.m_pairs;
  const int split = u % p.splits;
  const int l = u / p.splits;
  const int m0 = mp * 2 * BM + (int)rank * BM;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kblocks, kb0 + p.kb_per_split) - kb0;
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t a_bytes = BM * BKB, b_bytes = (uint32_t)(bn_tot / 2) * BKB;
  const uint32_t st_bytes = a_bytes + b_bytes;
  const uint32_t tcols = bn_tot <= 256 ? 256 : 512;

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
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc32::tc_fence_before();
  tc32::cluster_sync_all();
  tc32::tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    for (int i = 0; i < nkb; ++i) {
      const int s = i % p.stages;
      const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
      tc32::mbar_wait_t(smem_u32(&empty_bar[s]), ph ^ 1u);
      if (tc32::elect_one()) {
        const uint32_t fb_local = smem_u32(&full_bar[s]);
        const uint32_t fb = tc32::map_to_rank(fb_local, 0);
        if (rank == 0) mbar_expect_tx(fb_local, 2 * st_bytes);
        const uint32_t sA = sbase + s * st_bytes;
        const uint32_t sB = sA + a_bytes;
        const int kc = (kb0 + i) * BKB;
        tma_load_3d_pair(sA, &mA, kc, m0, l, fb);
        tma_load_3d_pair(sB, &mB, kc, (int)rank * hb, l, fb);
        if (p.bn2) tma_load_3d_pair(sB + (uint32_t)hb * BKB, &mB2, kc, p.bn + (int)rank * (p.bn2 / 2), l, fb);
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // kind::i8: D s32 (2), A/B signed int8 (1), K-major, M = 256, N = bn
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.bn >> 3) << 17) |
                             ((uint32_t)(2 * BM >> 4) << 24);
      const uint64_t da = desc_sw128(sbase), db = desc_sw128(sbase + a_bytes);
      const uint32_t idesc2 = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.bn2 >> 3) << 17) |
                              ((uint32_t)(2 * BM >> 4) << 24);
      const uint32_t b_half = (uint32_t)(hb * BKB) >> 4;
      const bool two = p.bn2 > 0;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (uint32_t)(i / p.stages) & 1u;
        tc32::mbar_wait_t(smem_u32(&full_bar[s]), ph);
        tc32::tc_fence_after();
        if (tc32::elect_one()) {
          const uint32_t so = (uint32_t)(s * st_bytes) >> 4;
#pragma unroll
          for (int kk = 0; kk < BKB / 32; ++kk) {   // 32 int8 K per MMA = 32 bytes
            const uint64_t a = da + so + kk * 2, b = db + so + kk * 2;
            const uint32_t acc0 = (i | kk) != 0;
            mma_i8_pair(tmem, a, b, idesc, acc0);
            if (two) mma_i8_pair(tmem + (uint32_t)p.bn, a, b + b_half, idesc2, acc0);
          }
          tc32::mma_commit_pair(smem_u32(&empty_bar[s]));
          if (i == nkb - 1) tc32::mma_commit_pair(smem_u32(&acc_bar));
        }
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int i = m0 + quad * 32 + lane;
    tc32::mbar_wait_t(smem_u32(&acc_bar), 0);
    tc32::tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    // |Σ| ≤ K_split·2^14 ≤ 2^29: Σ = hi·2^15 + lo, s = hi·(2^15 mod m) + lo (|s| < 2^23),
    // stored as a signed int8 representative of Σ mod m (m = 256: the low byte).
    const float m = c_modf[l], rm = c_rmodf[l];
    const float c15 = (float)(32768 % c_mod[l]);
    uint8_t* orow = p.out + (((long long)l * p.splits + split) * p.M + i) * p.ldo;
    for (int c0 = 0; c0 < bn_tot; c0 += 16) {
      float v[16];
      tc32::tmem_ld16(trow + (uint32_t)c0, v);
      if (i >= p.M) continue;
      uint32_t b[16];
      if (l == 0) {
#pragma unroll
        for (int e = 0; e < 16; ++e) b[e] = __float_as_uint(v[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int sv = __float_as_int(v[e]);
          const float hf = u2f_small((uint32_t)((sv >> 15) + 32768)) - 32768.0f;
          const float lf = u2f_small((uint32_t)sv & 32767u);
          float rr = sym_mod_f(fmaf(hf, c15, lf), m, rm);
          rr = rr > 127.5f ? rr - m : rr;
          b[e] = low_bits(rr);
        }
      }
      uint32_t w4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w4[q] = pack4(b[4 * q], b[4 * q + 1], b[4 * q + 2], b[4 * q + 3]);
      *reinterpret_cast<uint4*>(orow + c0) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
  }
  tc32::tc_fence_before();
  tc32::cluster_sync_all();
  if (warp == 1) {
    tc32::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tcols) : "memory");
  }
}

// ---- CRT reconstruction + scaling ----------------------------------------------------
// C[i][j] = C'·2^(e_i + f_j − 106), C' the symmetric residue of the product mod M:
//   y_ℓ = (Σ_split out[ℓ][s][i][j])·(M/m_ℓ)^{-1} mod m_ℓ,   S = Σ_ℓ y_ℓ·(M/m_ℓ),
//   S/M = Σ_ℓ y_ℓ/m_ℓ  →  k = rint(Σ_ℓ y_ℓ/m_ℓ) (fp32, error ≲ 2^-18: |C'|/M ≤
//   K·2^-19.4 — 0.19 at K = 2^17 (C4), 0.38 at the K ≤ 2^18 limit — stays below ½),
//   C' = S − k·M evaluated mod 2^128 (|C'| < 2^127, so the wrapped value is exact).
// Four columns per thread (ldo % 4 == 0; columns ≥ N are padding and not stored).
// alpha > 0: C = (C + α·S)/α (the shifted sketch of Alg. 3).
template <bool ONE>   // ONE: a single K split (all 16 plane words loaded up front)
__global__ void __launch_bounds__(256) crt_kernel(const uint8_t* __restrict__ res, int splits, long long M, int N,
                                                  long long ldo, const int* __restrict__ e,
                                                  const int* __restrict__ f, double* __restrict__ C, long long ldc,
                                                  double alpha, const double* __restrict__ S, long long lds) {
  const int n4 = (N + 3) / 4;
  const long long total = M * n4;
  const long long plane = M * ldo;
  const unsigned __int128 Mfull = ((unsigned __int128)c_M[1] << 64) | c_M[0];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n4;
    const int j0 = (int)(t % n4) * 4;
    const uint8_t* base = res + i * ldo + j0;
    uint32_t wv[kNumMod];
    if (ONE) {
#pragma unroll
      for (int l = 0; l < kNumMod; ++l) wv[l] = __ldcs(reinterpret_cast<const uint32_t*>(base + l * plane));
    }
    float ks[4] = {0.f, 0.f, 0.f, 0.f};
    unsigned __int128 acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int l = 0; l < kNumMod; ++l) {
      int sum[4] = {0, 0, 0, 0};
      if (ONE) {
#pragma unroll
        for (int q = 0; q < 4; ++q) sum[q] = (int)(int8_t)(wv[l] >> (8 * q));
      } else {
        for (int sp = 0; sp < splits; ++sp) {
          const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(base + ((long long)l * splits + sp) * plane));
#pragma unroll
          for (int q = 0; q < 4; ++q) sum[q] += (int)(int8_t)(w >> (8 * q));
        }
      }
      const float m = c_modf[l], rm = c_rmodf[l], winv = c_wInvf[l];
      const unsigned __int128 W = ((unsigned __int128)c_W[l][1] << 64) | c_W[l][0];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float sf = __int_as_float(sum[q] + 0x4B400000) - kMagic;   // exact: |sum| < 2^22
        float y = sym_mod_f(sf * winv, m, rm);                          // |sum·winv| < 2^19: exact
        y = y < 0.f ? y + m : y;                                         // y ∈ [0, m]
        ks[q] = fmaf(y, rm, ks[q]);
        const uint32_t yi = __float_as_uint(y + kMagic) - 0x4B400000u;
        acc[q] += W * yi;
      }
    }
    const int ei = e[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j >= N) break;
      const unsigned __int128 kM = Mfull * (unsigned)(int)rintf(ks[q]);
      const unsigned __int128 cs = acc[q] - kM;           // two's complement of C'
      const bool neg = (long long)(cs >> 64) < 0;
      const unsigned __int128 mag = neg ? (unsigned __int128)0 - cs : cs;
      const unsigned long long hi = (unsigned long long)(mag >> 64), lo = (unsigned long long)mag;
      double val = fma((double)hi, 18446744073709551616.0, (double)lo);
      if (neg) val = -val;
      const int ex = ei + f[j] - 106;
      if (ex > -1000 && ex < 1000) val *= __longlong_as_double((long long)(ex + 1023) << 52);   // exact 2^ex
      else val = ldexp(val, ex);
      if (alpha > 0.0) val = (val + alpha * S[i * lds + j]) / alpha;
      C[i * ldc + j] = val;
    }
  }
}

// Single-split CRT (the n×w products) with the per-modulus arithmetic moved into tables
// and exact integer limbs — the float path above spends ≈20 instructions per (modulus,
// column) on the residue → y_ℓ step and a 128-bit multiply-accumulate, which made the kernel
// issue-bound (ncu: 70% issue slots, not_selected the top stall):
//   y_ℓ = T_ℓ[b]                     one LDS.U8 (b = the stored residue byte)
//   κ  += y_ℓ·⌊2^27/m_ℓ⌉             k = rint(Σ y_ℓ/m_ℓ) in 5.27 fixed point: the rounding
//                                     of the 16 weights costs ≤ 16·255·2^-28 < 2^-14
//   s_t += y_ℓ·w_ℓt (t = 0..3)       the 32-bit limbs of M/m_ℓ; s_t < 16·2^8·2^32 = 2^44, so
//                                     four IMAD.WIDE per term and one carry pass per output
// then C' = Σ s_t·2^(32t) − k·M mod 2^128 exactly as before.
template <int L>
__host__ __device__ constexpr uint32_t kwt() { return (uint32_t)((134217728.0 / mod_at(L)) + 0.5); }   // ⌊2^27/m⌉

__global__ void __launch_bounds__(256, 3) crt1_kernel(const uint8_t* __restrict__ res, long long M, int N, long long ldo,
                                                   const int* __restrict__ e, const int* __restrict__ f,
                                                   double* __restrict__ C, long long ldc, double alpha,
                                                   const double* __restrict__ S, long long lds) {
  __shared__ uint32_t ty32[kNumMod * 64];
  for (int i = threadIdx.x; i < kNumMod * 64; i += blockDim.x) ty32[i] = g_ytab[i];
  __syncthreads();
  const uint8_t* ty = reinterpret_cast<const uint8_t*>(ty32);
  const int n4 = (N + 3) / 4;
  const long long total = M * n4;
  const long long plane = M * ldo;
  const unsigned __int128 Mfull = ((unsigned __int128)c_M[1] << 64) | c_M[0];
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = t / n4;
    const int j0 = (int)(t % n4) * 4;
    const uint8_t* base = res + i * ldo + j0;
    uint32_t wv[kNumMod];
#pragma unroll
    for (int l = 0; l < kNumMod; ++l) wv[l] = __ldcs(reinterpret_cast<const uint32_t*>(base + l * plane));
    unsigned long long s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0}, s2[4] = {0, 0, 0, 0}, s3[4] = {0, 0, 0, 0};
    uint32_t kap[4] = {0u, 0u, 0u, 0u};
    auto term = [&](auto lc) {
      constexpr int l = decltype(lc)::value;
      const uint32_t w0 = (uint32_t)c_W[l][0], w1 = (uint32_t)(c_W[l][0] >> 32);
      const uint32_t w2 = (uint32_t)c_W[l][1], w3 = (uint32_t)(c_W[l][1] >> 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t y = ty[l * 256 + ((wv[l] >> (8 * q)) & 255u)];
        kap[q] += y * kwt<l>();
        s0[q] += (unsigned long long)y * w0;
        s1[q] += (unsigned long long)y * w1;
        s2[q] += (unsigned long long)y * w2;
        s3[q] += (unsigned long long)y * w3;
      }
    };
    [&]<int... Ls>(std::integer_sequence<int, Ls...>) {
      (term(std::integral_constant<int, Ls>{}), ...);
    }(std::make_integer_sequence<int, kNumMod>{});
    const int ei = e[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j >= N) break;
      const unsigned k = (kap[q] + (1u << 26)) >> 27;
      const unsigned __int128 acc = (unsigned __int128)s0[q] + ((unsigned __int128)s1[q] << 32) +
                                    ((unsigned __int128)s2[q] << 64) + ((unsigned __int128)s3[q] << 96);
      const unsigned __int128 cs = acc - Mfull * k;        // two's complement of C'
      const bool neg = (long long)(cs >> 64) < 0;
      const unsigned __int128 mag = neg ? (unsigned __int128)0 - cs : cs;
      const unsigned long long hi = (unsigned long long)(mag >> 64), lo = (unsigned long long)mag;
      double val = fma((double)hi, 18446744073709551616.0, (double)lo);
      if (neg) val = -val;
      const int ex = ei + f[j] - 106;
      if (ex > -1000 && ex < 1000) val *= __longlong_as_double((long long)(ex + 1023) << 52);   // exact 2^ex
      else val = ldexp(val, ex);
      if (alpha > 0.0) val = (val + alpha * S[i * lds + j]) / alpha;
      C[i * ldc + j] = val;
    }
  }
}

}  // namespace oz

namespace {

void ensure_oz_constants() {
  static bool done[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (done[dev]) return;
  int mods[oz::kNumMod];
  double rm[oz::kNumMod];
  float rmf[oz::kNumMod];
  int inv[oz::kNumMod][oz::kNumMod] = {};
  for (int l = 0; l < oz::kNumMod; ++l) {
    mods[l] = oz::kMods[l];
    rm[l] = 1.0 / oz::kMods[l];
    rmf[l] = 1.0f / (float)oz::kMods[l];
  }
  for (int i = 0; i < oz::kNumMod; ++i)
    for (int j = i + 1; j < oz::kNumMod; ++j) {
      const int a = oz::kMods[i] % oz::kMods[j], m = oz::kMods[j];
      int x = 1;
      while ((a * x) % m != 1) ++x;
      inv[i][j] = x;
    }
  cudaMemcpyToSymbol(oz::c_mod, mods, sizeof(mods));
  cudaMemcpyToSymbol(oz::c_rmod, rm, sizeof(rm));
  cudaMemcpyToSymbol(oz::c_rmodf, rmf, sizeof(rmf));
  cudaMemcpyToSymbol(oz::c_inv, inv, sizeof(inv));
  unsigned __int128 M = 1;
  for (int l = 0; l < oz::kNumMod; ++l) M *= (unsigned)oz::kMods[l];
  const unsigned long long Mh[2] = {(unsigned long long)M, (unsigned long long)(M >> 64)};
  cudaMemcpyToSymbol(oz::c_M, Mh, sizeof(Mh));
  float modf[oz::kNumMod], pw[4][oz::kNumMod], winv[oz::kNumMod];
  unsigned long long W[oz::kNumMod][2];
  for (int l = 0; l < oz::kNumMod; ++l) {
    const int m = oz::kMods[l];
    modf[l] = (float)m;
    long long v = 1;
    for (int t = 0; t < 4; ++t) {
      const long long r = v % m;
      pw[t][l] = (float)(r > m / 2 ? r - m : r);
      v = (v * 8192) % m;
    }
    const unsigned __int128 w = M / (unsigned)m;
    W[l][0] = (unsigned long long)w;
    W[l][1] = (unsigned long long)(w >> 64);
    const int wm = (int)(w % (unsigned)m);
    int x = 1;
    while ((wm * x) % m != 1) ++x;
    winv[l] = (float)x;
  }
  cudaMemcpyToSymbol(oz::c_modf, modf, sizeof(modf));
  uint32_t nmod[oz::kNumMod];
  for (int l = 0; l < oz::kNumMod; ++l) nmod[l] = 0u - (uint32_t)oz::kMods[l];
  cudaMemcpyToSymbol(oz::c_nmod, nmod, sizeof(nmod));
  cudaMemcpyToSymbol(oz::c_pow13f, pw, sizeof(pw));
  cudaMemcpyToSymbol(oz::c_wInvf, winv, sizeof(winv));
  {
    uint8_t ytab[oz::kNumMod][256];
    for (int l = 0; l < oz::kNumMod; ++l) {
      const int m = oz::kMods[l], wi = (int)winv[l];
      for (int b = 0; b < 256; ++b) ytab[l][b] = (uint8_t)((((int)(int8_t)b * wi) % m + m) % m);
    }
    cudaMemcpyToSymbol(oz::g_ytab, ytab, sizeof(ytab));
  }
  cudaMemcpyToSymbol(oz::c_W, W, sizeof(W));
  // the copies are ordered on the legacy stream only: complete them before kernels on
  // non-blocking streams read the constants
  cudaDeviceSynchronize();
  done[dev] = true;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_oz() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r) == cudaSuccess &&
        r == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(q);
  });
  return fn;
}

// int8 planes [L][rows][ld]: box = 128 bytes of K × box_rows × 1 plane, SWIZZLE_128B
bool map_i8_3d(CUtensorMap* map, const int8_t* ptr, long long cols, long long rows, long long ld,
               long long planes, int box_rows) {
  auto fn = encode_oz();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)(ld * rows)};
  cuuint32_t box[3] = {(cuuint32_t)oz::BKB, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int grid_oz(long long total, int threads) {
  return (int)std::min<long long>(std::max<long long>((total + threads - 1) / threads, 1),
                                  (long long)device_info().sms * 16);
}

}  // namespace

int oz_num_moduli() { return oz::kNumMod; }
long long oz_max_k() { return oz::kMaxK; }

void oz_prepare_rows_max(const double* x, long long rows, long long cols, long long ldx,
                         const unsigned* rowmax, int* e, int8_t* r, long long ldr, cudaStream_t st,
                         long long grid_req, int threads) {
  ensure_oz_constants();
  if (cols % 8 == 0 && ldx % 2 == 0 && ldr % 8 == 0 && (uintptr_t)x % 16 == 0) {
    const unsigned grid = (unsigned)std::min<long long>(rows, grid_req > 0 ? grid_req : (long long)device_info().sms * 8);
    // threads < 256 (side-stream use): smaller CTAs pack beside the caller's register-heavy kernels
    const unsigned block = (unsigned)std::min(256, std::max(32, threads / 32 * 32));
    oz::residues_rows_max_kernel<<<grid, block, 0, st>>>(x, rows, cols, ldx, rowmax, e, r, ldr, ldr * rows);
    count_launch();
  } else {
    oz_prepare_rows(x, rows, cols, ldx, e, r, ldr, st);
  }
}

void oz_prepare_rows(const double* x, long long rows, long long cols, long long ldx, int* e, int8_t* r,
                     long long ldr, cudaStream_t st) {
  ensure_oz_constants();
  if (cols % 8 == 0 && ldx % 2 == 0 && ldr % 8 == 0 && (uintptr_t)x % 16 == 0) {
    // row exponents fused: one block per row.  Residues by paired moduli on the FP64 pipe
    // (PSD_OZ_RES=limb keeps the 13-bit-limb fp32 form)
    static const bool limb = [] { const char* v = getenv("PSD_OZ_RES"); return v && v[0] == 'l'; }();
    const unsigned grid = (unsigned)std::min<long long>(rows, (long long)device_info().sms * 8);
    if (limb)
      oz::residues_rows_kernel<<<grid, 256, 0, st>>>(x, rows, cols, ldx, e, r, ldr, ldr * rows);
    else
      oz::residues_rows_dp_kernel<<<grid, 256, 0, st>>>(x, rows, cols, ldx, e, r, ldr, ldr * rows);
    count_launch();
  } else {
    oz::row_exp_kernel<<<(unsigned)rows, 256, 0, st>>>(x, rows, cols, ldx, e);
    count_launch();
    oz::residues_rows1_kernel<<<grid_oz(rows * cols, 256), 256, 0, st>>>(x, rows, cols, ldx, e, r, ldr,
                                                                          ldr * rows);
    count_launch();
  }
}

// B = the panel P (K×N): column exponents and transposed residues into op.f / op.br.
int oz_prepare_panel(const OzOp& op, cudaStream_t st) {
  using namespace oz;
  ensure_oz_constants();
  if (op.N < 1 || op.K < 1) return 0;
  const int w_pad = (op.N + 15) / 16 * 16;
  if (w_pad > 512 || op.ldbr < op.K || op.ldbr % 16) return -2;
  cudaMemsetAsync(op.f, 0x80, (size_t)op.N * sizeof(int), st);   // very negative → atomicMax
  {
    dim3 grid((unsigned)std::min<long long>((op.K + 7) / 8, 256), (unsigned)((op.N + 31) / 32));
    col_exp_kernel<<<grid, 256, 0, st>>>(op.P, op.K, op.N, op.ldp, op.f);
    count_launch();
  }
  {
    dim3 grid((unsigned)((op.K + 31) / 32), (unsigned)((w_pad + 31) / 32));
    residues_panel_t_kernel<<<grid, dim3(32, 8), 0, st>>>(op.P, op.K, op.N, op.ldp, op.f, op.br, op.ldbr,
                                                          op.ldbr * w_pad, w_pad);
    count_launch();
  }
  return 0;
}

// The 16 residue GEMMs + CRT for prepared A (op.ar / op.e) and B (op.br / op.f).
int oz_gemm_prepared(const OzOp& op, cudaStream_t st) {
  using namespace oz;
  ensure_oz_constants();
  if (op.M < 1 || op.N < 1 || op.K < 1) return 0;
  if (op.K > kMaxK) return -4;
  const int w_pad = (op.N + 15) / 16 * 16;
  if (w_pad > 512 || op.ldbr < op.K || op.ldbr % 16 || op.ldar % 16) return -2;
  I8Params p{};
  p.M = op.M;
  p.N = op.N;
  p.K = op.K;
  // two balanced MMAs when w > 256 (e.g. 272 = 144 + 128): no padded columns, and
  // a tiny second MMA (256 + 16) measured slower than the pair of ~equal halves
  static const int nsplit = [] { const char* e = getenv("PSD_OZ_NSPLIT"); return e ? atoi(e) : 1; }();
  p.bn = w_pad <= 256 ? w_pad : (w_pad / 2 + 15) / 16 * 16;
  p.bn2 = w_pad - p.bn;
  if (w_pad > 256 && nsplit == 0) p.bn2 = p.bn;          // padded equal halves (288 for 272)
  if (w_pad > 256 && nsplit == 2) { p.bn = 256; p.bn2 = w_pad - 256; }
  const int bn_tot = p.bn + p.bn2;
  p.kblocks = (op.K + BKB - 1) / BKB;
  p.m_pairs = (op.M + 2 * BM - 1) / (2 * BM);
  const int slots = device_info().sms / 2;
  const long long base = (long long)p.m_pairs * kNumMod;
  // unit time ≈ T/s + c (setup, pipeline fill, epilogue; c ≈ 2% of a full-K unit at K = 32k);
  // the epilogue bound |Σ| ≤ 2^29 needs K per split ≤ 32768.
  const int min_splits = (p.kblocks + 255) / 256;
  int splits = min_splits;
  double best = 1e30;
  for (int s = min_splits; s <= std::max(8, min_splits) && s <= p.kblocks; ++s) {
    const double t = (double)((base * s + slots - 1) / slots) * (p.kblocks / 256.0 / s + 0.02);
    if (t < best - 1e-9) {
      best = t;
      splits = s;
    }
  }
  while (splits > min_splits && (size_t)kNumMod * splits * op.M * bn_tot > op.res_elems) --splits;
  if ((size_t)kNumMod * splits * op.M * bn_tot > op.res_elems) return -3;
  p.kb_per_split = (p.kblocks + splits - 1) / splits;
  p.splits = (p.kblocks + p.kb_per_split - 1) / p.kb_per_split;
  p.out = op.res;
  p.ldo = bn_tot;
  const int sb = BM * BKB + bn_tot / 2 * BKB;
  p.stages = std::min(8, ((int)device_info().max_smem - 3072) / sb);
  const size_t smem = (size_t)p.stages * sb + 1024;
  CUtensorMap ma, mb, mb2;
  if (!map_i8_3d(&ma, op.ar, op.K, op.ar_rows ? op.ar_rows : op.M, op.ldar, kNumMod, BM) ||
      !map_i8_3d(&mb, op.br, op.K, w_pad, op.ldbr, kNumMod, p.bn / 2) ||
      !map_i8_3d(&mb2, op.br, op.K, w_pad, op.ldbr, kNumMod, std::max(p.bn2, 16) / 2))
    return -5;
  static size_t attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr[dev] < smem) {
    cudaFuncSetAttribute(i8_gemm2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dev] = smem;
  }
  const long long units = base * p.splits;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * units));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr2[1];
  attr2[0].id = cudaLaunchAttributeClusterDimension;
  attr2[0].val.clusterDim.x = 2;
  attr2[0].val.clusterDim.y = 1;
  attr2[0].val.clusterDim.z = 1;
  cfg.attrs = attr2;
  cfg.numAttrs = 1;
  if (op.ev_gemm[0]) cudaEventRecord(op.ev_gemm[0], st);
  if (cudaLaunchKernelEx(&cfg, i8_gemm2_kernel, ma, mb, mb2, p) != cudaSuccess) return -6;
  if (op.ev_gemm[1]) cudaEventRecord(op.ev_gemm[1], st);
  count_launch();
  {
    const unsigned g = (unsigned)grid_oz((long long)op.M * ((op.N + 3) / 4), 256);
    static const bool crt_float = [] { const char* v = getenv("PSD_OZ_CRT"); return v && v[0] == 'f'; }();
    if (p.splits == 1 && !crt_float)
      crt1_kernel<<<g, 256, 0, st>>>(op.res, op.M, op.N, p.ldo, op.e, op.f, op.C, op.ldc, op.alpha, op.S, op.lds);
    else if (p.splits == 1)
      crt_kernel<true><<<g, 256, 0, st>>>(op.res, 1, op.M, op.N, p.ldo, op.e, op.f, op.C, op.ldc, op.alpha,
                                          op.S, op.lds);
    else
      crt_kernel<false><<<g, 256, 0, st>>>(op.res, p.splits, op.M, op.N, p.ldo, op.e, op.f, op.C, op.ldc,
                                           op.alpha, op.S, op.lds);
  }
  count_launch();
  return p.splits;
}

int oz_gemm(const OzOp& op, cudaStream_t st) {
  const int r = oz_prepare_panel(op, st);
  if (r < 0) return r;
  return oz_gemm_prepared(op, st);
}

// Workspace layout of oz_gemm_stream (bytes, 256-aligned pieces).  Panels wider
// than 512 columns (the TMEM budget) are cut into G column groups of ≤ 512.
struct OzStreamLayout {
  long long ldk, groups, gw, gw_pad, chunk;
  size_t ar, br, e, f, res, total;
};
static OzStreamLayout oz_stream_layout(long long m, long long n, long long k, long long chunk) {
  OzStreamLayout L{};
  L.ldk = (k + 127) / 128 * 128;
  L.groups = (n + 511) / 512;
  L.gw = (n + L.groups - 1) / L.groups;
  L.gw_pad = (L.gw + 15) / 16 * 16;
  L.chunk = std::max<long long>(1, std::min(m, chunk));
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const int nm = oz::kNumMod;
  const long long splits = std::max<long long>(8, (k + 32767) / 32768 + 1);
  L.ar = al((size_t)nm * L.chunk * L.ldk);
  L.br = al((size_t)nm * L.gw_pad * L.ldk) * L.groups;
  L.e = al((size_t)L.chunk * sizeof(int));
  L.f = al((size_t)L.gw_pad * sizeof(int)) * L.groups;
  L.res = al((size_t)nm * splits * L.chunk * L.gw_pad);
  L.total = L.ar + L.br + L.e + L.f + L.res;
  return L;
}

size_t oz_stream_ws_bytes(long long m, long long n, long long k, long long chunk) {
  return oz_stream_layout(m, n, k, chunk).total;
}

// C (M×N) = A·P (A any M×K fp64 matrix, row-major) — or (A·P + α·S)/α — with A
// streamed in row chunks: residues of a chunk, then for each ≤512-column group of
// the panel its 16 GEMMs and CRT; the panel groups are prepared once.
int oz_gemm_stream(const double* a, long long lda, const double* P, long long ldp, long long m, int n,
                   long long k, double* c, long long ldc, double alpha, const double* S, long long lds,
                   void* ws, size_t ws_bytes, long long chunk, cudaStream_t st) {
  if (k > oz::kMaxK) return -4;
  const OzStreamLayout L = oz_stream_layout(m, n, k, chunk);
  if (ws_bytes < L.total) return -3;
  uint8_t* base = static_cast<uint8_t*>(ws);
  int8_t* ar = reinterpret_cast<int8_t*>(base);
  uint8_t* br0 = base + L.ar;
  int* e = reinterpret_cast<int*>(base + L.ar + L.br);
  uint8_t* f0 = base + L.ar + L.br + L.e;
  uint8_t* res = base + L.ar + L.br + L.e + L.f;
  const size_t br_g = L.br / L.groups, f_g = L.f / L.groups;
  // K padding of both residue buffers stays zero
  cudaMemsetAsync(base, 0, L.ar + L.br, st);
  std::vector<OzOp> ops((size_t)L.groups);
  for (long long g = 0; g < L.groups; ++g) {
    OzOp& op = ops[(size_t)g];
    const long long c0 = g * L.gw;
    op.ar = ar;
    op.ldar = L.ldk;
    op.e = e;
    op.br = reinterpret_cast<int8_t*>(br0 + g * br_g);
    op.ldbr = L.ldk;
    op.f = reinterpret_cast<int*>(f0 + g * f_g);
    op.res = res;
    op.res_elems = L.res;
    op.P = P + c0;
    op.ldp = ldp;
    op.N = (int)std::min<long long>(L.gw, n - c0);
    op.K = (int)k;
    op.alpha = alpha;
    const int r = oz_prepare_panel(op, st);
    if (r < 0) return r;
  }
  for (long long r0 = 0; r0 < m; r0 += L.chunk) {
    const long long rows = std::min(L.chunk, m - r0);
    oz_prepare_rows(a + r0 * lda, rows, k, lda, e, ar, L.ldk, st);
    for (long long g = 0; g < L.groups; ++g) {
      OzOp& op = ops[(size_t)g];
      const long long c0 = g * L.gw;
      op.M = (int)rows;
      op.C = c + r0 * ldc + c0;
      op.ldc = ldc;
      op.S = S ? S + r0 * lds + c0 : nullptr;
      op.lds = lds;
      const int r = oz_gemm_prepared(op, st);
      if (r < 0) return r;
    }
  }
  return 0;
}

}  // namespace psd
