// Memory-bound kernels of the projection path (HBM roofline): symmetry
// validation, Gaussian test-matrix generation, the power-iteration GEMV,
// split-K reduction and small panel utilities.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "launch.h"

namespace psd {

// ---------------------------------------------------------------------------
// a1 — require_symmetric (symmetric.py:39-57).  One pass over (I,J)/(J,I)
// 32×32 tile pairs (I ≤ J): max|x|, max|x − xᵀ| and "bitwise symmetric".
// ---------------------------------------------------------------------------
constexpr int kSymT = 64;
#ifndef PSD_SYM_MINB
#define PSD_SYM_MINB 3   // blocks per SM the register budget is cut for (4: 64 regs, spills with row maxima)
#endif

// Persistent blocks walk the lower-triangular list of 64×64 tile pairs
// (I ≥ J): tile (J,I) is staged transposed through shared memory, tile (I,J)
// is read straight into registers, so every element of X is read once
// (diagonal tiles twice).  One atomic per block per statistic at the end.
// rowmax != nullptr: also the HIGH WORD of max_j |x_ij| per row i (non-negative doubles
// order like their bit patterns; the high word carries the exponent, all the INT8
// engine's residue pass needs for its row scale — ozaki.cu — so that pass reads X once
// instead of twice).  One REDUX.MAX per tile row and warp, one 32-bit atomic per tile
// row; zeroed by the caller.
template <typename T>
__global__ void __launch_bounds__(256, PSD_SYM_MINB) sym_stats_kernel(const T* __restrict__ x, long long n,
                                                        long long ldx, long long npairs,
                                                        double* stats, unsigned* __restrict__ rowmax,
                                                        int diag) {
  __shared__ T tj[kSymT][kSymT + 1];
  __shared__ unsigned rred[8][kSymT];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
  double mabs = 0.0, mdef = 0.0;
  unsigned diffbits = 0u, hmax = 0u;   // FP64: bitwise-difference and |x| high-word accumulators
  int flags = 0;
  const long long nt = (n + kSymT - 1) / kSymT;
  for (long long b = blockIdx.x; b < npairs; b += gridDim.x) {
    // diag: diagonal-major order — pair b lies on diagonal d = ti − tjx, which starts at
    // o(d) = d·nt − d(d−1)/2; concurrently running blocks then hold distinct row blocks,
    // so the row-maximum atomics below do not pile onto the same addresses.
    long long ti, tjx;
    if (diag) {
      const double fn = (double)nt + 0.5;
      long long d = (long long)(fn - sqrt(fmax(fn * fn - 2.0 * (double)b, 0.0)));
      while (d > 0 && d * nt - d * (d - 1) / 2 > b) --d;
      while ((d + 1) * nt - (d + 1) * d / 2 <= b) ++d;
      tjx = b - (d * nt - d * (d - 1) / 2);
      ti = tjx + d;
    } else {   // row-major over the lower triangle
      ti = (long long)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
      while ((ti + 1) * (ti + 2) / 2 <= b) ++ti;
      while (ti * (ti + 1) / 2 > b) --ti;
      tjx = b - ti * (ti + 1) / 2;
    }
    const long long r0 = ti * kSymT, c0 = tjx * kSymT;
    T a[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        // x[c0 + r][r0 + c] → smem (tile (J, I)); x[r0 + r][c0 + c] → registers (tile (I, J))
        const long long gr = c0 + r, gc = r0 + c;
        tj[r][c] = (gr < n && gc < n) ? __ldcs(x + gr * ldx + gc) : T(0);
        const long long ar = r0 + r, ac = c0 + c;
        a[q][h] = (ar < n && ac < n) ? __ldcs(x + ar * ldx + ac) : T(0);
      }
    }
    __syncthreads();
    // compute: defect / max|x| / flags; with rowmax also the row maxima — rows r0 + r from the
    // register tile (one REDUX across the lanes per q), rows c0 + c from the values this thread
    // reads transposed out of smem (max over q in registers, then over the 8 warps in smem)
    unsigned bm[2] = {0u, 0u};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        const double av = (double)a[q][h];
        const double bt = (double)tj[c][r];  // x[c0 + c][r0 + r] = x[j][i]
        mabs = fmax(mabs, fmax(fabs(av), fabs(bt)));
        mdef = fmax(mdef, fabs(av - bt));
        if constexpr (sizeof(T) == 8) {
          // integer side of the checks (off the FP64 pipe): bitwise equality from the bit
          // patterns, non-finite from the largest |x| high word (≥ 0x7ff00000 ⇔ Inf/NaN)
          const unsigned ahi = (unsigned)__double2hiint(av), bhi = (unsigned)__double2hiint(bt);
          diffbits |= ((unsigned)__double2loint(av) ^ (unsigned)__double2loint(bt)) | (ahi ^ bhi);
          hmax = max(hmax, max(ahi & 0x7fffffffu, bhi & 0x7fffffffu));
          if (rowmax != nullptr) bm[h] = max(bm[h], bhi & 0x7fffffffu);
        } else {
          if (!isfinite(av) || !isfinite(bt)) flags |= 2;
          if (av != bt) flags |= 1;
          if (rowmax != nullptr) bm[h] = max(bm[h], (unsigned)__double2hiint(fabs(bt)));
        }
      }
      if (rowmax != nullptr && r0 != c0) {
        const unsigned mi = __reduce_max_sync(
            0xffffffffu, (unsigned)__double2hiint(fmax(fabs((double)a[q][0]), fabs((double)a[q][1]))));
        if (tx == 0 && r0 + r < n && mi) atomicMax(&rowmax[r0 + r], mi);
      }
    }
    if (rowmax != nullptr) {
      rred[ty][tx] = bm[0];
      rred[ty][tx + 32] = bm[1];
    }
    __syncthreads();
    if (rowmax != nullptr && threadIdx.x < kSymT) {
      unsigned m = rred[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < 8; ++w) m = max(m, rred[w][threadIdx.x]);
      if (c0 + threadIdx.x < n && m) atomicMax(&rowmax[c0 + threadIdx.x], m);
    }
    __syncthreads();
  }
  if (diffbits) flags |= 1;
  if (hmax >= 0x7ff00000u) flags |= 2;
  __shared__ double rmax[8], rdef[8];
  __shared__ int rfl[8];
  mabs = warp_max(mabs);
  mdef = warp_max(mdef);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (tx == 0) {
    rmax[ty] = mabs;
    rdef[ty] = mdef;
    rfl[ty] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m1 = 0.0, m2 = 0.0;
    int f = 0;
    for (int w = 0; w < 8; ++w) {
      m1 = fmax(m1, rmax[w]);
      m2 = fmax(m2, rdef[w]);
      f |= rfl[w];
    }
    if (m1 > 0.0) atomic_max_nonneg(&stats[0], m1);
    if (m2 > 0.0) atomic_max_nonneg(&stats[1], m2);
    if (f) atomicOr(reinterpret_cast<int*>(stats + 2), f);
  }
}

template <typename T>
static void sym_stats_t(const T* x, long long n, long long ldx, double* stats, unsigned* rowmax,
                        cudaStream_t st, long long grid = 0) {
  cudaMemsetAsync(stats, 0, 3 * sizeof(double), st);
  if (rowmax) cudaMemsetAsync(rowmax, 0, (size_t)n * sizeof(unsigned), st);
  const long long nt = (n + kSymT - 1) / kSymT;
  const long long npairs = nt * (nt + 1) / 2;
  const long long blocks = std::min<long long>(npairs, grid > 0 ? grid : (long long)device_info().sms * PSD_SYM_MINB * 2);
  static const int diag = [] { const char* e = getenv("PSD_SYM_ORDER"); return e && e[0] == 'd' ? 1 : 0; }();
  sym_stats_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(x, n, ldx, npairs, stats, rowmax, diag);
  count_launch();
}
// Off-diagonal block pair of a row-sharded X (SURVEY §8(e) symmetry check):
// A = X[rows_g, cols_h] (rows × cols, lda) held locally, B = X[rows_h, cols_g]
// (cols × rows, ldb) received from rank h.  Accumulates into stats (same layout
// as sym_stats: max|x|, max|a_ij − b_ji|, flags 1 = not bitwise equal,
// 2 = non-finite).  64×64 tiles, B staged transposed through shared memory.
__global__ void __launch_bounds__(256, 4) pair_defect_kernel(const double* __restrict__ a, long long lda,
                                                          const double* __restrict__ b, long long ldb,
                                                          long long rows, long long cols, long long tiles_c,
                                                          long long ntiles, double* stats) {
  __shared__ double tb[kSymT][kSymT + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double mabs = 0.0, mdef = 0.0;
  int flags = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long r0 = (t / tiles_c) * kSymT, c0 = (t % tiles_c) * kSymT;
    double av[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        // b[c0 + r][r0 + c] → smem; a[r0 + r][c0 + c] → registers
        tb[r][c] = (c0 + r < cols && r0 + c < rows) ? __ldcs(b + (c0 + r) * ldb + r0 + c) : 0.0;
        av[q][h] = (r0 + r < rows && c0 + c < cols) ? __ldcs(a + (r0 + r) * lda + c0 + c) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = ty + 8 * q;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = tx + 32 * h;
        const double x = av[q][h], y = tb[c][r];   // a[i][j], b[j][i]
        if (!isfinite(x) || !isfinite(y)) flags |= 2;
        mabs = fmax(mabs, fmax(fabs(x), fabs(y)));
        mdef = fmax(mdef, fabs(x - y));
        if (x != y) flags |= 1;
      }
    }
    __syncthreads();
  }
  __shared__ double rmax[8], rdef[8];
  __shared__ int rfl[8];
  mabs = warp_max(mabs);
  mdef = warp_max(mdef);
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (tx == 0) {
    rmax[ty] = mabs;
    rdef[ty] = mdef;
    rfl[ty] = flags;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m1 = 0.0, m2 = 0.0;
    int f = 0;
    for (int w = 0; w < 8; ++w) {
      m1 = fmax(m1, rmax[w]);
      m2 = fmax(m2, rdef[w]);
      f |= rfl[w];
    }
    if (m1 > 0.0) atomic_max_nonneg(&stats[0], m1);
    if (m2 > 0.0) atomic_max_nonneg(&stats[1], m2);
    if (f) atomicOr(reinterpret_cast<int*>(stats + 2), f);
  }
}

void pair_defect(const double* a, long long lda, const double* b, long long ldb, long long rows,
                 long long cols, double* stats, bool reset, cudaStream_t st) {
  if (reset) cudaMemsetAsync(stats, 0, 3 * sizeof(double), st);
  if (rows < 1 || cols < 1) return;
  const long long tr = (rows + kSymT - 1) / kSymT, tc = (cols + kSymT - 1) / kSymT;
  const long long blocks = std::min<long long>(tr * tc, (long long)device_info().sms * 6);
  pair_defect_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, lda, b, ldb, rows, cols, tc, tr * tc, stats);
  count_launch();
}

// out[0] = max_ij |G_ij − δ_ij| for a w×w Gram (orthogonality defect of Q).
__global__ void identity_defect_kernel(const double* __restrict__ g, int w, long long ldg, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < w; i += nw)   // warp per row: coalesced, no index division
    for (int j = lane; j < w; j += 32) m = fmax(m, fabs(g[(long long)i * ldg + j] - (i == j ? 1.0 : 0.0)));
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t = fmax(t, red[k]);
    out[0] = t;
  }
}
void identity_defect(const double* g, int w, long long ldg, double* out, cudaStream_t st) {
  identity_defect_kernel<<<1, 1024, 0, st>>>(g, w, ldg, out);
  count_launch();
}

void sym_stats(const double* x, long long n, long long ldx, double* stats, cudaStream_t st,
               unsigned* rowmax, long long grid) {
  sym_stats_t(x, n, ldx, stats, rowmax, st, grid);
}
void sym_stats_f32(const float* x, long long n, long long ldx, double* stats, cudaStream_t st) {
  sym_stats_t(x, n, ldx, stats, static_cast<unsigned*>(nullptr), st);
}

__global__ void convert_f32_f64_kernel(const float* __restrict__ src, long long lds, double* dst,
                                       long long ldd, long long rows, int cols) {
  const long long total = rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols;
    const int c = (int)(e % cols);
    dst[r * ldd + c] = (double)src[r * lds + c];
  }
}
void convert_f32_f64(const float* src, long long lds, double* dst, long long ldd, long long rows,
                     int cols, cudaStream_t st) {
  const long long total = rows * cols;
  const long long blocks = std::min<long long>((total + 255) / 256, (long long)device_info().sms * 16);
  convert_f32_f64_kernel<<<(unsigned)std::max<long long>(blocks, 1), 256, 0, st>>>(src, lds, dst, ldd,
                                                                                  rows, cols);
  count_launch();
}

// A ← (A + Aᵀ)/2 in place (symmetric.py:31-36): one 32×32 tile pair (I ≥ J)
// per block, both tiles staged through shared memory so reads and writes
// stay coalesced; the mirrored pair is written with one value (exactly
// symmetric result).
__global__ void __launch_bounds__(256) symmetrize_kernel(double* x, long long m, long long ld) {
  __shared__ double ta[32][33], tb[32][33];
  const long long b = blockIdx.x;
  long long ti = (long long)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= b) ++ti;
  while (ti * (ti + 1) / 2 > b) --ti;
  const long long tj = b - ti * (ti + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const long long r0 = ti * 32, c0 = tj * 32;
  for (int r = ty; r < 32; r += 8) {
    const long long ar = r0 + r, ac = c0 + tx;
    ta[r][tx] = (ar < m && ac < m) ? x[ar * ld + ac] : 0.0;   // tile (I, J)
    const long long br = c0 + r, bc = r0 + tx;
    tb[r][tx] = (br < m && bc < m) ? x[br * ld + bc] : 0.0;   // tile (J, I)
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long long ar = r0 + r, ac = c0 + tx;
    // (A + Aᵀ)/2 at (r0 + r, c0 + tx) uses x[c0 + tx][r0 + r] = tb[tx][r]
    const double v = (ta[r][tx] + tb[tx][r]) / 2.0;
    const double w = (tb[r][tx] + ta[tx][r]) / 2.0;   // value at (c0 + r, r0 + tx)
    if (ar < m && ac < m) x[ar * ld + ac] = v;
    const long long br = c0 + r, bc = r0 + tx;
    if (ti != tj && br < m && bc < m) x[br * ld + bc] = w;
  }
}

void symmetrize_small(double* x, int m, long long ld, cudaStream_t st) {
  const long long nt = ((long long)m + 31) / 32;
  symmetrize_kernel<<<(unsigned)(nt * (nt + 1) / 2), 256, 0, st>>>(x, m, ld);
  count_launch();
}

// ---------------------------------------------------------------------------
// Ω on device: Philox4x32-10 → 2×53-bit uniforms → Box–Muller.
// Used only when the caller does not supply Ω (perf mode); parity runs pass
// the host numpy Ω (symmetric.py:135) instead.
// ---------------------------------------------------------------------------
PSD_DEVINL void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                             uint32_t k1) {
  const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
  const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
  c0 = n0;
  c1 = n1;
  c2 = n2;
  c3 = n3;
}

__global__ void philox_normal_kernel(double* out, long long rows, int cols, long long ld,
                                     uint64_t seed, uint64_t offset) {
  const long long total = rows * (long long)cols;
  const long long pair = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * pair >= total) return;
  uint32_t c0 = (uint32_t)(pair + offset), c1 = (uint32_t)((pair + offset) >> 32), c2 = 0x5053u,
           c3 = 0x44u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const double two53 = 1.0 / 9007199254740992.0;
  const uint64_t b1 = ((uint64_t)c0 << 21) | (uint64_t)(c1 >> 11);  // 53 bits
  const uint64_t b2 = ((uint64_t)c2 << 21) | (uint64_t)(c3 >> 11);
  const double u1 = ((double)b1 + 0.5) * two53;  // (0, 1)
  const double u2 = (double)b2 * two53;          // [0, 1)
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  const long long e0 = 2 * pair, e1 = 2 * pair + 1;
  out[(e0 / cols) * ld + (e0 % cols)] = r * c;
  if (e1 < total) out[(e1 / cols) * ld + (e1 % cols)] = r * s;
}

__global__ void sym_gaussian_kernel(double* out, long long ldo, long long r0, long long rows,
                                    long long n, uint64_t seed, double scale, double beta) {
  const long long total = rows * n;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long i = r0 + idx / n, j = idx % n;
    const long long lo = i < j ? i : j, hi = i < j ? j : i;
    const unsigned long long key = (unsigned long long)lo * (unsigned long long)n + (unsigned long long)hi;
    uint32_t c0 = (uint32_t)key, c1 = (uint32_t)(key >> 32), c2 = 0x53594d4du, c3 = 0x45u;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      philox_round(c0, c1, c2, c3, k0, k1);
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const double two53 = 1.0 / 9007199254740992.0;
    const uint64_t b1 = ((uint64_t)c0 << 21) | (uint64_t)(c1 >> 11);
    const uint64_t b2 = ((uint64_t)c2 << 21) | (uint64_t)(c3 >> 11);
    const double u1 = ((double)b1 + 0.5) * two53;
    const double u2 = (double)b2 * two53;
    const double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    double* o = out + (idx / n) * ldo + j;
    *o = (beta != 0.0 ? beta * *o : 0.0) + scale * z;
  }
}

void sym_gaussian_rows(double* out, long long ldo, long long r0, long long rows, long long n,
                       uint64_t seed, double scale, double beta, cudaStream_t st) {
  const long long total = rows * n;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)device_info().sms * 32);
  sym_gaussian_kernel<<<blocks, 256, 0, st>>>(out, ldo, r0, rows, n, seed, scale, beta);
  count_launch();
}

void philox_normal(double* out, long long rows, int cols, long long ld, uint64_t seed,
                   uint64_t offset, cudaStream_t st) {
  const long long pairs = (rows * (long long)cols + 1) / 2;
  philox_normal_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(out, rows, cols, ld, seed,
                                                                        offset);
  count_launch();
}

// ---------------------------------------------------------------------------
// a8 — power_iteration GEMV (sketch.py:109,114): y = (X − σI)v, HBM-bound.
// One warp per 4 rows, 16-byte loads, per-block partial Σy² (deterministic).
// ---------------------------------------------------------------------------
constexpr int kGemvRowsPerWarp = 4;
constexpr int kGemvWarps = 8;

__global__ void __launch_bounds__(256) gemv_kernel(const double* __restrict__ x, long long n,
                                                   long long ldx, const double* __restrict__ v,
                                                   double shift, double* __restrict__ y,
                                                   double* __restrict__ partials, int vec) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long row0 = ((long long)blockIdx.x * kGemvWarps + warp) * kGemvRowsPerWarp;
  double acc[kGemvRowsPerWarp] = {0.0, 0.0, 0.0, 0.0};
  if (vec) {
    for (long long c = 2 * lane; c + 1 < n; c += 64) {
      const double2 vv = *reinterpret_cast<const double2*>(v + c);
#pragma unroll
      for (int r = 0; r < kGemvRowsPerWarp; ++r) {
        const long long row = row0 + r;
        if (row < n) {
          const double2 xx = __ldcs(reinterpret_cast<const double2*>(x + row * ldx + c));
          acc[r] = fma(xx.x, vv.x, acc[r]);
          acc[r] = fma(xx.y, vv.y, acc[r]);
        }
      }
    }
    if ((n & 1) && lane == 0) {
      const long long c = n - 1;
#pragma unroll
      for (int r = 0; r < kGemvRowsPerWarp; ++r)
        if (row0 + r < n) acc[r] = fma(x[(row0 + r) * ldx + c], v[c], acc[r]);
    }
  } else {
    for (long long c = lane; c < n; c += 32) {
      const double vv = v[c];
#pragma unroll
      for (int r = 0; r < kGemvRowsPerWarp; ++r)
        if (row0 + r < n) acc[r] = fma(x[(row0 + r) * ldx + c], vv, acc[r]);
    }
  }
  double sq = 0.0;
#pragma unroll
  for (int r = 0; r < kGemvRowsPerWarp; ++r) {
    double s = warp_sum(acc[r]);
    const long long row = row0 + r;
    if (row < n) {
      s = s - shift * v[row];
      if (lane == 0) y[row] = s;
      sq = fma(s, s, sq);
    }
  }
  __shared__ double red[kGemvWarps];
  if (lane == 0) red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < kGemvWarps; ++w) tot += red[w];
    partials[blockIdx.x] = tot;
  }
}

int gemv_blocks(long long n) {
  const long long rows_per_block = kGemvWarps * kGemvRowsPerWarp;
  return (int)((n + rows_per_block - 1) / rows_per_block);
}

int gemv_shift(const double* x, long long n, long long ldx, const double* v, double shift,
               double* y, double* partials, cudaStream_t st) {
  const int blocks = gemv_blocks(n);
  const int vec = ((uintptr_t)x % 16 == 0) && (ldx % 2 == 0) && ((uintptr_t)v % 16 == 0);
  gemv_kernel<<<blocks, 256, 0, st>>>(x, n, ldx, v, shift, y, partials, vec);
  count_launch();
  return blocks;
}

// a8 for a BITWISE-symmetric X: y = (X − σI)v reading only the lower triangle of 64×64
// tiles (half the HBM bytes of the row GEMV).  Pass 1: each lower tile (I, J) yields its row
// sums X_IJ·v_J and, off the diagonal, its column sums X_IJᵀ·v_I (= the (J, I) tile's row
// sums), stored per tile; pass 2 adds them per row in a fixed order (deterministic) and
// writes y and per-block Σy² like the GEMV.  n % 64 == 0, 16-byte rows.
constexpr int kSymvT = 64;

__global__ void __launch_bounds__(256) symv_tiles_kernel(const double* __restrict__ x, long long ldx,
                                                         const double* __restrict__ v, long long ntri,
                                                         double* __restrict__ pr, double* __restrict__ pc) {
  __shared__ double cs[8][kSymvT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long long t = blockIdx.x; t < ntri; t += gridDim.x) {
    long long I = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const long long J = t - I * (I + 1) / 2;
    const long long r0 = I * kSymvT + warp * 8, c0 = J * kSymvT + 2 * lane;
    const double2 vc = *reinterpret_cast<const double2*>(v + c0);
    const bool off = I != J;
    double acc[8], ca0 = 0.0, ca1 = 0.0;
    double2 xx[8];
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) xx[rr] = __ldcs(reinterpret_cast<const double2*>(x + (r0 + rr) * ldx + c0));
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      acc[rr] = fma(xx[rr].x, vc.x, xx[rr].y * vc.y);
      if (off) {
        const double vr = v[r0 + rr];
        ca0 = fma(xx[rr].x, vr, ca0);
        ca1 = fma(xx[rr].y, vr, ca1);
      }
    }
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const double s = warp_sum(acc[rr]);
      if (lane == 0) pr[t * kSymvT + warp * 8 + rr] = s;
    }
    if (off) {
      cs[warp][2 * lane] = ca0;
      cs[warp][2 * lane + 1] = ca1;
    }
    __syncthreads();
    if (off && threadIdx.x < kSymvT) {
      double c = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) c += cs[w][threadIdx.x];
      pc[t * kSymvT + threadIdx.x] = c;
    }
    __syncthreads();
  }
}

// one block per 64-row tile K: thread (q, o) adds every 4th of the row's nt partials — the
// (K, J) row sums for J ≤ K, then the (I, K) column sums for I > K — in a fixed order, and
// the four quarters are added in a fixed order (deterministic, independent loads in flight)
__global__ void __launch_bounds__(256) symv_reduce_kernel(const double* __restrict__ pr, const double* __restrict__ pc,
                                                          long long nt, long long n, const double* __restrict__ v,
                                                          double shift, double* __restrict__ y,
                                                          double* __restrict__ partials) {
  __shared__ double qs[4][kSymvT];
  const long long K = blockIdx.x;
  const int q = threadIdx.x >> 6, o = threadIdx.x & 63;
  double s0 = 0.0, s1 = 0.0;
  long long e = q;
#pragma unroll 4
  for (; e + 4 < nt; e += 8) {
    const long long e2 = e + 4;
    const double a = e <= K ? pr[(K * (K + 1) / 2 + e) * kSymvT + o] : pc[(e * (e + 1) / 2 + K) * kSymvT + o];
    const double b = e2 <= K ? pr[(K * (K + 1) / 2 + e2) * kSymvT + o] : pc[(e2 * (e2 + 1) / 2 + K) * kSymvT + o];
    s0 += a;
    s1 += b;
  }
  if (e < nt) s0 += e <= K ? pr[(K * (K + 1) / 2 + e) * kSymvT + o] : pc[(e * (e + 1) / 2 + K) * kSymvT + o];
  qs[q][o] = s0 + s1;
  __syncthreads();
  double sq = 0.0;
  if (threadIdx.x < kSymvT) {
    const long long i = K * kSymvT + threadIdx.x;
    const double yi = ((qs[0][threadIdx.x] + qs[1][threadIdx.x]) + (qs[2][threadIdx.x] + qs[3][threadIdx.x])) -
                      shift * v[i];
    y[i] = yi;
    sq = yi * yi;
  }
  sq = warp_sum(sq);
  if (threadIdx.x == 0) partials[blockIdx.x] = sq;
  __syncthreads();
  if (threadIdx.x == 32) partials[blockIdx.x] += sq;   // the second warp of the 64 rows
}

size_t symv_ws_elems(long long n) {
  const long long nt = n / kSymvT;
  return (size_t)nt * (nt + 1) / 2 * kSymvT * 2;
}

bool symv_ok(const double* x, long long n, long long ldx, const double* v) {
  return n % kSymvT == 0 && n >= kSymvT && ldx % 2 == 0 && (uintptr_t)x % 16 == 0 && (uintptr_t)v % 16 == 0;
}

int symv_shift(const double* x, long long n, long long ldx, const double* v, double shift, double* y,
               double* partials, double* ws, cudaStream_t st) {
  const long long nt = n / kSymvT, ntri = nt * (nt + 1) / 2;
  double* pr = ws;
  double* pc = ws + ntri * kSymvT;
  const long long blocks = std::min<long long>(ntri, (long long)device_info().sms * 8);
  symv_tiles_kernel<<<(unsigned)blocks, 256, 0, st>>>(x, ldx, v, ntri, pr, pc);
  const int rb = (int)nt;
  symv_reduce_kernel<<<rb, 256, 0, st>>>(pr, pc, nt, n, v, shift, y, partials);
  count_launch(2);
  return rb;
}

__global__ void normalize_kernel(const double* __restrict__ y, const double* __restrict__ partials,
                                 int nparts, long long n, double floor, double* __restrict__ v,
                                 double* out, int* flag) {
  __shared__ double red[32];
  __shared__ double nrm_s;
  double s = 0.0;
  // fixed-order reduction so every launch (and every block) gets the same value
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    nrm_s = sqrt(t);
    if (blockIdx.x == 0) {
      if (out) out[0] = nrm_s;
      if (flag && !(nrm_s > floor)) *flag = 1;
    }
  }
  __syncthreads();
  const double nrm = nrm_s;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = y[i] / nrm;
}

void normalize(const double* y, const double* partials, int nparts, long long n, double floor,
               double* v, double* out, int* flag, cudaStream_t st) {
  int blocks = (int)std::min<long long>((n + 1023) / 1024, 64);
  if (blocks < 1) blocks = 1;
  normalize_kernel<<<blocks, 1024, 0, st>>>(y, partials, nparts, n, floor, v, out, flag);
  count_launch();
}

__global__ void sum_partials_kernel(const double* partials, long long nparts, double* out,
                                    int do_sqrt) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[0] = do_sqrt ? sqrt(t) : t;
  }
}

void sum_partials(const double* partials, long long nparts, double* out, int do_sqrt,
                  cudaStream_t st) {
  sum_partials_kernel<<<1, 1024, 0, st>>>(partials, nparts, out, do_sqrt);
  count_launch();
}

// ---------------------------------------------------------------------------
// split-K reduction + epilogue
// ---------------------------------------------------------------------------
__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits,
                                     long long split_stride, int M, int N, long long ldw,
                                     double* C, long long ldc, int mode, double alpha,
                                     const double* S, long long lds) {
  const long long total = (long long)M * N;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(idx / N), n = (int)(idx % N);
    double v = 0.0;
    for (int s = 0; s < splits; ++s) v += ws[s * split_stride + (long long)m * ldw + n];
    if (mode == 10) {  // symmetric part of a square result: (T + Tᵀ)/2
      if (m < n) continue;
      double u = 0.0;
      for (int s = 0; s < splits; ++s) u += ws[s * split_stride + (long long)n * ldw + m];
      const double sv = (v + u) / 2.0;
      C[(long long)m * ldc + n] = sv;
      C[(long long)n * ldc + m] = sv;
      continue;
    }
    if (mode == EPI_SHIFT) v = (v + alpha * S[(long long)m * lds + n]) / alpha;
    else if (mode == EPI_SUB) v = S[(long long)m * lds + n] - v;
    C[(long long)m * ldc + n] = v;
  }
}

void splitk_reduce(const double* ws, int splits, long long split_stride, int M, int N,
                   long long ldw, double* C, long long ldc, int mode, double alpha,
                   const double* S, long long lds, cudaStream_t st) {
  const long long total = (long long)M * N;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, splits, split_stride, M, N, ldw, C, ldc, mode,
                                               alpha, S, lds);
  count_launch();
}

// ---------------------------------------------------------------------------
// panel utilities
// ---------------------------------------------------------------------------
__global__ void copy_matrix_kernel(const double* src, long long lds, double* dst, long long ldd,
                                   long long rows, int cols) {
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols;
    const int c = (int)(i % cols);
    dst[r * ldd + c] = src[r * lds + c];
  }
}

void copy_matrix(const double* src, long long lds, double* dst, long long ldd, long long rows,
                 int cols, cudaStream_t st) {
  const long long total = rows * cols;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  copy_matrix_kernel<<<blocks, 256, 0, st>>>(src, lds, dst, ldd, rows, cols);
  count_launch();
}

__global__ void fill_zero_kernel(double* dst, long long ld, long long rows, long long cols) {
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    dst[(i / cols) * ld + (i % cols)] = 0.0;
}

void fill_zero(double* dst, long long ld, long long rows, long long cols, cudaStream_t st) {
  if (ld == cols) {
    cudaMemsetAsync(dst, 0, (size_t)rows * cols * sizeof(double), st);
    return;
  }
  const long long total = rows * cols;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  fill_zero_kernel<<<blocks, 256, 0, st>>>(dst, ld, rows, cols);
  count_launch();
}

// out[m][k] = w[m][k] · d[k]  — (w_kept * d_kept) of projection.py:77
__global__ void scale_columns_kernel(const double* w, long long ldw, const double* d, double* out,
                                     long long ldo, long long rows, int cols) {
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / cols;
    const int c = (int)(i % cols);
    out[r * ldo + c] = w[r * ldw + c] * d[c];
  }
}

void scale_columns(const double* w, long long ldw, const double* d, double* out, long long ldo,
                   long long rows, int cols, cudaStream_t st) {
  const long long total = rows * cols;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  scale_columns_kernel<<<blocks, 256, 0, st>>>(w, ldw, d, out, ldo, rows, cols);
  count_launch();
}

__global__ void gather_columns_kernel(const double* src, long long lds, const int* idx, int ncols,
                                      double* dst, long long ldd, long long rows) {
  const long long total = rows * ncols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ncols;
    const int c = (int)(i % ncols);
    dst[r * ldd + c] = src[r * lds + idx[c]];
  }
}

void gather_columns(const double* src, long long lds, const int* idx, int ncols, double* dst,
                    long long ldd, long long rows, cudaStream_t st) {
  const long long total = rows * ncols;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 32);
  gather_columns_kernel<<<blocks, 256, 0, st>>>(src, lds, idx, ncols, dst, ldd, rows);
  count_launch();
}

__global__ void __launch_bounds__(256) max_abs_kernel(const double* __restrict__ x, long long rows,
                                                      long long cols, long long ldx, double* out) {
  double m = 0.0;
  const long long total = rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[(i / cols) * ldx + (i % cols)]));
  m = warp_max(m);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t = fmax(t, red[w]);
    if (t > 0.0) atomic_max_nonneg(out, t);
  }
}

void max_abs(const double* x, long long rows, long long cols, long long ldx, double* out,
             cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(double), st);
  const long long total = rows * cols;
  if (total == 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)device_info().sms * 8);
  max_abs_kernel<<<blocks, 256, 0, st>>>(x, rows, cols, ldx, out);
  count_launch();
}

__global__ void add_diag_kernel(double* a, long long ld, int m, double s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) a[(long long)i * ld + i] += s;
}

void add_diag(double* a, long long ld, int m, double s, cudaStream_t st) {
  add_diag_kernel<<<(m + 255) / 256, 256, 0, st>>>(a, ld, m, s);
  count_launch();
}

__global__ void set_identity_kernel(double* a, long long ld, int m) {
  const long long total = (long long)m * m;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / m), c = (int)(i % m);
    a[(long long)r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
}

void set_identity(double* a, long long ld, int m, cudaStream_t st) {
  const long long total = (long long)m * m;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 4096);
  set_identity_kernel<<<blocks, 256, 0, st>>>(a, ld, m);
  count_launch();
}

// ---------------------------------------------------------------------------
// Small device→host status reads through a kernel storing into host-mapped
// pinned memory instead of cudaMemcpy: device→host DMA copies share the copy
// engine with any big transfer in flight on other streams (ran_proj_many's
// 8.6 GB downloads), and a status read queued behind one waits for all of it.
// ---------------------------------------------------------------------------
__global__ void copy_to_mapped_kernel(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src,
                                      size_t bytes) {
  for (size_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

// Asynchronous variant for one early status word block: the copy kernel and an event are
// enqueued, the caller keeps enqueueing work and collects the bytes later
// (read_small_wait), so the stream is never drained for the read.
struct AsyncSlot {
  unsigned char* h = nullptr;
  unsigned char* d = nullptr;
  cudaEvent_t ev = nullptr;
};
static AsyncSlot& async_slot() {
  thread_local AsyncSlot slot[16];
  int dev = 0;
  cudaGetDevice(&dev);
  return slot[dev & 15];
}

cudaError_t read_small_async(const void* dev_src, size_t bytes, cudaStream_t st) {
  AsyncSlot& sl = async_slot();
  if (bytes > 4096) return cudaErrorInvalidValue;
  if (!sl.h) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&sl.h), 4096, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&sl.d), sl.h, 0);
    if (e != cudaSuccess) return e;
    e = cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  copy_to_mapped_kernel<<<1, 256, 0, st>>>(sl.d, static_cast<const unsigned char*>(dev_src), bytes);
  return cudaEventRecord(sl.ev, st);
}

void copy_to_mapped(void* mapped_dev_dst, const void* dev_src, size_t bytes, cudaStream_t st) {
  copy_to_mapped_kernel<<<1, 256, 0, st>>>(static_cast<unsigned char*>(mapped_dev_dst),
                                           static_cast<const unsigned char*>(dev_src), bytes);
  count_launch();
}

cudaError_t read_small_wait(void* host_dst, size_t bytes) {
  AsyncSlot& sl = async_slot();
  cudaError_t e = cudaEventSynchronize(sl.ev);
  if (e != cudaSuccess) return e;
  std::memcpy(host_dst, sl.h, bytes);
  return cudaGetLastError();
}

cudaError_t read_small(void* host_dst, const void* dev_src, size_t bytes, cudaStream_t st) {
  return read_small2(host_dst, dev_src, bytes, nullptr, nullptr, 0, st);
}

// two status blocks in one host round trip (two copy kernels, one stream sync)
cudaError_t read_small2(void* host_dst, const void* dev_src, size_t bytes, void* host_dst2, const void* dev_src2,
                        size_t bytes2, cudaStream_t st) {
  constexpr size_t kCap = 64 << 10;
  struct Staging {
    unsigned char* h = nullptr;
    unsigned char* d = nullptr;
  };
  thread_local Staging stage[16];
  int dev = 0;
  cudaGetDevice(&dev);
  Staging& sg = stage[dev & 15];
  if (bytes + bytes2 > kCap) {   // not a status read: plain copies
    cudaError_t e = cudaMemcpyAsync(host_dst, dev_src, bytes, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && bytes2) e = cudaMemcpyAsync(host_dst2, dev_src2, bytes2, cudaMemcpyDeviceToHost, st);
    return e != cudaSuccess ? e : cudaStreamSynchronize(st);
  }
  if (!sg.h) {
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&sg.h), kCap, cudaHostAllocMapped);
    if (e != cudaSuccess) return e;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&sg.d), sg.h, 0);
    if (e != cudaSuccess) return e;
  }
  const size_t off2 = (bytes + 15) / 16 * 16;
  copy_to_mapped_kernel<<<1, 256, 0, st>>>(sg.d, static_cast<const unsigned char*>(dev_src), bytes);
  if (bytes2)
    copy_to_mapped_kernel<<<1, 256, 0, st>>>(sg.d + off2, static_cast<const unsigned char*>(dev_src2), bytes2);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  std::memcpy(host_dst, sg.h, bytes);
  if (bytes2) std::memcpy(host_dst2, sg.h + off2, bytes2);
  return cudaGetLastError();
}

}  // namespace psd
