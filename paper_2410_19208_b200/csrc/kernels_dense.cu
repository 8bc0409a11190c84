// Small dense (w×w) kernels: blocked Cholesky for CholeskyQR, triangular
// inverse, block-Jacobi symmetric eigensolver (symmetric.py:68-86 semantics)
// and the descending sort / sign convention.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "launch.h"

namespace psd {

// ---------------------------------------------------------------------------
// Cholesky: panel factor in shared memory + DMMA trailing update.
// ---------------------------------------------------------------------------
constexpr int kCholNB = 32;

__global__ void __launch_bounds__(512) chol_panel_kernel(double* a, long long lda, int m, int p0,
                                                         int nb, int* info) {
  extern __shared__ double P[];
  const int rows = m - p0;
  const int st = nb + 1;
  for (int idx = threadIdx.x; idx < rows * nb; idx += blockDim.x) {
    const int r = idx / nb, c = idx % nb;
    P[r * st + c] = a[(long long)(p0 + r) * lda + p0 + c];
  }
  __syncthreads();
  __shared__ double piv_s;
  for (int j = 0; j < nb; ++j) {
    if (threadIdx.x == 0) {
      const double d = P[j * st + j];
      if (!(d > 0.0) || !isfinite(d)) {
        if (info[0] == 0) info[0] = p0 + j + 1;
      }
      const double pv = sqrt(fmax(d, 0.0));
      P[j * st + j] = pv;
      piv_s = pv;
    }
    __syncthreads();
    const double pv = piv_s;
    for (int r = j + 1 + threadIdx.x; r < rows; r += blockDim.x) P[r * st + j] /= pv;
    __syncthreads();
    const int nc = nb - j - 1;
    if (nc > 0) {
      // P[r][c] -= P[r][j]·P[c][j]  for j < c ≤ r
      const int cnt = (rows - j - 1) * nc;
      for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
        const int r = j + 1 + idx / nc, c = j + 1 + idx % nc;
        if (r >= c) P[r * st + c] -= P[r * st + j] * P[c * st + j];
      }
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < rows * nb; idx += blockDim.x) {
    const int r = idx / nb, c = idx % nb;
    a[(long long)(p0 + r) * lda + p0 + c] = (r >= c) ? P[r * st + c] : 0.0;
  }
}

__global__ void zero_upper_kernel(double* a, long long lda, int m) {
  const long long total = (long long)m * m;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / m), c = (int)(i % m);
    if (c > r) a[(long long)r * lda + c] = 0.0;
  }
}

int cholesky_lower(double* a, long long lda, int m, int* info, double* ws, size_t ws_elems,
                   cudaStream_t st) {
  static size_t attr_bytes[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = (size_t)m * (kCholNB + 1) * sizeof(double);
  if (need > device_info().max_smem - 1024) return -1;
  if (need > attr_bytes[dev]) {
    if (cudaFuncSetAttribute(chol_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)need) != cudaSuccess)
      return -1;
    attr_bytes[dev] = need;
  }
  cudaMemsetAsync(info, 0, sizeof(int), st);
  for (int p0 = 0; p0 < m; p0 += kCholNB) {
    const int nb = std::min(kCholNB, m - p0);
    const size_t smem = (size_t)(m - p0) * (nb + 1) * sizeof(double);
    chol_panel_kernel<<<1, 512, smem, st>>>(a, lda, m, p0, nb, info);
    count_launch();
    const int rest = m - p0 - nb;
    if (rest > 0) {
      GemmOp op;
      op.a_layout = A_MK;
      op.b_layout = B_NK;
      op.A = a + (long long)(p0 + nb) * lda + p0;
      op.lda = lda;
      op.B = op.A;
      op.ldb = lda;
      op.C = a + (long long)(p0 + nb) * lda + p0 + nb;
      op.ldc = lda;
      op.S = op.C;
      op.lds = lda;
      op.M = rest;
      op.N = rest;
      op.K = nb;
      op.epi = EPI_SUB;
      op.max_splits = 1;
      gemm_f64(op, ws, ws_elems, st);
    }
  }
  const long long total = (long long)m * m;
  zero_upper_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 4096), 256, 0, st>>>(a, lda,
                                                                                              m);
  count_launch();
  return 0;
}

// rinv row j = column j of L⁻¹ (forward substitution, one warp per column).
__global__ void tri_inv_kernel(const double* __restrict__ l, long long ldl, int m, double* rinv,
                               long long ldr) {
  extern __shared__ double xs[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + warp;
  if (j >= m) return;
  double* x = xs + (size_t)warp * m;
  if (lane == 0) x[j] = 1.0 / l[(long long)j * ldl + j];
  __syncwarp();
  for (int i = j + 1; i < m; ++i) {
    const double* row = l + (long long)i * ldl;
    double s = 0.0;
    for (int k = j + lane; k < i; k += 32) s = fma(row[k], x[k], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = -s / row[i];
    __syncwarp();
  }
  double* out = rinv + (long long)j * ldr;
  for (int i = lane; i < m; i += 32) out[i] = (i >= j) ? x[i] : 0.0;
}

void tri_inv_upper_from_lower(const double* l, long long ldl, int m, double* rinv,
                              long long ldr, cudaStream_t st) {
  const int warps = 8;
  const size_t smem = (size_t)warps * m * sizeof(double);
  static size_t attr_bytes[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && smem > attr_bytes[dev]) {
    cudaFuncSetAttribute(tri_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_bytes[dev] = smem;
  }
  tri_inv_kernel<<<(m + warps - 1) / warps, warps * 32, smem, st>>>(l, ldl, m, rinv, ldr);
  count_launch();
}

__global__ void accumulate_diag_kernel(const double* l, long long ldl, int m, double* rdiag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) rdiag[i] *= fabs(l[(long long)i * ldl + i]);
}

void accumulate_diag(const double* l, long long ldl, int m, double* rdiag, cudaStream_t st) {
  accumulate_diag_kernel<<<(m + 255) / 256, 256, 0, st>>>(l, ldl, m, rdiag);
  count_launch();
}

// ---------------------------------------------------------------------------
// symmetric.py:80-85: reverse to descending order, orient each eigenvector so
// its largest-|entry| (first on ties) is positive.
// ---------------------------------------------------------------------------
__global__ void sort_eigs_kernel(const double* vals, const double* vecs, long long ldv, int m,
                                 double offset, double* vals_out, double* vecs_out, long long ldo,
                                 int* npos, int* perm) {
  __shared__ int pos_count;
  constexpr int kSm = 2048;
  __shared__ double sv[kSm];
  if (threadIdx.x == 0) pos_count = 0;
  for (int i = threadIdx.x; i < min(m, kSm); i += blockDim.x) sv[i] = vals[i];
  __syncthreads();
  const double* v = m <= kSm ? sv : vals;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double li = v[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = v[j];
      rank += (lj > li) || (lj == li && j < i);
    }
    perm[rank] = i;
    vals_out[rank] = li;
    if (li - offset > 0.0) atomicAdd(&pos_count, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) npos[0] = pos_count;
}

// one CTA per output column: gather the permuted source column, find its first
// largest-|entry| (block argmax), store it with that entry made positive
__global__ void __launch_bounds__(256) orient_columns_kernel(const double* __restrict__ vecs, long long ldv, int m,
                                                             const int* __restrict__ perm,
                                                             double* __restrict__ vecs_out, long long ldo) {
  const int col = blockIdx.x;
  const int src = perm[col];
  __shared__ double sb[8];
  __shared__ int si[8];
  double best = -1.0;
  int bidx = 0x7fffffff;
  for (int r = threadIdx.x; r < m; r += blockDim.x) {
    const double x = fabs(vecs[(long long)r * ldv + src]);
    if (x > best) {
      best = x;
      bidx = r;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) {
      best = ob;
      bidx = oi;
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sb[warp] = best;
    si[warp] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sb[w] > sb[0] || (sb[w] == sb[0] && si[w] < si[0])) {
        sb[0] = sb[w];
        si[0] = si[w];
      }
  }
  __syncthreads();
  const double sg = (vecs[(long long)si[0] * ldv + src] < 0.0) ? -1.0 : 1.0;
  for (int r = threadIdx.x; r < m; r += blockDim.x) vecs_out[(long long)r * ldo + col] = sg * vecs[(long long)r * ldv + src];
}

void sort_eigs(const double* vals, const double* vecs, long long ldv, int m, double offset,
               double* vals_out, double* vecs_out, long long ldo, int* npos, int* perm,
               cudaStream_t st) {
  sort_eigs_kernel<<<1, 1024, 0, st>>>(vals, vecs, ldv, m, offset, vals_out, vecs_out, ldo, npos,
                                       perm);
  orient_columns_kernel<<<m, 256, 0, st>>>(vecs, ldv, m, perm, vecs_out, ldo);
  count_launch(2);
}

}  // namespace psd

namespace psd {

// ---------------------------------------------------------------------------
// One-launch CholeskyQR pass kernel (single CTA, 1024 threads):
//   L = chol(G + shift·I) (right-looking, 32-column panels in shared memory,
//   trailing update on the FP64 tensor cores), then Rinv = L⁻ᵀ by block
//   forward substitution.  G is read, not modified.
//   status = {info, trace(G), min L_ii, max L_ii} (info = first failing
//   pivot + 1, 0 if none).  Everything stays in L2 (m ≤ 544 → ≤ 2.4 MB).
// ---------------------------------------------------------------------------
constexpr int kCI_NB = 32;
constexpr int kCI_LD = kCI_NB + 4;  // panel stride ≡ 4 (mod 16): conflict-free DMMA fragments

__global__ void __launch_bounds__(1024, 1)
    chol_inv_kernel(const double* __restrict__ G, long long ldg, int m, double shift, double* L,
                    long long ldl, double* Rinv, long long ldr, double* Xs, long long ldx,
                    double* status) {
  extern __shared__ double sm[];
  double* P = sm;  // panel: rows × kCI_LD
  __shared__ double piv_s;
  __shared__ int info_s;
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // trace of G and copy G (+ shift on the diagonal) → L (full square, lower used)
  double tr = 0.0;
  for (long long e = tid; e < (long long)m * m; e += blockDim.x) {
    const int i = (int)(e / m), j = (int)(e % m);
    double v = G[(long long)i * ldg + j];
    if (i == j) {
      tr += v;
      v += shift;
    }
    L[(long long)i * ldl + j] = v;
  }
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  if (tid == 0) info_s = 0;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += red[w];
    status[1] = t;
  }

  // ---------------------------------------------------------------- Cholesky
  for (int p0 = 0; p0 < m; p0 += kCI_NB) {
    const int nb = min(kCI_NB, m - p0);
    const int rows = m - p0;
    for (int e = tid; e < rows * kCI_NB; e += blockDim.x) {
      const int r = e / kCI_NB, c = e % kCI_NB;
      P[r * kCI_LD + c] = (c < nb) ? L[(long long)(p0 + r) * ldl + p0 + c] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
      if (tid == 0) {
        const double d = P[j * kCI_LD + j];
        if ((!(d > 0.0) || !isfinite(d)) && info_s == 0) info_s = p0 + j + 1;
        const double pv = sqrt(fmax(d, 0.0));
        P[j * kCI_LD + j] = pv;
        piv_s = pv;
      }
      __syncthreads();
      const double pv = piv_s;
      for (int r = j + 1 + tid; r < rows; r += blockDim.x) P[r * kCI_LD + j] /= pv;
      __syncthreads();
      const int nc = nb - j - 1;
      if (nc > 0) {
        const int cnt = (rows - j - 1) * nc;
        for (int idx = tid; idx < cnt; idx += blockDim.x) {
          const int r = j + 1 + idx / nc, c = j + 1 + idx % nc;
          if (r >= c) P[r * kCI_LD + c] -= P[r * kCI_LD + j] * P[c * kCI_LD + j];
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < rows * nb; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      L[(long long)(p0 + r) * ldl + p0 + c] = (r >= c) ? P[r * kCI_LD + c] : 0.0;
    }
    // trailing update A22 −= L21 L21ᵀ (lower 8×8 blocks) with DMMA, K = 32
    const int t0 = p0 + nb;
    const int tn = m - t0;
    if (tn > 0) {
      const int tb = (tn + 7) / 8;
      const long long nblocks = (long long)tb * (tb + 1) / 2;
      const int g = lane >> 2, t = lane & 3;
      for (long long b = warp; b < nblocks; b += 32) {
        int bi = (int)((sqrt(8.0 * (double)b + 1.0) - 1.0) * 0.5);
        while ((long long)(bi + 1) * (bi + 2) / 2 <= b) ++bi;
        while ((long long)bi * (bi + 1) / 2 > b) --bi;
        const int bj = (int)(b - (long long)bi * (bi + 1) / 2);
        // panel rows of this block: (t0 − p0) + 8·bi + g
        const int ra = nb + 8 * bi + g, rb = nb + 8 * bj + g;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < kCI_NB; k0 += 4) {
          const double a = (ra < rows) ? P[ra * kCI_LD + k0 + t] : 0.0;
          const double bb = (rb < rows) ? P[rb * kCI_LD + k0 + t] : 0.0;
          dmma_8x8x4(c0, c1, a, bb);
        }
        const int gi = t0 + 8 * bi + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int gj = t0 + 8 * bj + 2 * t + e;
          if (gi < m && gj < m && gi >= gj) L[(long long)gi * ldl + gj] -= (e ? c1 : c0);
        }
      }
    }
    __syncthreads();
  }
  // zero the strict upper triangle (trailing updates left stale values there)
  for (long long e = tid; e < (long long)m * m; e += blockDim.x) {
    const int i = (int)(e / m), j = (int)(e % m);
    if (j > i) L[(long long)i * ldl + j] = 0.0;
  }
  __syncthreads();

  // diagonal statistics + R diagonal accumulation
  double dmin = INFINITY, dmax = 0.0;
  for (int i = tid; i < m; i += blockDim.x) {
    const double d = L[(long long)i * ldl + i];
    dmin = fmin(dmin, d);
    dmax = fmax(dmax, d);
  }
  for (int o = 16; o > 0; o >>= 1) {
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  __shared__ double rmin[32], rmax[32];
  if (lane == 0) {
    rmin[warp] = dmin;
    rmax[warp] = dmax;
  }
  __syncthreads();
  if (tid == 0) {
    double a = INFINITY, b2 = 0.0;
    for (int w = 0; w < 32; ++w) {
      a = fmin(a, rmin[w]);
      b2 = fmax(b2, rmax[w]);
    }
    status[0] = (double)info_s;
    status[2] = a;
    status[3] = b2;
  }
  if (info_s != 0) return;  // caller retries with a shift; Rinv not needed

  // ------------------------------------------- Rinv = L⁻ᵀ by block rows of X = L⁻¹
  // X row-block i: X_i = inv(L_ii) (E_i − Σ_{k<i} L_ik X_k).  X is kept
  // row-major in Xs (coalesced reads across lanes), Rinv[c][r] = X[r][c].
  double* Dl = sm;                              // L_ii   32 × 33
  double* Dinv = sm + kCI_NB * (kCI_NB + 1);    // inv    32 × 33
  double* Z = sm + 2 * kCI_NB * (kCI_NB + 1);   // 32 × m
  for (int r0 = 0; r0 < m; r0 += kCI_NB) {
    const int rows = min(kCI_NB, m - r0);
    for (int e = tid; e < kCI_NB * kCI_NB; e += blockDim.x) {
      const int r = e / kCI_NB, c = e % kCI_NB;
      Dl[r * (kCI_NB + 1) + c] = (r < rows && c <= r) ? L[(long long)(r0 + r) * ldl + r0 + c] : 0.0;
    }
    __syncthreads();
    // inverse of the diagonal block: thread c owns column c (forward substitution)
    if (tid < rows) {
      const int c = tid;
      Dinv[c * (kCI_NB + 1) + c] = 1.0 / Dl[c * (kCI_NB + 1) + c];
      for (int r = 0; r < c; ++r) Dinv[r * (kCI_NB + 1) + c] = 0.0;
      for (int r = c + 1; r < rows; ++r) {
        double sacc = 0.0;
        for (int k = c; k < r; ++k) sacc = fma(Dl[r * (kCI_NB + 1) + k], Dinv[k * (kCI_NB + 1) + c], sacc);
        Dinv[r * (kCI_NB + 1) + c] = -sacc / Dl[r * (kCI_NB + 1) + r];
      }
    }
    // Z[r][c] = −Σ_{k<r0} L[r0+r][k] X[k][c], c < r0   (warp = row r, lanes = c)
    if (warp < rows) {
      const double* lrow = L + (long long)(r0 + warp) * ldl;
      for (int cb = 0; cb < r0; cb += 32) {
        const int c = cb + lane;
        if (c < r0) {
          double sacc = 0.0;
#pragma unroll 8
          for (int k = cb; k < r0; ++k) sacc = fma(lrow[k], Xs[(long long)k * ldx + c], sacc);
          Z[warp * m + c] = -sacc;
        }
      }
    }
    __syncthreads();
    // X[r0 + r][c] = Σ_j Dinv[r][j] Z[j][c] (c < r0);  X_ii = Dinv; zero above
    for (int e = tid; e < rows * m; e += blockDim.x) {
      const int r = e / m, c = e % m;
      double v;
      if (c < r0) {
        v = 0.0;
        for (int j = 0; j <= r; ++j) v = fma(Dinv[r * (kCI_NB + 1) + j], Z[j * m + c], v);
      } else if (c < r0 + rows) {
        v = (c - r0 <= r) ? Dinv[r * (kCI_NB + 1) + (c - r0)] : 0.0;
      } else {
        v = 0.0;
      }
      Xs[(long long)(r0 + r) * ldx + c] = v;
      Rinv[(long long)c * ldr + r0 + r] = v;
    }
    __syncthreads();
  }
}

size_t chol_inv_smem(int m) {
  const size_t chol = (size_t)m * kCI_LD * sizeof(double);
  const size_t inv = ((size_t)2 * kCI_NB * (kCI_NB + 1) + (size_t)kCI_NB * m) * sizeof(double);
  return std::max(chol, inv);
}

int chol_inv(const double* G, long long ldg, int m, double shift, double* L, long long ldl,
             double* Rinv, long long ldr, double* Xs, double* status, cudaStream_t st) {
  const size_t smem = chol_inv_smem(m);
  if (smem > device_info().max_smem - 2048) return -1;
  static size_t attr[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > attr[dev]) {
    if (cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return -1;
    attr[dev] = smem;
  }
  chol_inv_kernel<<<1, 1024, smem, st>>>(G, ldg, m, shift, L, ldl, Rinv, ldr, Xs, m, status);
  count_launch();
  return 0;
}

}  // namespace psd

namespace psd {

// ---------------------------------------------------------------------------
// Fast CholeskyQR factor step (two launches, no explicit full-matrix loops
// on the critical path):
//   chol_blocked_kernel  (1 CTA):  L = chol(G + shift I) with 32-column
//     panels — the 32×32 diagonal block is factored by one warp in
//     registers (row per lane, shuffles), the panel below by a smem TRSM
//     against inv(L_jj), the trailing matrix by DMMA; also writes
//     Dinv_j = inv(L_jj) for every diagonal block and the status vector.
//   tri_inv_blocked_kernel (1 CTA per block column j): X = L⁻¹ column block
//     j by block forward substitution X_ij = −Dinv_i Σ_{k=j}^{i−1} L_ik X_kj,
//     written transposed into Rinv (Rinv = L⁻ᵀ, row block j contiguous).
// ---------------------------------------------------------------------------
constexpr int kFB = 32;
constexpr int kFL = kFB + 4;  // smem stride ≡ 4 (mod 16)

__device__ long long g_chol_t[6];

// Element (i, j), i ≥ j, of the matrix being factored at panel step p0:
// G + shift·I before any update (p0 == 0), the partially updated L after.
PSD_DEVINL double chol_src(const double* __restrict__ G, long long ldg, const double* L,
                           long long ldl, bool first, double shift, int i, int j) {
  if (first) return G[(long long)i * ldg + j] + (i == j ? shift : 0.0);
  return L[(long long)i * ldl + j];
}

// Dual candidates (gridDim.x == 2): CTA 0 factors G + shift·I into (L, Dinv, status), CTA 1
// factors G + shift_factor·trace(G)·I into (L1, Dinv1, status1) at the same time — the
// shifted CholeskyQR fallback is then ready without a second launch and host round trip.
template <int kNT>
__global__ void __launch_bounds__(kNT, 1)
    chol_blocked_kernel(const double* __restrict__ G, long long ldg, int m, double shift, double* L,
                        long long ldl, double* Dinv, double* status, double shift_factor, double* L1,
                        double* Dinv1, double* status1) {
  extern __shared__ double sm[];
  double* P = sm;                      // panel rows × kFL
  double* Di = sm + (size_t)max(m, kFB) * kFL;   // current inv(L_jj), 32 × 33
  __shared__ int info_s;
  __shared__ double red[32];
  __shared__ __align__(16) double colb[kFB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kNW = kNT / 32;
  double tr = 0.0;
  for (int i = tid; i < m; i += kNT) tr += G[(long long)i * ldg + i];
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  if (tid == 0) info_s = 0;
  __syncthreads();
  double trace_all = 0.0;
  for (int w = 0; w < kNW; ++w) trace_all += red[w];
  if (blockIdx.x == 1) {   // the shifted candidate (fixed-order trace: same value in both CTAs)
    shift = shift_factor * trace_all;
    L = L1;
    Dinv = Dinv1;
    status = status1;
  }
  if (tid == 0) {
    status[1] = trace_all;
    status[4] = shift;
  }
  long long tc0 = clock64();
  for (int p0 = 0; p0 < m; p0 += kFB) {
    const int nb = min(kFB, m - p0);
    const int rows = m - p0;
    const bool first = p0 == 0;
    const long long ta = clock64();
    // ---- stage the panel (rows × 32) in shared memory: 8 loads in flight per thread
    {
      const int tot = rows * kFB;
      for (int e0 = tid; e0 < tot; e0 += kNT * 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kNT, r = e >> 5, c = e & 31;
          v[u] = (e < tot && c < nb && c <= r) ? chol_src(G, ldg, L, ldl, first, shift, p0 + r, p0 + c) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kNT;
          if (e < tot) P[(e >> 5) * kFL + (e & 31)] = v[u];
        }
      }
    }
    __syncthreads();
    // ---- diagonal block: warp 0, lane i owns row i in registers.  The block
    //      is padded to 32×32 with the identity so no step needs a predicate;
    //      column j is broadcast through shared memory (one LDS per two
    //      entries) — compact code: the whole phase stays in the i-cache.
    if (warp == 0) {
      double d[kFB];
#pragma unroll
      for (int k = 0; k < kFB; ++k)
        d[k] = (lane < nb && k < nb) ? (k <= lane ? P[lane * kFL + k] : 0.0) : (lane == k ? 1.0 : 0.0);
      double rdl = 0.0;  // 1 / L_ll of this lane's row
#pragma unroll
      for (int j = 0; j < kFB; ++j) {
        const double piv = __shfl_sync(0xffffffffu, d[j], j);
        if (lane == 0 && (!(piv > 0.0) || !isfinite(piv)) && info_s == 0 && j < nb) info_s = p0 + j + 1;
        const double inv = rsqrt(fmax(piv, 1e-300));
        d[j] = (lane == j) ? piv * inv : d[j] * inv;
        if (lane == j) rdl = inv;
        colb[lane] = d[j];
        __syncwarp();
#pragma unroll
        for (int k = j + 1; k < kFB; ++k) d[k] = fma(-d[j], colb[k], d[k]);   // upper entries: don't-care
        __syncwarp();
      }
#pragma unroll
      for (int k = 0; k < kFB; ++k) P[lane * kFL + k] = (lane < nb && k <= lane) ? d[k] : 0.0;
      colb[lane] = rdl;
      __syncwarp();
      // inverse of the (padded) diagonal block: lane c → column c,
      // x_r = (δ_rc − Σ_{k<r} L_rk x_k) / L_rr ; x_r = 0 for r < c falls out.
      double x[kFB];
      const int c = lane;
#pragma unroll
      for (int r = 0; r < kFB; ++r) {
        double s0 = (r == c) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
        for (int k = 0; k + 1 < r; k += 2) {
          s0 = fma(-P[r * kFL + k], x[k], s0);
          s1 = fma(-P[r * kFL + k + 1], x[k + 1], s1);
        }
        if (r & 1) s0 = fma(-P[r * kFL + r - 1], x[r - 1], s0);
        x[r] = (s0 + s1) * colb[r];
      }
#pragma unroll
      for (int r = 0; r < kFB; ++r) {
        const double v = (r < nb && c < nb) ? x[r] : 0.0;
        Di[r * (kFB + 1) + c] = v;
        Dinv[((size_t)(p0 / kFB) * kFB + r) * kFB + c] = v;
      }
    }
    __syncthreads();
    const long long tb_ = clock64();
    // ---- panel below: L21 = A21 · Dinvᵀ on DMMA (8×8 output blocks).  Rows are
    //      independent, so waves of 16 row-blocks are computed into registers,
    //      then written back in place after a barrier.
    {
      const int rb_n = (rows - nb + 7) / 8;   // 8-row blocks below the diagonal block
      const int g = lane >> 2, t = lane & 3;
      constexpr int kU = 8;                   // blocks per warp per wave
      const int nblk = rb_n * 4;
      for (int base = 0; base < nblk; base += kNW * kU) {
        double o[kU][2];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int bidx = base + warp + u * kNW;
          double c0 = 0.0, c1 = 0.0;
          if (bidx < nblk) {
            const int ra = nb + 8 * (bidx >> 2) + g, cb = bidx & 3;
#pragma unroll
            for (int k0 = 0; k0 < kFB; k0 += 4) {
              const double av = (ra < rows) ? P[ra * kFL + k0 + t] : 0.0;
              const double bv = Di[(8 * cb + g) * (kFB + 1) + k0 + t];   // (Dinvᵀ)[k][n] = Dinv[n][k]
              dmma_8x8x4(c0, c1, av, bv);
            }
          }
          o[u][0] = c0;
          o[u][1] = c1;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int bidx = base + warp + u * kNW;
          if (bidx < nblk) {
            const int ra = nb + 8 * (bidx >> 2) + g, col = 8 * (bidx & 3) + 2 * t;
            if (ra < rows) {
              P[ra * kFL + col] = (col < nb) ? o[u][0] : 0.0;
              P[ra * kFL + col + 1] = (col + 1 < nb) ? o[u][1] : 0.0;
            }
          }
        }
        __syncthreads();
      }
    }
    // store the factored panel (zeros above the diagonal of the panel columns)
    for (int e = tid; e < m * kFB; e += kNT) {
      const int r = e >> 5, c = e & 31;
      if (c < nb) {
        const int rl = r - p0;
        L[(long long)r * ldl + p0 + c] = (rl >= c) ? P[rl * kFL + c] : 0.0;
      }
    }
    const long long tcc = clock64();
    // ---- trailing update A22 −= L21 L21ᵀ (lower 8×8 blocks) on DMMA; block row bi → warp
    //      bi mod 8, eight blocks per round, all their loads issued before the MMAs
    const int t0 = p0 + nb, tn = m - t0;
    if (tn > 0) {
      const int tbn = (tn + 7) / 8;
      const int g = lane >> 2, t = lane & 3;
      for (int bi = warp; bi < tbn; bi += kNW) {
        const int ii = t0 + 8 * bi + g;
        const int ra = nb + 8 * bi + g;
        double afr[kFB / 4];
#pragma unroll
        for (int k0 = 0; k0 < kFB / 4; ++k0) afr[k0] = (ra < rows) ? P[ra * kFL + 4 * k0 + t] : 0.0;
        for (int bj0 = 0; bj0 <= bi; bj0 += 8) {
          double cv[8][2];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int jj = t0 + 8 * (bj0 + u) + 2 * t + e;
              cv[u][e] = (bj0 + u <= bi && ii < m && jj <= ii) ? chol_src(G, ldg, L, ldl, first, shift, ii, jj) : 0.0;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (bj0 + u > bi) break;
            const int rb = nb + 8 * (bj0 + u) + g;
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int k0 = 0; k0 < kFB / 4; ++k0) {
              const double bb = (rb < rows) ? P[rb * kFL + 4 * k0 + t] : 0.0;
              dmma_8x8x4(c0, c1, afr[k0], bb);
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int jj = t0 + 8 * (bj0 + u) + 2 * t + e;
              if (ii < m && jj <= ii) L[(long long)ii * ldl + jj] = cv[u][e] - (e ? c1 : c0);
            }
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      const long long td = clock64();
      g_chol_t[1] += tb_ - ta;
      g_chol_t[2] += tcc - tb_;
      g_chol_t[3] += td - tcc;
    }
  }
  if (tid == 0) g_chol_t[0] += clock64() - tc0;
  double dmin = INFINITY, dmax = 0.0;
  for (int i = tid; i < m; i += kNT) {
    const double dd = L[(long long)i * ldl + i];
    dmin = fmin(dmin, dd);
    dmax = fmax(dmax, dd);
  }
  for (int o = 16; o > 0; o >>= 1) {
    dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  __shared__ double rmin[32], rmax[32];
  if (lane == 0) {
    rmin[warp] = dmin;
    rmax[warp] = dmax;
  }
  __syncthreads();
  if (tid == 0) {
    double a = INFINITY, b2 = 0.0;
    for (int w = 0; w < kNW; ++w) {
      a = fmin(a, rmin[w]);
      b2 = fmax(b2, rmax[w]);
    }
    status[0] = (double)info_s;
    status[2] = a;
    status[3] = b2;
  }
}

// Block column j of X = L⁻¹ (rows ≥ j): X_jj = Dinv_j; X_ij = −Dinv_i Σ_{k=j}^{i−1} L_ik X_kj.
// Both products on DMMA (8 warps × two 8×8 output blocks); L_i,[j..i) is
// streamed through shared memory in 128-column chunks.  Writes
// Rinv[j-block rows][c] = X[c][j-block cols] (Rinv = Xᵀ), zero elsewhere.
constexpr int kTiChunk = 128;
constexpr int kTiLdL = kTiChunk + 4;
constexpr int kTiLdX = kFB + 4;
__global__ void __launch_bounds__(256) tri_inv_blocked_kernel(const double* __restrict__ L,
                                                              long long ldl, int m,
                                                              const double* __restrict__ Dinv,
                                                              double* Rinv, long long ldr,
                                                              const double* __restrict__ L1,
                                                              const double* __restrict__ Dinv1,
                                                              double* Rinv1) {
  extern __shared__ double xs[];
  if (blockIdx.y == 1) {   // second candidate of chol_fast_dual
    L = L1;
    Dinv = Dinv1;
    Rinv = Rinv1;
  }
  const int j = blockIdx.x;
  const int nblk = (m + kFB - 1) / kFB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int nk = nblk - j;                              // block rows j..nblk-1 of column block j
  double* X = xs;                                       // nk·32 rows × kTiLdX (row r ↔ global row 32j + r)
  double* Lb = X + (size_t)nk * kFB * kTiLdX;           // 32 × kTiLdL chunk of L_i,[j..i)
  double* Zs = Lb + (size_t)kFB * kTiLdL;               // 32 × kTiLdX
  double* Ds = Zs + (size_t)kFB * kTiLdX;               // 32 × kTiLdX (Dinv_i)
  for (int e = tid; e < kFB * kFB; e += blockDim.x)
    X[(e >> 5) * kTiLdX + (e & 31)] = Dinv[(size_t)j * kFB * kFB + e];
  const int br = warp >> 1, bc0 = 2 * (warp & 1);       // this warp's output blocks: (br, bc0), (br, bc0+1)
  __syncthreads();
  for (int i = j + 1; i < nblk; ++i) {
    const int ri = i * kFB;
    const int K = (i - j) * kFB;                        // columns 32j .. 32i of L's row block i
    double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
    for (int e = tid; e < kFB * kFB; e += blockDim.x)
      Ds[(e >> 5) * kTiLdX + (e & 31)] = Dinv[(size_t)i * kFB * kFB + e];
    for (int k0 = 0; k0 < K; k0 += kTiChunk) {
      const int kc = min(kTiChunk, K - k0);
      for (int e = tid; e < kFB * kTiChunk; e += blockDim.x) {
        const int r = e / kTiChunk, c = e % kTiChunk;
        Lb[r * kTiLdL + c] = (c < kc && ri + r < m) ? L[(long long)(ri + r) * ldl + j * kFB + k0 + c] : 0.0;
      }
      __syncthreads();
      for (int kk = 0; kk < kc; kk += 4) {
        const double av = Lb[(8 * br + g) * kTiLdL + kk + t];
        const double b0 = X[(k0 + kk + t) * kTiLdX + 8 * bc0 + g];
        const double b1 = X[(k0 + kk + t) * kTiLdX + 8 * (bc0 + 1) + g];
        dmma_8x8x4(z0[0], z0[1], av, b0);
        dmma_8x8x4(z1[0], z1[1], av, b1);
      }
      __syncthreads();
    }
    Zs[(8 * br + g) * kTiLdX + 8 * bc0 + 2 * t] = z0[0];
    Zs[(8 * br + g) * kTiLdX + 8 * bc0 + 2 * t + 1] = z0[1];
    Zs[(8 * br + g) * kTiLdX + 8 * (bc0 + 1) + 2 * t] = z1[0];
    Zs[(8 * br + g) * kTiLdX + 8 * (bc0 + 1) + 2 * t + 1] = z1[1];
    __syncthreads();
    // X_ij = −Dinv_i · Z
    double w0[2] = {0.0, 0.0}, w1[2] = {0.0, 0.0};
#pragma unroll
    for (int kk = 0; kk < kFB; kk += 4) {
      const double av = Ds[(8 * br + g) * kTiLdX + kk + t];
      const double b0 = Zs[(kk + t) * kTiLdX + 8 * bc0 + g];
      const double b1 = Zs[(kk + t) * kTiLdX + 8 * (bc0 + 1) + g];
      dmma_8x8x4(w0[0], w0[1], av, b0);
      dmma_8x8x4(w1[0], w1[1], av, b1);
    }
    double* Xi = X + (size_t)(i - j) * kFB * kTiLdX;
    Xi[(8 * br + g) * kTiLdX + 8 * bc0 + 2 * t] = -w0[0];
    Xi[(8 * br + g) * kTiLdX + 8 * bc0 + 2 * t + 1] = -w0[1];
    Xi[(8 * br + g) * kTiLdX + 8 * (bc0 + 1) + 2 * t] = -w1[0];
    Xi[(8 * br + g) * kTiLdX + 8 * (bc0 + 1) + 2 * t + 1] = -w1[1];
    __syncthreads();
  }
  // Rinv rows [32j, 32j+32) = X[:, j-block]ᵀ  (row < 32j → 0)
  const int cj = j * kFB;
  for (int e = tid; e < kFB * m; e += blockDim.x) {
    const int c = e / m, row = e % m;   // Rinv[cj + c][row] = X[row][cj + c]
    if (cj + c >= m) continue;
    const double v = (row >= cj) ? X[(row - cj) * kTiLdX + c] : 0.0;
    Rinv[(long long)(cj + c) * ldr + row] = v;
  }
}

int chol_fast(const double* G, long long ldg, int m, double shift, double* L, long long ldl,
              double* Rinv, long long ldr, double* Dinv, double* status, cudaStream_t st,
              double shift_factor, double* L1, double* Rinv1, double* Dinv1, double* status1) {
  const size_t smem1 = ((size_t)std::max(m, kFB) * kFL + kFB * (kFB + 1)) * sizeof(double);
  const int nblk = (m + kFB - 1) / kFB;
  const size_t smem2 = ((size_t)nblk * kFB * kTiLdX + kFB * kTiLdL + 2 * kFB * kTiLdX) * sizeof(double);
  if (smem1 > device_info().max_smem - 4096 || smem2 > device_info().max_smem - 1024) return -1;
  static size_t attr1[16] = {}, attr2[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem1 > attr1[dev]) {
    cudaFuncSetAttribute(chol_blocked_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    cudaFuncSetAttribute(chol_blocked_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
    attr1[dev] = smem1;
  }
  if (smem2 > attr2[dev]) {
    cudaFuncSetAttribute(tri_inv_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem2);
    attr2[dev] = smem2;
  }
  static const bool timers = getenv("PSD_CHOL_TIMERS") != nullptr;
  if (timers) {
    const long long z[6] = {0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbolAsync(g_chol_t, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  }
  const bool dual = L1 != nullptr;
  // 16 warps: the TRSM and trailing-update rounds per warp (dependent global round trips) halve
  static const int chol_nt = [] { const char* e = getenv("PSD_CHOL_NT"); return e ? atoi(e) : 512; }();
  if (chol_nt == 512 && m > 64)
    chol_blocked_kernel<512><<<dual ? 2 : 1, 512, smem1, st>>>(G, ldg, m, shift, L, ldl, Dinv, status,
                                                             shift_factor, L1, Dinv1, status1);
  else
    chol_blocked_kernel<256><<<dual ? 2 : 1, 256, smem1, st>>>(G, ldg, m, shift, L, ldl, Dinv, status,
                                                             shift_factor, L1, Dinv1, status1);
  count_launch();
  tri_inv_blocked_kernel<<<dim3(nblk, dual ? 2 : 1), 256, smem2, st>>>(L, ldl, m, Dinv, Rinv, ldr, L1,
                                                                     Dinv1, Rinv1);
  count_launch();
  if (timers) {
    long long h[6];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_chol_t, sizeof(h));
    fprintf(stderr, "chol m=%d cycles: total %lld diag %lld trsm+store %lld trailing %lld\n", m, h[0],
            h[1], h[2], h[3]);
  }
  return 0;
}

}  // namespace psd
