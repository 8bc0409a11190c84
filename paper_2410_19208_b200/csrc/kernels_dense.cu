// Small dense (w×w) kernels: blocked Cholesky for CholeskyQR, triangular
// inverse, block-Jacobi symmetric eigensolver (symmetric.py:68-86 semantics)
// and the descending sort / sign convention.
#include <algorithm>
#include <cmath>
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
  if (threadIdx.x == 0) pos_count = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double li = vals[i];
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      const double lj = vals[j];
      rank += (lj > li) || (lj == li && j < i);
    }
    perm[rank] = i;
    vals_out[rank] = li;
    if (li - offset > 0.0) atomicAdd(&pos_count, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) npos[0] = pos_count;
  // orientation + column permutation: one warp per output column
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int col = warp; col < m; col += blockDim.x >> 5) {
    const int src = perm[col];
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int r = lane; r < m; r += 32) {
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
    const double anchor = vecs[(long long)bidx * ldv + src];
    const double sg = (anchor < 0.0) ? -1.0 : 1.0;
    for (int r = lane; r < m; r += 32) vecs_out[(long long)r * ldo + col] = sg * vecs[(long long)r * ldv + src];
  }
}

void sort_eigs(const double* vals, const double* vecs, long long ldv, int m, double offset,
               double* vals_out, double* vecs_out, long long ldo, int* npos, int* perm,
               cudaStream_t st) {
  sort_eigs_kernel<<<1, 1024, 0, st>>>(vals, vecs, ldv, m, offset, vals_out, vecs_out, ldo, npos,
                                       perm);
  count_launch();
}

}  // namespace psd
