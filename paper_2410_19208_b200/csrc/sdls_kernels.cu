// Solver-loop kernels (sdls.py:76-89, :221-245; BASELINE config 5):
// sparse dual assembly, traces against the factored projection, and the
// gradient-ascent step.  X₊ is never materialised inside the loop:
// Tr(A_i X₊) is evaluated from X₊ = sym((W·D)·Wᵀ) on the constraint's
// nonzeros only.
#include <algorithm>

#include "launch.h"

namespace psd {

// x[pos] = cr[pos] + Σ_t y[econ[t]]·evals[t] for t ∈ [ptr[p], ptr[p+1]) in
// stored order (x already holds a copy of C/ρ).
__global__ void sdls_scatter_kernel(const long long* __restrict__ pos, const int* __restrict__ ptr,
                                    const int* __restrict__ econ,
                                    const double* __restrict__ evals,
                                    const double* __restrict__ y, int npos, double* x) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npos) return;
  double s = 0.0;
  for (int t = ptr[p]; t < ptr[p + 1]; ++t) s = fma(y[econ[t]], evals[t], s);
  x[pos[p]] += s;
}

void sdls_assemble(const double* cr, long long n, const long long* pos, const int* ptr,
                   const int* econ, const double* evals, const double* y, int npos, double* x,
                   cudaStream_t st) {
  cudaMemcpyAsync(x, cr, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (npos > 0) {
    sdls_scatter_kernel<<<(npos + 255) / 256, 256, 0, st>>>(pos, ptr, econ, evals, y, npos, x);
    count_launch();
  }
}

// One warp per constraint: t_i = Σ_{entries} v · ½(M[a][b] + M[b][a]),
// M = (W·D)·Wᵀ restricted to the entry (projection.py:78 symmetrisation).
__global__ void sdls_traces_kernel(const double* __restrict__ wd, const double* __restrict__ w,
                                   long long ldw, int r, const int* __restrict__ rows,
                                   const int* __restrict__ cols, const double* __restrict__ vals,
                                   const int* __restrict__ cptr, int m, double* __restrict__ t) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  double acc = 0.0;
  for (int e = cptr[warp]; e < cptr[warp + 1]; ++e) {
    const long long a = rows[e], b = cols[e];
    double sab = 0.0, sba = 0.0;
    for (int k = lane; k < r; k += 32) {
      sab = fma(wd[a * ldw + k], w[b * ldw + k], sab);
      sba = fma(wd[b * ldw + k], w[a * ldw + k], sba);
    }
    sab = warp_sum(sab);
    sba = warp_sum(sba);
    acc = fma(vals[e], (sab + sba) / 2.0, acc);
  }
  if (lane == 0) t[warp] = acc;
}

void sdls_traces(const double* wd, const double* w, long long ldw, int r, const int* rows,
                 const int* cols, const double* vals, const int* cptr, int m, double* t,
                 cudaStream_t st) {
  if (m <= 0) return;
  const int warps_per_block = 8;
  sdls_traces_kernel<<<(m + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
      wd, w, ldw, r, rows, cols, vals, cptr, m, t);
  count_launch();
}

// One warp per constraint: t_i = Σ_{entries} v·X[a][b] on a dense n×n X
// (constraint_traces, sdls.py:76-80, for the exact / polar projectors whose
// result is formed densely); the lanes split the entries, fixed-order warp sum.
__global__ void sdls_traces_dense_kernel(const double* __restrict__ x, long long ldx,
                                         const int* __restrict__ rows, const int* __restrict__ cols,
                                         const double* __restrict__ vals,
                                         const int* __restrict__ cptr, int m, double* __restrict__ t) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  double acc = 0.0;
  for (int e = cptr[warp] + lane; e < cptr[warp + 1]; e += 32)
    acc = fma(vals[e], x[(long long)rows[e] * ldx + cols[e]], acc);
  acc = warp_sum(acc);
  if (lane == 0) t[warp] = acc;
}

void sdls_traces_dense(const double* x, long long ldx, const int* rows, const int* cols,
                       const double* vals, const int* cptr, int m, double* t, cudaStream_t st) {
  if (m <= 0) return;
  const int warps_per_block = 8;
  sdls_traces_dense_kernel<<<(m + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0,
                             st>>>(x, ldx, rows, cols, vals, cptr, m, t);
  count_launch();
}

// grad = b − t; out[0] = ‖grad‖₂ (fixed-order reduction); if out[0] > eps:
// y ← y + β·grad (sdls.py:236-245).  Single block.
__global__ void sdls_step_kernel(const double* __restrict__ b, const double* __restrict__ t,
                                 double* __restrict__ y, double* __restrict__ grad, int m,
                                 double beta, double eps, double* out) {
  __shared__ double red[32];
  __shared__ double nrm_s;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double g = b[i] - t[i];
    grad[i] = g;
    s = fma(g, g, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    nrm_s = sqrt(tot);
    out[0] = nrm_s;
  }
  __syncthreads();
  if (nrm_s > eps)
    for (int i = threadIdx.x; i < m; i += blockDim.x) y[i] = y[i] + beta * grad[i];
}

void sdls_step(const double* b, const double* t, double* y, double* grad, int m, double beta,
               double eps, double* out, cudaStream_t st) {
  sdls_step_kernel<<<1, 1024, 0, st>>>(b, t, y, grad, m, beta, eps, out);
  count_launch();
}

}  // namespace psd
