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
// Block-Jacobi eigensolver.  Blocks of JB indices; each round pairs blocks
// (circle method) and every pair's 2JB×2JB principal submatrix is rotated
// towards diagonal form by one CTA in shared memory (cyclic parallel Jacobi),
// producing an orthogonal J_pair.  A second launch applies Jᵀ A J to all
// tile pairs and V ← V J.  A sweep with no rotation above threshold ends it.
// ---------------------------------------------------------------------------
constexpr int kJB = 16;
constexpr int kSub = 2 * kJB;

struct JacobiGeom {
  int m, nblk, P, round;
};

PSD_DEVINL void round_pair(int nblk, int r, int i, int& a, int& b) {
  const int M = nblk - 1;
  if (i == 0) {
    a = M;
    b = r % M;
  } else {
    a = (r + i) % M;
    b = (r - i + M) % M;
  }
}

PSD_DEVINL int sub_index(int nblk, int r, int pair, int k) {
  int a, b;
  round_pair(nblk, r, pair, a, b);
  return (k < kJB) ? a * kJB + k : b * kJB + (k - kJB);
}

// inner cyclic Jacobi on a kSub×kSub matrix in smem; returns #rotations
__device__ int inner_jacobi(double (*S)[kSub + 1], double (*V)[kSub + 1], int sweeps, double abs_tol,
                            double* cs, double* sn, double* tt) {
  __shared__ int rot_count;
  if (threadIdx.x == 0) rot_count = 0;
  __syncthreads();
  int total = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    for (int r = 0; r < kSub - 1; ++r) {
      if (threadIdx.x < kSub / 2) {
        int p, q;
        round_pair(kSub, r, threadIdx.x, p, q);
        const double app = S[p][p], aqq = S[q][q], apq = S[p][q];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > abs_tol && fabs(apq) > 1e-15 * sqrt(fabs(app * aqq))) {
          const double tau = (aqq - app) / (2.0 * apq);
          t = (tau >= 0.0) ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                           : -1.0 / (-tau + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + t * t);
          s = t * c;
          atomicAdd(&rot_count, 1);
        }
        cs[threadIdx.x] = c;
        sn[threadIdx.x] = s;
        tt[threadIdx.x] = t;
      }
      __syncthreads();
      // rows p,q (Jᵀ A)
      for (int idx = threadIdx.x; idx < (kSub / 2) * kSub; idx += blockDim.x) {
        const int k = idx / kSub, j = idx % kSub;
        if (sn[k] == 0.0) continue;
        int p, q;
        round_pair(kSub, r, k, p, q);
        const double c = cs[k], s = sn[k];
        const double sp = S[p][j], sq = S[q][j];
        S[p][j] = c * sp - s * sq;
        S[q][j] = s * sp + c * sq;
      }
      __syncthreads();
      // columns p,q (A J) and V ← V J
      for (int idx = threadIdx.x; idx < (kSub / 2) * kSub; idx += blockDim.x) {
        const int k = idx / kSub, i = idx % kSub;
        if (sn[k] == 0.0) continue;
        int p, q;
        round_pair(kSub, r, k, p, q);
        const double c = cs[k], s = sn[k];
        const double sp = S[i][p], sq = S[i][q];
        S[i][p] = c * sp - s * sq;
        S[i][q] = s * sp + c * sq;
        const double vp = V[i][p], vq = V[i][q];
        V[i][p] = c * vp - s * vq;
        V[i][q] = s * vp + c * vq;
      }
      __syncthreads();
      if (threadIdx.x < kSub / 2 && sn[threadIdx.x] != 0.0) {
        int p, q;
        round_pair(kSub, r, threadIdx.x, p, q);
        S[p][q] = 0.0;
        S[q][p] = 0.0;
      }
      __syncthreads();
    }
    const int rc = rot_count;
    __syncthreads();
    if (threadIdx.x == 0) rot_count = 0;
    __syncthreads();
    total += rc;
    if (rc == 0) break;
  }
  return total;
}

__global__ void __launch_bounds__(256) jacobi_solve_kernel(const double* __restrict__ a,
                                                           long long lda, int m, int nblk,
                                                           int round, int sweeps,
                                                           const double* norm, double* jbuf,
                                                           double* sbuf, int* dflags) {
  __shared__ double S[kSub][kSub + 1];
  __shared__ double V[kSub][kSub + 1];
  __shared__ double cs[kSub / 2], sn[kSub / 2], tt[kSub / 2];
  __shared__ int idx_s[kSub];
  const int pair = blockIdx.x;
  if (threadIdx.x < kSub) idx_s[threadIdx.x] = sub_index(nblk, round, pair, threadIdx.x);
  __syncthreads();
  for (int e = threadIdx.x; e < kSub * kSub; e += blockDim.x) {
    const int i = e / kSub, j = e % kSub;
    const int gi = idx_s[i], gj = idx_s[j];
    S[i][j] = (gi < m && gj < m) ? a[(long long)gi * lda + gj] : 0.0;
    V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double abs_tol = 1e-18 * norm[0];
  const int rots = inner_jacobi(S, V, sweeps, abs_tol, cs, sn, tt);
  double* J = jbuf + (size_t)pair * kSub * kSub;
  double* Sout = sbuf + (size_t)pair * kSub * kSub;
  for (int e = threadIdx.x; e < kSub * kSub; e += blockDim.x) {
    J[e] = V[e / kSub][e % kSub];
    Sout[e] = S[e / kSub][e % kSub];
  }
  if (threadIdx.x == 0 && rots > 0) atomicAdd(dflags, rots);
}

// blocks [0, P*P): A_new[Ia, Ib] = J_aᵀ A[Ia, Ib] J_b ; blocks [P*P, ...): V[:, Ib] ← V[:, Ib] J_b
__global__ void __launch_bounds__(256) jacobi_apply_kernel(const double* __restrict__ a,
                                                           long long lda, double* anew,
                                                           long long ldn, int m,
                                                           int nblk, int round,
                                                           const double* __restrict__ jbuf,
                                                           const double* __restrict__ sbuf,
                                                           double* v, long long ldv) {
  __shared__ double T[kSub][kSub + 1];
  __shared__ double U[kSub][kSub + 1];
  __shared__ double Jb[kSub][kSub + 1];
  __shared__ int ia[kSub], ib[kSub];
  const int P = nblk / 2;
  const int bid = blockIdx.x;
  if (bid < P * P) {
    const int pa = bid / P, pb = bid % P;
    if (threadIdx.x < kSub) {
      ia[threadIdx.x] = sub_index(nblk, round, pa, threadIdx.x);
      ib[threadIdx.x] = sub_index(nblk, round, pb, threadIdx.x);
    }
    __syncthreads();
    if (pa == pb) {
      // the solve kernel's rotated subproblem: exact zeros on rotated pairs,
      // no GEMM rounding mixed into the diagonal block
      const double* Sp = sbuf + (size_t)pa * kSub * kSub;
      for (int e = threadIdx.x; e < kSub * kSub; e += blockDim.x) {
        const int gi = ia[e / kSub], gj = ib[e % kSub];
        if (gi < m && gj < m) anew[(long long)gi * ldn + gj] = Sp[e];
      }
      return;
    }
    const double* Ja = jbuf + (size_t)pa * kSub * kSub;
    const double* Jbp = jbuf + (size_t)pb * kSub * kSub;
    for (int e = threadIdx.x; e < kSub * kSub; e += blockDim.x) {
      const int i = e / kSub, j = e % kSub;
      const int gi = ia[i], gj = ib[j];
      T[i][j] = (gi < m && gj < m) ? a[(long long)gi * lda + gj] : 0.0;
      U[i][j] = Ja[e];   // J_a[i][j]
      Jb[i][j] = Jbp[e];
    }
    __syncthreads();
    // W = J_aᵀ T  → store in registers then reuse T
    double wv[kSub * kSub / 256];
#pragma unroll
    for (int u = 0; u < kSub * kSub / 256; ++u) {
      const int e = threadIdx.x + u * 256;
      const int i = e / kSub, j = e % kSub;
      double s = 0.0;
#pragma unroll 8
      for (int k = 0; k < kSub; ++k) s = fma(U[k][i], T[k][j], s);
      wv[u] = s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kSub * kSub / 256; ++u) {
      const int e = threadIdx.x + u * 256;
      T[e / kSub][e % kSub] = wv[u];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kSub * kSub / 256; ++u) {
      const int e = threadIdx.x + u * 256;
      const int i = e / kSub, j = e % kSub;
      double s = 0.0;
#pragma unroll 8
      for (int k = 0; k < kSub; ++k) s = fma(T[i][k], Jb[k][j], s);
      const int gi = ia[i], gj = ib[j];
      if (gi < m && gj < m) anew[(long long)gi * ldn + gj] = s;
    }
  } else {
    const int vb = bid - P * P;
    const int pb = vb % P;
    const int r0 = (vb / P) * kSub;
    if (threadIdx.x < kSub) ib[threadIdx.x] = sub_index(nblk, round, pb, threadIdx.x);
    __syncthreads();
    const double* Jbp = jbuf + (size_t)pb * kSub * kSub;
    for (int e = threadIdx.x; e < kSub * kSub; e += blockDim.x) {
      const int i = e / kSub, j = e % kSub;
      const int gr = r0 + i, gj = ib[j];
      T[i][j] = (gr < m && gj < m) ? v[(long long)gr * ldv + gj] : 0.0;
      Jb[i][j] = Jbp[e];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kSub * kSub / 256; ++u) {
      const int e = threadIdx.x + u * 256;
      const int i = e / kSub, j = e % kSub;
      double s = 0.0;
#pragma unroll 8
      for (int k = 0; k < kSub; ++k) s = fma(T[i][k], Jb[k][j], s);
      const int gr = r0 + i, gj = ib[j];
      if (gr < m && gj < m) v[(long long)gr * ldv + gj] = s;
    }
  }
}

__global__ void frob_norm_kernel(const double* a, long long lda, int m, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) {
    const double x = a[(e / m) * lda + e % m];
    s = fma(x, x, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[0] = sqrt(t);
  }
}

__global__ void diag_extract_kernel(const double* a, long long lda, int m, double* vals) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) vals[i] = a[(long long)i * lda + i];
}

size_t jacobi_ws_elems(int m) {
  const int nblk0 = (m + kJB - 1) / kJB;
  const int nblk = nblk0 + (nblk0 & 1);
  const int P = std::max(1, nblk / 2);
  return (size_t)m * m + (size_t)2 * P * kSub * kSub + 8;
}

int jacobi_eigh(double* a, long long lda, int m, double* values, double* v, long long ldv,
                double* ws, size_t ws_elems, int* dflags, cudaStream_t st) {
  if (m == 1) {
    cudaMemcpyAsync(values, a, sizeof(double), cudaMemcpyDeviceToDevice, st);
    set_identity(v, ldv, 1, st);
    return 1;
  }
  const int nblk0 = (m + kJB - 1) / kJB;
  const int nblk = std::max(2, nblk0 + (nblk0 & 1));
  const int P = nblk / 2;
  if (ws_elems < jacobi_ws_elems(m)) return -2;
  double* anew = ws;                       // m×m, ld m
  double* jbuf = ws + (size_t)m * m;       // P × kSub² rotations
  double* sbuf = jbuf + (size_t)P * kSub * kSub;  // P × kSub² rotated subproblems
  double* norm = sbuf + (size_t)P * kSub * kSub;
  set_identity(v, ldv, m, st);
  frob_norm_kernel<<<1, 1024, 0, st>>>(a, lda, m, norm);
  count_launch();
  double* cur = a;
  long long ldcur = lda;
  double* nxt = anew;
  long long ldnxt = m;
  const int rounds = nblk - 1;
  const int inner = (P == 1) ? 30 : 1;
  const int vchunks = (m + kSub - 1) / kSub;
  int sweep = 0;
  bool converged = false;
  int h_rot = 0;
  for (sweep = 0; sweep < 40 && !converged; ++sweep) {
    cudaMemsetAsync(dflags, 0, sizeof(int), st);
    for (int r = 0; r < rounds; ++r) {
      jacobi_solve_kernel<<<P, 256, 0, st>>>(cur, ldcur, m, nblk, r, inner, norm, jbuf, sbuf,
                                             dflags);
      count_launch();
      jacobi_apply_kernel<<<P * P + P * vchunks, 256, 0, st>>>(cur, ldcur, nxt, ldnxt, m, nblk, r,
                                                               jbuf, sbuf, v, ldv);
      count_launch();
      std::swap(cur, nxt);
      std::swap(ldcur, ldnxt);
    }
    cudaMemcpyAsync(&h_rot, dflags, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (h_rot == 0) converged = true;
  }
  diag_extract_kernel<<<(m + 255) / 256, 256, 0, st>>>(cur, ldcur, m, values);
  count_launch();
  if (cur != a) copy_matrix(cur, ldcur, a, lda, m, m, st);
  return converged ? sweep : -1;
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
