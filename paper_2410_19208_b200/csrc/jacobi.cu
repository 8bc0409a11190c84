// Symmetric eigensolver for the k×k compressed matrix T = sym(QᵀXQ)
// (symmetric.py:68-86 via projection.py:105): block-cyclic two-sided Jacobi
// in ONE persistent cooperative kernel.
//
// The m×m matrix is cut into 16-index blocks; every round the circle method
// pairs the blocks and each pair's 32×32 principal submatrix is rotated by
// one CTA in shared memory.  A parallel Jacobi step is one phase with one
// barrier: every warp recomputes the step's 16 rotations redundantly (lane
// l ↔ pair l, broadcast by shuffles, no shared-memory hand-off), then each
// thread applies J_kᵀ·[2×2 block]·J_l to its block and to two (row, pair)
// slots of the local rotation product, reading one buffer and writing the
// other.  The CTA's rotation product J_P is applied to the whole matrix
// (A ← Jᵀ A J, V ← V J) by all CTAs as 32×32 DMMA tile products.  Grid-wide
// barriers separate solve and apply; convergence (a sweep with no rotation
// above threshold) is decided on the device: one launch, one host sync.
//
// Per-pair threshold: rotate (p,q) iff |a_pq| > 1e-15·sqrt(|a_pp a_qq|) and
// |a_pq| > 1e-15·‖A‖_F.  Off-diagonal mass left below that bound perturbs
// the reconstructed T₊ by ≲ m·1e-15·‖A‖_F (≈3e-13 relative at m = 272).
// Diagonal sub-blocks are copied from the solve CTA (exact zeros on rotated
// pairs) instead of being re-multiplied.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "launch.h"

namespace psd {

// Block size JB (indices per block) is a template parameter: 16 (32×32 subproblems,
// 256 threads; the default) or 32 (64×64 subproblems, 1024 threads; see jacobi_eigh).
template <int JB>
struct JTraits {
  static constexpr int kJB = JB;             // indices per block
  static constexpr int kJS = 2 * JB;         // subproblem size
  static constexpr int kJT = JB * JB;        // threads per CTA: one per (row pair, column pair)
  static constexpr int kJLd = kJS + 4;       // smem row stride ≡ 4 (mod 16): conflict-free DMMA fragments
  static constexpr int kJTile = kJS * kJLd;
  static constexpr unsigned kMask = JB == 32 ? 0xffffffffu : ((1u << JB) - 1u);
  static constexpr size_t kSmemBytes = (size_t)6 * kJTile * sizeof(double);
};

struct JacobiArgs {
  double* a;        // m×m, ld lda (input; may end up holding the result)
  long long lda;
  double* b;        // m×m scratch, ld m
  double* v;        // m×m eigenvectors, ld ldv
  long long ldv;
  double* jbuf;     // P × kJS²
  double* sbuf;     // P × kJS²
  int* counters;    // per-sweep rotation counts (zeroed)
  unsigned long long* maxoff;   // per sweep: max |a_ij|, i ≠ j, after its last round (double bits, zeroed)
  int* flags;       // dataflow flags: sflag[P], aflag[P²], vflag[P·vch], jread[2P] (zeroed)
  double* norm;     // [0] = ‖A‖_F
  int* out;         // [0] = sweeps (or −1), [1] = 1 if result is in b
  int m, nblk, max_sweeps;
  int inner;        // inner sweeps per pair solve
  long long* timers;  // optional: block 0 clock64 per phase [solve, bar1, apply, bar2]
};

constexpr int kFS = 32;   // flag stride in ints (128 bytes)
#ifndef PSD_JACOBI_BACKOFF
#define PSD_JACOBI_BACKOFF 128
#endif
constexpr unsigned kPollBackoff = PSD_JACOBI_BACKOFF;   // ns between polls of off-critical-path waiters

PSD_DEVINL void circle_pair(int nplayers, int r, int i, int& a, int& b) {
  const int M = nplayers - 1;
  if (i == 0) {
    a = M;
    b = r % M;
  } else {
    a = (r + i) % M;
    b = (r - i + M) % M;
  }
}

template <int JB>
PSD_DEVINL int sub_index(int nblk, int r, int pair, int k) {
  int a, b;
  circle_pair(nblk, r, pair, a, b);
  return (k < JB) ? a * JB + k : b * JB + (k - JB);
}

__device__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gen += 1;
    const unsigned target = gen * gridDim.x;
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned seen;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(seen) : "l"(bar) : "memory");
    } while (seen < target);
  }
  __syncthreads();
}

// Optional task timeline (PSD_JACOBI_TRACE): per (round, task) three %globaltimer stamps —
// task begin, dependencies satisfied, flag released — for critical-path analysis.
__device__ long long* g_jtrace = nullptr;
PSD_DEVINL long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
PSD_DEVINL void jtrace(int R, int ntask, int task, int slot, long long t) {
  long long* tr = g_jtrace;
  if (tr != nullptr && R < 1024) tr[((long long)R * ntask + task) * 3 + slot] = t;
}

// Rotation for pair (p,q) (GVL sym.schur2 in the cos 2θ / sin 2θ form).
PSD_DEVINL bool rotation(double app, double aqq, double apq, double abs_tol, double& c, double& s,
                         double& t) {
  // two reciprocal-square-root chains instead of sqrt + division + rsqrt (the rotation is
  // on the critical path of every inner step): with y = 1/r, r = hypot(d, e),
  // h = (1 + |d|/r)/2 = cos²θ (|θ| ≤ π/4), z = h^-½:  c = h·z, s = ±e·y·z/2, t = s·z = tan θ.
  // Computed unconditionally (the threshold test runs beside the chain, not before it); the
  // clamp keeps rsqrt off its slow path for a zero pair (padding), whose result is discarded.
  const double d = aqq - app, e = 2.0 * apq;
  const double y = rsqrt(fmax(fma(d, d, e * e), 2.2250738585072014e-308));
  const double h = fma(0.5 * fabs(d), y, 0.5);
  const double z = rsqrt(h);
  const bool rot = fabs(apq) > abs_tol && apq * apq > 1e-30 * fabs(app * aqq);
  const double sr = (d >= 0.0 ? 0.5 : -0.5) * e * y * z;
  c = rot ? h * z : 1.0;
  s = rot ? sr : 0.0;
  t = rot ? sr * z : 0.0;
  return rot;
}

// Pair k of inner step ir: full sweep = circle method over 32 indices
// (31 steps), cross sweep = (k, 16 + (k + ir) mod 16) (16 steps).
template <int JB>
PSD_DEVINL void step_pair(bool full, int ir, int k, int& p, int& q) {
  constexpr int kJS = 2 * JB;
  if (full) {
    if (k == 0) {
      p = kJS - 1;
      q = ir;
    } else {
      p = ir + k;
      if (p >= kJS - 1) p -= kJS - 1;
      q = ir - k + kJS - 1;
      if (q >= kJS - 1) q -= kJS - 1;
    }
  } else {
    p = k;
    q = JB + ((k + ir) & (JB - 1));
  }
}

// One parallel step: reads (Sc, Vc), writes every element of (Sn, Vn).
// Returns #rotations (block-uniform); 0 ⇒ nothing written.
template <int JB>
__device__ int jacobi_step(const double* Sc, const double* Vc, double* Sn, double* Vn, bool full,
                           int ir, double abs_tol) {
  using T = JTraits<JB>;
  constexpr int L = T::kJLd;
  const int lane = threadIdx.x & 31;
  const int l = lane & (JB - 1);           // this lane's column rotation (pair l of the step)
  const int k = (int)threadIdx.x / JB;     // thread → (k, l): rows {p_k, q_k} × cols {p_l, q_l}
  int p, q, pk, qk;
  step_pair<JB>(full, ir, l, p, q);
  step_pair<JB>(full, ir, k, pk, qk);
  // every shared-memory read of the step issued up front (they depend on the indices only),
  // so the step's critical path is one LDS round, the rotation chain, the shuffles, the 2×2
  // products and the barrier.  (Computing rotation k in this thread too, instead of the
  // shuffles, measured slower: the rotation is MUFU/FP64-throughput-heavy.)
  const double lpp = Sc[p * L + p], lqq = Sc[q * L + q], lpq = Sc[p * L + q];
  double b00 = Sc[pk * L + p], b01 = Sc[pk * L + q];
  double b10 = Sc[qk * L + p], b11 = Sc[qk * L + q];
  const double v00 = Vc[k * L + p], v01 = Vc[k * L + q];
  const double v10 = Vc[(k + JB) * L + p], v11 = Vc[(k + JB) * L + q];
  double c, s, t;
  const bool r = rotation(lpp, lqq, lpq, abs_tol, c, s, t);
  const int nrot = __popc(__ballot_sync(0xffffffffu, r) & T::kMask);
  if (nrot == 0) return 0;
  // lane k of every warp holds rotation k (k < JB ≤ 32)
  const double ck = __shfl_sync(0xffffffffu, c, k & (JB - 1));
  const double sk = __shfl_sync(0xffffffffu, s, k & (JB - 1));
  // for k == l the rotated pair's own entries are (b00, b11, b01) = (a_pp, a_qq, a_pq)
  const double kpp = b00, kqq = b11, kpq = b01;
  // Jₖᵀ·(B·J_l): the column rotation (own c, s) overlaps the shuffles' latency
  const double r00 = c * b00 - s * b01, r01 = s * b00 + c * b01;
  const double r10 = c * b10 - s * b11, r11 = s * b10 + c * b11;
  b00 = ck * r00 - sk * r10;
  b01 = ck * r01 - sk * r11;
  b10 = sk * r00 + ck * r10;
  b11 = sk * r01 + ck * r11;
  if (k == l && sk != 0.0) {  // the rotated pair itself: exact form from its tan θ
    b00 = kpp - t * kpq;
    b11 = kqq + t * kpq;
    b01 = 0.0;
    b10 = 0.0;
  }
  Sn[pk * L + p] = b00;
  Sn[pk * L + q] = b01;
  Sn[qk * L + p] = b10;
  Sn[qk * L + q] = b11;
  // V ← V J for rows k and k + JB, pair l
  Vn[k * L + p] = c * v00 - s * v01;
  Vn[k * L + q] = s * v00 + c * v01;
  Vn[(k + JB) * L + p] = c * v10 - s * v11;
  Vn[(k + JB) * L + q] = s * v10 + c * v11;
  __syncthreads();
  return nrot;
}

// C (kJS×kJS) = op(A)·B for A, B in shared memory (row stride kJLd) on the FP64
// tensor cores: warp w owns rows (w mod JB/4)·8 … +8, cols (w div JB/4)·16 … +16.
// aT: A is stored transposed (A[m][k] = Asmem[k][m]).
template <int JB>
PSD_DEVINL void mm_dmma(const double* A, bool aT, const double* B, double (&c)[2][2]) {
  using T = JTraits<JB>;
  constexpr int L = T::kJLd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp % (JB / 4)) * 8, n0 = (warp / (JB / 4)) * 16;
  c[0][0] = c[0][1] = c[1][0] = c[1][1] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < T::kJS; k0 += 4) {
    const double a = aT ? A[(k0 + t) * L + m0 + g] : A[(m0 + g) * L + k0 + t];
    const double b0 = B[(k0 + t) * L + n0 + g];
    const double b1 = B[(k0 + t) * L + n0 + 8 + g];
    dmma_8x8x4(c[0][0], c[0][1], a, b0);
    dmma_8x8x4(c[1][0], c[1][1], a, b1);
  }
}

// Two independent products of the mm_dmma form interleaved (same per-element arithmetic).
template <int JB>
PSD_DEVINL void mm_dmma2(const double* A1, bool a1T, const double* B1, double (&c1)[2][2], const double* A2,
                         bool a2T, const double* B2, double (&c2)[2][2]) {
  using T = JTraits<JB>;
  constexpr int L = T::kJLd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m0 = (warp % (JB / 4)) * 8, n0 = (warp / (JB / 4)) * 16;
  c1[0][0] = c1[0][1] = c1[1][0] = c1[1][1] = 0.0;
  c2[0][0] = c2[0][1] = c2[1][0] = c2[1][1] = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < T::kJS; k0 += 4) {
    const double a1 = a1T ? A1[(k0 + t) * L + m0 + g] : A1[(m0 + g) * L + k0 + t];
    const double a2 = a2T ? A2[(k0 + t) * L + m0 + g] : A2[(m0 + g) * L + k0 + t];
    const double b10 = B1[(k0 + t) * L + n0 + g], b11 = B1[(k0 + t) * L + n0 + 8 + g];
    const double b20 = B2[(k0 + t) * L + n0 + g], b21 = B2[(k0 + t) * L + n0 + 8 + g];
    dmma_8x8x4(c1[0][0], c1[0][1], a1, b10);
    dmma_8x8x4(c1[1][0], c1[1][1], a1, b11);
    dmma_8x8x4(c2[0][0], c2[0][1], a2, b20);
    dmma_8x8x4(c2[1][0], c2[1][1], a2, b21);
  }
}

// (row, col) within the kJS×kJS tile of accumulator (j, e) of this thread
template <int JB>
PSD_DEVINL void mm_coord(int j, int e, int& row, int& col) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  row = (warp % (JB / 4)) * 8 + (lane >> 2);
  col = (warp / (JB / 4)) * 16 + 8 * j + 2 * (lane & 3) + e;
}

// ---- dataflow synchronisation (no grid-wide barrier) -----------------------
// backoff > 0: pause between polls (waiters off the critical path leave the flags' L2
// lines to the solves that poll them on it)
PSD_DEVINL void flag_wait(const int* f, int target, unsigned backoff = 0) {
  int v;
  unsigned spins = 0;
  do {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
    if (v >= target) break;
    if (++spins > (1u << 26)) __trap();   // a dependency that never resolves: fail loudly
    if (backoff) __nanosleep(backoff);
  } while (true);
}
// Called by thread 0 after a __syncthreads that orders the CTA's data writes
// before it; st.release is cumulative over them (PTX memory model).
PSD_DEVINL void flag_set(int* f, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(f), "r"(v) : "memory");
}

// pair index of block x in round R (inverse of circle_pair)
PSD_DEVINL int pair_of(int nblk, int R, int x) {
  const int M = nblk - 1, r = R % M;
  if (x == M) return 0;
  if (x == r) return 0;
  // x = (r + i) mod M  or  x = (r − i) mod M  for i ∈ [1, P)
  const int i1 = (x - r + M) % M;   // x = r + i1
  return i1 < (nblk / 2) ? i1 : M - i1;
}

// One persistent cooperative kernel; every round R = sweep·rounds + r is a set
// of tasks — P pair solves, P² A-items (J_aᵀ A_ab J_b), P·⌈m/64⌉ V-items
// (V ← V·J) — spread over the CTAs.  Instead of grid barriers each task
// waits only on the flags of the tasks it reads from:
//   solve p (R):   the R−1 A-items holding its four blocks;
//   A-item (a,b):  solves a, b of round R + the four R−1 A-items of its blocks;
//   V-item (c,b):  solve b + the two R−1 V-items of its columns;
// and a solve first waits until every reader of its J/S slot (R−2) is done.
template <int JB>
__global__ void __launch_bounds__(JB * JB) jacobi_persistent_kernel(JacobiArgs A) {
  using T = JTraits<JB>;
  constexpr int kJS = T::kJS, kJT = T::kJT, kJLd = T::kJLd, kJTile = T::kJTile;
  extern __shared__ __align__(16) double sm[];
  double* S0 = sm;
  double* V0 = sm + kJTile;
  double* S1 = sm + 2 * kJTile;
  double* V1 = sm + 3 * kJTile;
  double* X = sm + 4 * kJTile;
  double* Y = sm + 5 * kJTile;
  __shared__ int ia[kJS], ib[kJS], ic[kJS];
  __shared__ int stop_flag;
  __shared__ double red8[kJT / 32];
  const int m = A.m, nblk = A.nblk, P = nblk / 2, rounds = nblk - 1;
  const int vch = (m + 2 * kJS - 1) / (2 * kJS);       // 64-row V chunks
  const int ntask = P + P * P + P * vch;
  // tasks reading J_p / S_p of a round: its A-items and V-items, and the next round's
  // solves holding its two blocks (one solve when P = 1)
  const int readers = (2 * P - 1) + vch + (P == 1 ? 1 : 2);
  const double abs_tol = 1e-15 * A.norm[0];
  double* buf[2] = {A.a, A.b};
  const long long ldb[2] = {A.lda, (long long)m};
  // each flag on its own 128-byte line: a writer's release and its pollers' acquires
  // do not queue behind the polling of unrelated flags at the same L2 line
  int* sflag = A.flags;
  int* aflag = sflag + kFS * P;
  int* vflag = aflag + kFS * P * P;
  int* jread = vflag + kFS * P * vch;                  // [2][P]
  const int tid = threadIdx.x;
  int sweeps_done = -1;
  for (int sweep = 0; sweep < A.max_sweeps; ++sweep) {
    for (int r = 0; r < rounds; ++r) {
      const int R = sweep * rounds + r;
      const double* cur = buf[R & 1];
      const long long ldc = ldb[R & 1];
      double* nxt = buf[(R + 1) & 1];
      const long long ldn = ldb[(R + 1) & 1];
      double* Jslot = A.jbuf + (size_t)(R & 1) * P * kJS * kJS;
      double* Sslot = A.sbuf + (size_t)(R & 1) * P * kJS * kJS;
      for (int task = blockIdx.x; task < ntask; task += gridDim.x) {
        if (task < P) {
          // ------------------------------------------------------- solve
          const int pair = task;
          const long long tw0 = clock64();
          // R ≥ 1: this pair's blocks a, b sat in pairs pa, pb of round R−1 (halves ha, hb).
          // Its subproblem is assembled here from round R−1's solves — A_R(a,a), A_R(b,b) from
          // S_pa, S_pb; A_R(a,b) = [J_paᵀ A_{R−1}(pa,pb) J_pb](a,b) and A_R(b,a) likewise, the
          // same DMMA products (bit for bit) round R−1's A-items write — so a round's solves
          // wait only on the previous round's solves, not on its A-items (one flag hop and the
          // A-item work off the critical path of every round).
          const int rp = (R + rounds - 1) % rounds;
          int pa = 0, pb = 0, ha = 0, hb = 0;
          if (R >= 1) {
            int ba, bb, x0, x1, y0, y1;
            circle_pair(nblk, r, pair, ba, bb);
            pa = pair_of(nblk, R - 1, ba);
            pb = pair_of(nblk, R - 1, bb);
            circle_pair(nblk, rp, pa, x0, x1);
            circle_pair(nblk, rp, pb, y0, y1);
            ha = ba == x0 ? 0 : 1;
            hb = bb == y0 ? 0 : 1;
            // every dependency polled by its own thread (a flag check is an L2 round trip;
            // eleven of them in one thread's sequence cost microseconds per round)
            if (tid == 0) jtrace(R, ntask, task, 0, gtimer());
            const int* fp = nullptr;
            int ft = 0;
            if (tid == 0 && R >= 2) {   // the J/S slot this solve overwrites: all its readers done
              fp = &jread[kFS * ((R & 1) * P + pair)];
              ft = (R / 2) * readers;
            } else if (tid >= 1 && tid <= 8 && R >= 2 && pa != pb) {
              // tiles (pa,pb), (pb,pa) of A_{R−1}: written by round R−2's A-items
              const int w = tid - 1, i = (w >> 2) & 1, j = (w >> 1) & 1;
              const int qx = pair_of(nblk, R - 2, i ? x1 : x0), qy = pair_of(nblk, R - 2, j ? y1 : y0);
              fp = &aflag[kFS * ((w & 1) ? qy * P + qx : qx * P + qy)];
              ft = R - 1;
            }
            if (fp) flag_wait(fp, ft, kPollBackoff);
          } else if (tid == 0) {
            jtrace(R, ntask, task, 0, gtimer());
          }
          if (tid < kJS) {
            ia[tid] = sub_index<JB>(nblk, r, pair, tid);
            if (R >= 1) {
              ib[tid] = sub_index<JB>(nblk, rp, pa, tid);
              ic[tid] = sub_index<JB>(nblk, rp, pb, tid);
            }
          }
          __syncthreads();
          constexpr int NS = kJS * kJS / kJT;
          const bool prod = R >= 1 && pa != pb;
          // the A_{R−1} tiles are final already: their loads fly while round R−1's solves finish
          double t1[NS], t2[NS];
          if (prod) {
            const double* prev = buf[(R - 1) & 1];
            const long long ldp = ldb[(R - 1) & 1];
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
              t1[u] = (ib[i] < m && ic[j] < m) ? __ldcg(prev + (long long)ib[i] * ldp + ic[j]) : 0.0;
              t2[u] = (ic[i] < m && ib[j] < m) ? __ldcg(prev + (long long)ic[i] * ldp + ib[j]) : 0.0;
            }
          }
          if (R >= 1) {
            if (tid == 0) flag_wait(&sflag[kFS * pa], R);
            if (tid == 32) flag_wait(&sflag[kFS * pb], R);
            __syncthreads();
          }
          if (tid == 0) jtrace(R, ntask, task, 1, gtimer());
          const long long tw1 = clock64();
          if (R == 0) {
            // all loads of this thread in flight at once (register staging)
            double vs[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, gi = ia[e / kJS], gj = ia[e % kJS];
              vs[u] = (gi < m && gj < m) ? __ldcg(cur + (long long)gi * ldc + gj) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
              S0[i * kJLd + j] = vs[u];
              V0[i * kJLd + j] = (i == j) ? 1.0 : 0.0;
            }
          } else {
            const size_t prev_slot = (size_t)((R - 1) & 1) * P * kJS * kJS;
            const double* Sa = A.sbuf + prev_slot + (size_t)pa * kJS * kJS;
            const double* Sb = A.sbuf + prev_slot + (size_t)pb * kJS * kJS;
            // diagonal blocks: (a,a) = S_pa[ha-half], (b,b) = S_pb[hb-half]; for pa == pb
            // (a single pair, P = 1) the off-diagonal blocks come from S_pa as well
            double dv[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
              const int hi = i < JB ? ha : hb, hj = j < JB ? ha : hb;
              const bool diag = (i < JB) == (j < JB);
              const double* Ss = (diag && i >= JB) ? Sb : Sa;
              dv[u] = (diag || pa == pb) ? __ldcg(Ss + (size_t)(hi * JB + i % JB) * kJS + hj * JB + j % JB) : 0.0;
            }
            if (prod) {
              {
                const double* Ja = A.jbuf + prev_slot + (size_t)pa * kJS * kJS;
                const double* Jb = A.jbuf + prev_slot + (size_t)pb * kJS * kJS;
                double va[NS], vb[NS];
#pragma unroll
                for (int u = 0; u < NS; ++u) {
                  va[u] = __ldcg(Ja + tid + u * kJT);
                  vb[u] = __ldcg(Jb + tid + u * kJT);
                }
#pragma unroll
                for (int u = 0; u < NS; ++u) {
                  const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
                  S0[i * kJLd + j] = t1[u];
                  V1[i * kJLd + j] = t2[u];
                  V0[i * kJLd + j] = va[u];
                  X[i * kJLd + j] = vb[u];
                }
              }
              __syncthreads();
              // both off-diagonal products side by side (two accumulator chains per warp)
              double c1[2][2], c2[2][2];
              mm_dmma2<JB>(V0, true, S0, c1, X, true, V1, c2);   // J_paᵀ T(pa,pb), J_pbᵀ T(pb,pa)
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  int row, col;
                  mm_coord<JB>(j, e, row, col);
                  S1[row * kJLd + col] = c1[j][e];
                  Y[row * kJLd + col] = c2[j][e];
                }
              __syncthreads();
              mm_dmma2<JB>(S1, false, X, c1, Y, false, V0, c2);  // (·) J_pb, (·) J_pa
              __syncthreads();
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  int row, col;
                  mm_coord<JB>(j, e, row, col);
                  if (row / JB == ha && col / JB == hb) S0[(row % JB) * kJLd + JB + col % JB] = c1[j][e];
                  if (row / JB == hb && col / JB == ha) S0[(JB + row % JB) * kJLd + col % JB] = c2[j][e];
                }
            }
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
              if ((i < JB) == (j < JB) || pa == pb) S0[i * kJLd + j] = dv[u];
              V0[i * kJLd + j] = (i == j) ? 1.0 : 0.0;
            }
            __syncthreads();
            if (tid == 0) {   // J/S of round R−1 read: count this solve among the slot's readers
              atomicAdd(&jread[kFS * (((R - 1) & 1) * P + pa)], 1);
              if (pb != pa) atomicAdd(&jread[kFS * (((R - 1) & 1) * P + pb)], 1);
            }
          }
          __syncthreads();
          const long long tw2 = clock64();
          int rots = 0;
          const bool full = (r == 0) || (P == 1);
          const int inner_sweeps = (P == 1) ? 40 : A.inner;
          double *Sc = S0, *Vc = V0, *Sn = S1, *Vn = V1;
          for (int isw = 0; isw < inner_sweeps; ++isw) {
            int srot = 0;
            const int nsteps = full ? kJS - 1 : JB;
            for (int ir = 0; ir < nsteps; ++ir) {
              const int nr = jacobi_step<JB>(Sc, Vc, Sn, Vn, full, ir, abs_tol);
              if (nr) {
                double* tp = Sc;
                Sc = Sn;
                Sn = tp;
                tp = Vc;
                Vc = Vn;
                Vn = tp;
              }
              srot += nr;
            }
            rots += srot;
            if (srot == 0) break;
          }
          double* J = Jslot + (size_t)pair * kJS * kJS;
          double* So = Sslot + (size_t)pair * kJS * kJS;
          for (int e = tid; e < kJS * kJS; e += kJT) {
            J[e] = Vc[(e / kJS) * kJLd + e % kJS];
            So[e] = Sc[(e / kJS) * kJLd + e % kJS];
          }
          __syncthreads();
          if (tid == 0) {
            if (rots > 0) atomicAdd(&A.counters[sweep], rots);
            flag_set(&sflag[kFS * (pair)], R + 1);
            jtrace(R, ntask, task, 2, gtimer());
            if (A.timers && pair == 0) {
              A.timers[0] += tw1 - tw0;
              A.timers[1] += tw2 - tw1;
              A.timers[2] += clock64() - tw2;
            }
          }
        } else if (task < P + P * P) {
          // ------------------------------------------------------- A-item
          const int it = task - P;
          const int pa = it / P, pb = it % P;
          const long long tw0 = clock64();
          if (tid < kJS) {
            ia[tid] = sub_index<JB>(nblk, r, pa, tid);
            ib[tid] = sub_index<JB>(nblk, r, pb, tid);
          }
          {
            // one thread per dependency: every solve of round R (not only pa and pb — they
            // read A_{R−1} from the buffer this item overwrites, nxt; see the solve), and the
            // four round-(R−1) A-items holding this tile's blocks
            if (tid == 0) jtrace(R, ntask, task, 0, gtimer());
            const int* fp = nullptr;
            int ft = 0;
            if (tid < P) {
              fp = &sflag[kFS * tid];
              ft = R + 1;
            } else if (tid < P + 4 && R >= 1) {
              const int w = tid - P;
              int a0, a1, b0, b1;
              circle_pair(nblk, r, pa, a0, a1);
              circle_pair(nblk, r, pb, b0, b1);
              const int qa = pair_of(nblk, R - 1, (w >> 1) ? a1 : a0), qb = pair_of(nblk, R - 1, (w & 1) ? b1 : b0);
              fp = &aflag[kFS * (qa * P + qb)];
              ft = R;
            }
            if (fp) flag_wait(fp, ft, kPollBackoff);
          }
          __syncthreads();
          if (tid == 0) jtrace(R, ntask, task, 1, gtimer());
          const long long tw1 = clock64();
          double c[2][2];
          const bool last = (r == rounds - 1);
          double lmax = 0.0;
          if (pa == pb) {
            const double* Sp = Sslot + (size_t)pa * kJS * kJS;
            constexpr int NS = kJS * kJS / kJT;
            double vs[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) vs[u] = __ldcg(Sp + tid + u * kJT);
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, gi = ia[e / kJS], gj = ib[e % kJS];
              if (gi < m && gj < m) {
                nxt[(long long)gi * ldn + gj] = vs[u];
                if (gi != gj) lmax = fmax(lmax, fabs(vs[u]));
              }
            }
          } else {
            const double* Ja = Jslot + (size_t)pa * kJS * kJS;
            const double* Jb = Jslot + (size_t)pb * kJS * kJS;
            {
              constexpr int NS = kJS * kJS / kJT;
              double vs[NS], va[NS], vb[NS];
#pragma unroll
              for (int u = 0; u < NS; ++u) {
                const int e = tid + u * kJT, gi = ia[e / kJS], gj = ib[e % kJS];
                vs[u] = (gi < m && gj < m) ? __ldcg(cur + (long long)gi * ldc + gj) : 0.0;
                va[u] = __ldcg(Ja + e);
                vb[u] = __ldcg(Jb + e);
              }
#pragma unroll
              for (int u = 0; u < NS; ++u) {
                const int e = tid + u * kJT, i = e / kJS, j = e % kJS;
                S0[i * kJLd + j] = vs[u];
                V0[i * kJLd + j] = va[u];
                X[i * kJLd + j] = vb[u];
              }
            }
            __syncthreads();
            mm_dmma<JB>(V0, true, S0, c);  // J_aᵀ T
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                int row, col;
                mm_coord<JB>(j, e, row, col);
                S1[row * kJLd + col] = c[j][e];
              }
            __syncthreads();
            mm_dmma<JB>(S1, false, X, c);  // (J_aᵀ T) J_b
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                int row, col;
                mm_coord<JB>(j, e, row, col);
                const int gi = ia[row], gj = ib[col];
                if (gi < m && gj < m) {
                  nxt[(long long)gi * ldn + gj] = c[j][e];
                  lmax = fmax(lmax, fabs(c[j][e]));   // pa ≠ pb: all entries off-diagonal
                }
              }
          }
          if (last) {
            lmax = warp_max(lmax);
            if ((tid & 31) == 0) red8[tid >> 5] = lmax;
          }
          __syncthreads();
          if (tid == 0) {
            if (last) {
              double bm = 0.0;
              for (int w = 0; w < kJT / 32; ++w) bm = fmax(bm, red8[w]);
              if (bm > 0.0) atomicMax(&A.maxoff[sweep], (unsigned long long)__double_as_longlong(bm));
            }
            atomicAdd(&jread[kFS * ((R & 1) * P + pa)], 1);
            if (pb != pa) atomicAdd(&jread[kFS * ((R & 1) * P + pb)], 1);
            flag_set(&aflag[kFS * (pa * P + pb)], R + 1);
            jtrace(R, ntask, task, 2, gtimer());
            if (A.timers && it == 1) {
              A.timers[3] += tw1 - tw0;
              A.timers[4] += clock64() - tw1;
            }
          }
        } else {
          // ------------------------------------------------------- V-item
          const int vb = task - P - P * P;
          const int pb = vb % P, vc = vb / P;
          if (tid < kJS) ib[tid] = sub_index<JB>(nblk, r, pb, tid);
          if (tid == 0) {
            jtrace(R, ntask, task, 0, gtimer());
            flag_wait(&sflag[kFS * pb], R + 1, kPollBackoff);
          } else if (tid >= 32 && tid < 34 && R >= 1) {   // other warp: polled concurrently
            int b0, b1;
            circle_pair(nblk, r, pb, b0, b1);
            flag_wait(&vflag[kFS * (vc * P + pair_of(nblk, R - 1, tid == 32 ? b0 : b1))], R, kPollBackoff);
          }
          __syncthreads();
          if (tid == 0) jtrace(R, ntask, task, 1, gtimer());
          const double* Jb = Jslot + (size_t)pb * kJS * kJS;
          constexpr int NS = kJS * kJS / kJT;
          {
            double vb[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) vb[u] = __ldcg(Jb + tid + u * kJT);
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT;
              X[(e / kJS) * kJLd + e % kJS] = vb[u];
            }
          }
          for (int h = 0; h < 2; ++h) {
            const int r0 = vc * 2 * kJS + h * kJS;
            if (r0 >= m) break;
            double c[2][2];
            double vs[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT, gr = r0 + e / kJS, gj = ib[e % kJS];
              vs[u] = (gr < m && gj < m) ? __ldcg(A.v + (long long)gr * A.ldv + gj) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NS; ++u) {
              const int e = tid + u * kJT;
              S0[(e / kJS) * kJLd + e % kJS] = vs[u];
            }
            __syncthreads();
            mm_dmma<JB>(S0, false, X, c);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                int row, col;
                mm_coord<JB>(j, e, row, col);
                const int gr = r0 + row, gj = ib[col];
                if (gr < m && gj < m) A.v[(long long)gr * A.ldv + gj] = c[j][e];
              }
            __syncthreads();
          }
          if (tid == 0) {
            atomicAdd(&jread[kFS * ((R & 1) * P + pb)], 1);
            flag_set(&vflag[kFS * (vc * P + pb)], R + 1);
            jtrace(R, ntask, task, 2, gtimer());
          }
        }
        __syncthreads();
      }
    }
    // convergence: every solve of this sweep is done once its last round's flags are up
    const int Rlast = sweep * rounds + rounds - 1;
    // (flags polled one per thread, concurrently)
    for (int p = tid; p < P; p += kJT) flag_wait(&sflag[kFS * p], Rlast + 1);
    __syncthreads();
    const int rots = *((volatile int*)&A.counters[sweep]);
    if (rots != 0) {
      // every off-diagonal entry already at or below the rotation threshold: the next sweep
      // would rotate nothing — stop now instead of running it (the last A-items finish a
      // flag hop after the last solves; a wasted sweep costs a whole sweep of rounds)
      for (int q = tid; q < P * P; q += kJT) flag_wait(&aflag[kFS * q], Rlast + 1);
      __syncthreads();
    }
    if (tid == 0) {
      int stop = rots == 0;
      if (!stop) {
        const double mo = __longlong_as_double((long long)*((volatile unsigned long long*)&A.maxoff[sweep]));
        stop = mo <= abs_tol;
      }
      stop_flag = stop;
    }
    __syncthreads();
    if (stop_flag) {
      sweeps_done = sweep + 1;
      break;
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    A.out[0] = sweeps_done;
    A.out[1] = sweeps_done > 0 ? ((sweeps_done * rounds) & 1) : 0;
  }
}

__global__ void jacobi_norm_kernel(const double* a, long long lda, int m, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = warp; i < m; i += nw)   // warp per row: coalesced, no index division
    for (int j = lane; j < m; j += 32) {
      const double x = a[(long long)i * lda + j];
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

__global__ void jacobi_diag_kernel(const double* a, long long lda, const double* b, int m,
                                   const int* out, double* vals, int* dsweeps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) *dsweeps = out[0];
  if (i >= m) return;
  vals[i] = out[1] ? b[(long long)i * m + i] : a[(long long)i * lda + i];
}

constexpr int kJacobiMaxSweeps = 40;

// 64×64 subproblems (JB = 32, PSD_JACOBI_JB=32) halve the rounds per sweep but not the
// sweeps (13 at m = 272 either way), and each round's 1024-thread solve steps cost 4× the
// 256-thread ones: measured on the B200 6.77 vs 3.90 ms at m = 272, 13.4 vs 11.1 ms at
// m = 544 — so JB = 16 is the default at every size.
constexpr int kJacobiWideMin = 1 << 30;

static void jacobi_geometry(int m, int jb, int& nblk, int& P) {
  const int nb0 = (m + jb - 1) / jb;
  nblk = std::max(2, nb0 + (nb0 & 1));
  P = nblk / 2;
}

static int jacobi_nflags(int m, int jb, int P) {
  const int vch = (m + 4 * jb - 1) / (4 * jb);
  return kFS * (P + P * P + P * vch + 2 * P);
}

static size_t jacobi_ws_elems_jb(int m, int jb) {
  int nblk, P;
  jacobi_geometry(m, jb, nblk, P);
  const size_t js = 2 * (size_t)jb;
  return (size_t)m * m + (size_t)4 * P * js * js + 8 + kJacobiMaxSweeps + 8 +
         (size_t)(jacobi_nflags(m, jb, P) + 1) / 2 + 8 + kJacobiMaxSweeps + 1;
}

size_t jacobi_ws_elems(int m) {
  return std::max(jacobi_ws_elems_jb(m, 16), jacobi_ws_elems_jb(m, 32));
}

template <int JB>
static int jacobi_run(double* a, long long lda, int m, double* values, double* v, long long ldv,
                      double* ws, int* dsweeps, cudaStream_t st) {
  using T = JTraits<JB>;
  constexpr int kJS = T::kJS, kJT = T::kJT;
  int nblk, P;
  jacobi_geometry(m, JB, nblk, P);
  JacobiArgs A{};
  A.a = a;
  A.lda = lda;
  A.b = ws;
  A.v = v;
  A.ldv = ldv;
  A.jbuf = ws + (size_t)m * m;                    // [2 slots][P] rotation products
  A.sbuf = A.jbuf + (size_t)2 * P * kJS * kJS;     // [2 slots][P] rotated subproblems
  A.norm = A.sbuf + (size_t)2 * P * kJS * kJS;
  int* ints = reinterpret_cast<int*>(A.norm + 8);
  A.counters = ints;
  A.out = ints + kJacobiMaxSweeps + 2;
  A.flags = ints + kJacobiMaxSweeps + 8;
  const int nflags = jacobi_nflags(m, JB, P);
  {
    const size_t int_words = (size_t)kJacobiMaxSweeps + 8 + nflags;
    A.maxoff = reinterpret_cast<unsigned long long*>(A.norm + 8 + (int_words + 1) / 2 + 1);
    cudaMemsetAsync(A.maxoff, 0, kJacobiMaxSweeps * sizeof(unsigned long long), st);
  }
  A.m = m;
  A.nblk = nblk;
  A.max_sweeps = kJacobiMaxSweeps;
  {
    const char* e = getenv("PSD_JACOBI_INNER");
    A.inner = e ? std::max(1, atoi(e)) : 1;
  }
  A.timers = nullptr;
  static long long* dtimers = nullptr;
  if (getenv("PSD_JACOBI_TIMERS")) {
    if (!dtimers) cudaMalloc(&dtimers, 6 * sizeof(long long));
    cudaMemsetAsync(dtimers, 0, 6 * sizeof(long long), st);
    A.timers = dtimers;
  }
  cudaMemsetAsync(ints, 0, (kJacobiMaxSweeps + 8 + nflags) * sizeof(int), st);
  static const char* trace_path = getenv("PSD_JACOBI_TRACE");
  static long long* dtrace = nullptr;
  const int vch0 = (m + 2 * kJS - 1) / (2 * kJS);
  const size_t trace_elems = (size_t)1024 * (P + P * P + P * vch0) * 3;
  if (trace_path) {
    if (!dtrace) cudaMalloc(&dtrace, trace_elems * sizeof(long long) * 4);
    cudaMemsetAsync(dtrace, 0, trace_elems * sizeof(long long), st);
    cudaMemcpyToSymbolAsync(g_jtrace, &dtrace, sizeof(dtrace), 0, cudaMemcpyHostToDevice, st);
  }
  set_identity(v, ldv, m, st);
  jacobi_norm_kernel<<<1, 1024, 0, st>>>(a, lda, m, A.norm);
  count_launch();

  static int max_blocks[16] = {};
  static bool attr_set[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(jacobi_persistent_kernel<JB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)T::kSmemBytes);
    attr_set[dev] = true;
  }
  if (!max_blocks[dev]) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_persistent_kernel<JB>, kJT, T::kSmemBytes);
    max_blocks[dev] = std::max(1, per_sm) * device_info().sms;
  }
  const int vch = (m + 2 * kJS - 1) / (2 * kJS);
  const int tasks = P + P * P + P * vch;
  const int grid = std::max(1, std::min({tasks, max_blocks[dev], device_info().sms}));
  void* args[] = {&A};
  if (cudaLaunchCooperativeKernel((const void*)jacobi_persistent_kernel<JB>, dim3(grid), dim3(kJT),
                                  args, T::kSmemBytes, st) != cudaSuccess)
    return -3;
  count_launch();
  // the diagonal comes from whichever buffer holds the result (decided on the device);
  // `a` is documented as destroyed, so no copy-back — no host round trip here
  jacobi_diag_kernel<<<(m + 255) / 256, 256, 0, st>>>(a, lda, ws, m, A.out, values, dsweeps);
  count_launch();
  static const bool stats = getenv("PSD_JACOBI_STATS") != nullptr;
  int out[2] = {0, 0};
  if (stats || trace_path || A.timers) read_small(out, A.out, 2 * sizeof(int), st);   // diagnostics only
  if (stats) {   // per sweep: rotations above threshold, max |off-diagonal| after the sweep
    std::vector<int> cnt(kJacobiMaxSweeps);
    std::vector<unsigned long long> mo(kJacobiMaxSweeps);
    double nrm = 0.0;
    cudaMemcpy(cnt.data(), A.counters, cnt.size() * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(mo.data(), A.maxoff, mo.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(&nrm, A.norm, sizeof(double), cudaMemcpyDeviceToHost);
    fprintf(stderr, "jacobi m=%d sweeps=%d |A|=%.3e:", m, out[0], nrm);
    for (int sw = 0; sw < std::max(out[0], 0); ++sw) {
      double d;
      std::memcpy(&d, &mo[sw], sizeof(d));
      fprintf(stderr, " [%d %.1e]", cnt[sw], d / nrm);
    }
    fprintf(stderr, "\n");
  }
  if (trace_path) {   // binary dump: header (m, P, vch, rounds, ntask) then int64 [R][task][3]
    std::vector<long long> h(trace_elems);
    cudaMemcpy(h.data(), dtrace, trace_elems * sizeof(long long), cudaMemcpyDeviceToHost);
    long long* none = nullptr;
    cudaMemcpyToSymbol(g_jtrace, &none, sizeof(none));
    if (FILE* f = fopen(trace_path, "wb")) {
      const long long hdr[5] = {m, P, vch0, (long long)(nblk - 1) * std::max(out[0], 0), P + P * P + P * vch0};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(h.data(), sizeof(long long), h.size(), f);
      fclose(f);
    }
  }
  if (A.timers) {
    long long h[6];
    cudaMemcpy(h, A.timers, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr,
            "jacobi m=%d JB=%d sweeps=%d grid=%d cycles: solve0 wait %lld load %lld compute %lld | item(0,1) wait %lld work %lld\n",
            m, JB, out[0], grid, h[0], h[1], h[2], h[3], h[4]);
  }
  return 0;
}

__global__ void set_int_kernel(int* p, int v) { *p = v; }

int jacobi_eigh(double* a, long long lda, int m, double* values, double* v, long long ldv,
                double* ws, size_t ws_elems, int* dsweeps, cudaStream_t st) {
  if (m == 1) {
    cudaMemcpyAsync(values, a, sizeof(double), cudaMemcpyDeviceToDevice, st);
    set_identity(v, ldv, 1, st);
    set_int_kernel<<<1, 1, 0, st>>>(dsweeps, 1);
    count_launch();
    return 0;
  }
  if (ws_elems < jacobi_ws_elems(m)) return -2;
  static const int jb_env = [] { const char* e = getenv("PSD_JACOBI_JB"); return e ? atoi(e) : 0; }();
  const int jb = jb_env == 16 || jb_env == 32 ? jb_env : (m >= kJacobiWideMin ? 32 : 16);
  return jb == 32 ? jacobi_run<32>(a, lda, m, values, v, ldv, ws, dsweeps, st)
                  : jacobi_run<16>(a, lda, m, values, v, ldv, ws, dsweeps, st);
}

}  // namespace psd
