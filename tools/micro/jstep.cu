// Latency anatomy of one parallel Jacobi step (jacobi.cu, JB = 16: a 32×32 subproblem in
// shared memory, 256 threads) on one SM: cycles per step for the real step and for variants
// with the rotation or the barrier removed, plus dependent-chain latencies of DFMA, DMUL,
// rsqrt(double) and SHFL.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 jstep.cu -o jstep
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int JB = 16, JS = 32, L = JS + 4, NT = JB * JB;

__device__ __forceinline__ void step_pair(int ir, int k, int& p, int& q) {
  p = k;
  q = JB + ((k + ir) & (JB - 1));
}

__device__ __forceinline__ bool rotation(double app, double aqq, double apq, double tol, double& c, double& s,
                                         double& t) {
  const double d = aqq - app, e = 2.0 * apq;
  const double y = rsqrt(fmax(fma(d, d, e * e), 2.2250738585072014e-308));
  const double h = fma(0.5 * fabs(d), y, 0.5);
  const double z = rsqrt(h);
  const bool rot = fabs(apq) > tol && apq * apq > 1e-30 * fabs(app * aqq);
  const double sr = (d >= 0.0 ? 0.5 : -0.5) * e * y * z;
  c = rot ? h * z : 1.0;
  s = rot ? sr : 0.0;
  t = rot ? sr * z : 0.0;
  return rot;
}

// MODE 0: real step; 1: rotation from a fixed table (no rsqrt chain); 2: no barrier;
// 3: real step, rotations computed by one warp and broadcast through smem (extra barrier)
template <int MODE>
__device__ int step(const double* Sc, const double* Vc, double* Sn, double* Vn, int ir, double tol, double* rot_s) {
  const int lane = threadIdx.x & 31, l = lane & (JB - 1), k = threadIdx.x / JB;
  int p, q, pk, qk;
  step_pair(ir, l, p, q);
  step_pair(ir, k, pk, qk);
  const double lpp = Sc[p * L + p], lqq = Sc[q * L + q], lpq = Sc[p * L + q];
  double b00 = Sc[pk * L + p], b01 = Sc[pk * L + q], b10 = Sc[qk * L + p], b11 = Sc[qk * L + q];
  const double v00 = Vc[k * L + p], v01 = Vc[k * L + q], v10 = Vc[(k + JB) * L + p], v11 = Vc[(k + JB) * L + q];
  double c, s, t, ck, sk;
  bool r;
  if (MODE == 1) {
    c = 0.8 + 1e-3 * lpp;
    s = 0.6 + 1e-3 * lqq;
    t = lpq;
    r = true;
  } else if (MODE == 3) {
    if (threadIdx.x < JB) {
      double cc, ss, tt;
      rotation(lpp, lqq, lpq, tol, cc, ss, tt);
      rot_s[threadIdx.x] = cc;
      rot_s[JB + threadIdx.x] = ss;
      rot_s[2 * JB + threadIdx.x] = tt;
    }
    __syncthreads();
    c = rot_s[l];
    s = rot_s[JB + l];
    t = rot_s[2 * JB + l];
    r = s != 0.0;
  } else {
    r = rotation(lpp, lqq, lpq, tol, c, s, t);
  }
  const int nrot = __popc(__ballot_sync(0xffffffffu, r) & 0xffffu);
  if (nrot == 0) return 0;
  if (MODE == 3) {
    ck = rot_s[k];
    sk = rot_s[JB + k];
  } else {
    ck = __shfl_sync(0xffffffffu, c, k & (JB - 1));
    sk = __shfl_sync(0xffffffffu, s, k & (JB - 1));
  }
  const double kpp = b00, kqq = b11, kpq = b01;
  const double r00 = c * b00 - s * b01, r01 = s * b00 + c * b01;
  const double r10 = c * b10 - s * b11, r11 = s * b10 + c * b11;
  b00 = ck * r00 - sk * r10;
  b01 = ck * r01 - sk * r11;
  b10 = sk * r00 + ck * r10;
  b11 = sk * r01 + ck * r11;
  if (k == l && sk != 0.0) {
    b00 = kpp - t * kpq;
    b11 = kqq + t * kpq;
    b01 = 0.0;
    b10 = 0.0;
  }
  Sn[pk * L + p] = b00;
  Sn[pk * L + q] = b01;
  Sn[qk * L + p] = b10;
  Sn[qk * L + q] = b11;
  Vn[k * L + p] = c * v00 - s * v01;
  Vn[k * L + q] = s * v00 + c * v01;
  Vn[(k + JB) * L + p] = c * v10 - s * v11;
  Vn[(k + JB) * L + q] = s * v10 + c * v11;
  if (MODE == 2) __syncwarp(); else __syncthreads();
  return nrot;
}

template <int MODE>
__global__ void __launch_bounds__(NT) k_steps(const double* a, int nsteps, long long* cyc, double* out) {
  __shared__ double S0[JS * L], V0[JS * L], S1[JS * L], V1[JS * L], rs[3 * JB];
  for (int e = threadIdx.x; e < JS * JS; e += NT) {
    const int i = e / JS, j = e % JS;
    S0[i * L + j] = a[e];
    V0[i * L + j] = i == j;
  }
  __syncthreads();
  double *Sc = S0, *Vc = V0, *Sn = S1, *Vn = V1;
  const long long t0 = clock64();
  for (int it = 0; it < nsteps; ++it) {
    if (step<MODE>(Sc, Vc, Sn, Vn, it & 15, 1e-300, rs)) {
      double* x = Sc; Sc = Sn; Sn = x;
      x = Vc; Vc = Vn; Vn = x;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = Sc[threadIdx.x] + Vc[threadIdx.x];
}


// FP32 variant of the real step (same structure; rsqrtf, float smem, one SHFL per value)
__device__ __forceinline__ bool rotation_f(float app, float aqq, float apq, float& c, float& s, float& t) {
  const float d = aqq - app, e = 2.0f * apq;
  const float y = rsqrtf(fmaxf(fmaf(d, d, e * e), 1e-37f));
  const float h = fmaf(0.5f * fabsf(d), y, 0.5f);
  const float z = rsqrtf(h);
  const bool rot = fabsf(apq) > 1e-37f;
  const float sr = (d >= 0.f ? 0.5f : -0.5f) * e * y * z;
  c = rot ? h * z : 1.f;
  s = rot ? sr : 0.f;
  t = rot ? sr * z : 0.f;
  return rot;
}
__device__ int step_f(const float* Sc, const float* Vc, float* Sn, float* Vn, int ir) {
  const int lane = threadIdx.x & 31, l = lane & (JB - 1), k = threadIdx.x / JB;
  int p, q, pk, qk;
  step_pair(ir, l, p, q);
  step_pair(ir, k, pk, qk);
  const float lpp = Sc[p * L + p], lqq = Sc[q * L + q], lpq = Sc[p * L + q];
  float b00 = Sc[pk * L + p], b01 = Sc[pk * L + q], b10 = Sc[qk * L + p], b11 = Sc[qk * L + q];
  const float v00 = Vc[k * L + p], v01 = Vc[k * L + q], v10 = Vc[(k + JB) * L + p], v11 = Vc[(k + JB) * L + q];
  float c, s, t;
  const bool r = rotation_f(lpp, lqq, lpq, c, s, t);
  const int nrot = __popc(__ballot_sync(0xffffffffu, r) & 0xffffu);
  if (nrot == 0) return 0;
  const float ck = __shfl_sync(0xffffffffu, c, k & (JB - 1));
  const float sk = __shfl_sync(0xffffffffu, s, k & (JB - 1));
  const float kpp = b00, kqq = b11, kpq = b01;
  const float r00 = c * b00 - s * b01, r01 = s * b00 + c * b01;
  const float r10 = c * b10 - s * b11, r11 = s * b10 + c * b11;
  b00 = ck * r00 - sk * r10;
  b01 = ck * r01 - sk * r11;
  b10 = sk * r00 + ck * r10;
  b11 = sk * r01 + ck * r11;
  if (k == l && sk != 0.f) {
    b00 = kpp - t * kpq;
    b11 = kqq + t * kpq;
    b01 = 0.f;
    b10 = 0.f;
  }
  Sn[pk * L + p] = b00;
  Sn[pk * L + q] = b01;
  Sn[qk * L + p] = b10;
  Sn[qk * L + q] = b11;
  Vn[k * L + p] = c * v00 - s * v01;
  Vn[k * L + q] = s * v00 + c * v01;
  Vn[(k + JB) * L + p] = c * v10 - s * v11;
  Vn[(k + JB) * L + q] = s * v10 + c * v11;
  __syncthreads();
  return nrot;
}
__global__ void __launch_bounds__(NT) k_steps_f(const double* a, long long* cyc, double* out) {
  __shared__ float S0[JS * L], V0[JS * L], S1[JS * L], V1[JS * L];
  for (int e = threadIdx.x; e < JS * JS; e += NT) {
    const int i = e / JS, j = e % JS;
    S0[i * L + j] = (float)a[e];
    V0[i * L + j] = i == j;
  }
  __syncthreads();
  float *Sc = S0, *Vc = V0, *Sn = S1, *Vn = V1;
  const long long t0 = clock64();
  for (int it = 0; it < 16; ++it) {
    if (step_f(Sc, Vc, Sn, Vn, it & 15)) {
      float* x = Sc; Sc = Sn; Sn = x;
      x = Vc; Vc = Vn; Vn = x;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = Sc[threadIdx.x] + Vc[threadIdx.x];
}

// dependent-chain latencies (cycles per op)
__global__ void k_lat(double x, long long* cyc, double* out) {
  double v = x, w = x;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) v = fma(v, 0.999, 1e-3);
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) w = w * 1.0000001;
  long long t2 = clock64();
  double z = x + 2.0;
  for (int i = 0; i < 256; ++i) z = rsqrt(z) + 1.5;
  long long t3 = clock64();
  double u = x;
  for (int i = 0; i < 256; ++i) u = __shfl_sync(0xffffffffu, u, (threadIdx.x + 1) & 31) + 1.0;
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / 256;
    cyc[1] = (t2 - t1) / 256;
    cyc[2] = (t3 - t2) / 256;
    cyc[3] = (t4 - t3) / 256;
  }
  out[threadIdx.x] = v + w + z + u;
}

int main() {
  double* a;
  long long* cyc;
  double* out;
  cudaMalloc(&a, JS * JS * sizeof(double));
  cudaMalloc(&cyc, 64 * sizeof(long long));
  cudaMalloc(&out, 1024 * sizeof(double));
  double h[JS * JS];
  srand(1);
  for (int i = 0; i < JS; ++i)
    for (int j = 0; j <= i; ++j) h[i * JS + j] = h[j * JS + i] = (rand() / (double)RAND_MAX - 0.5) + (i == j) * i;
  cudaMemcpy(a, h, sizeof(h), cudaMemcpyHostToDevice);
  long long hc[4];
  k_lat<<<1, 32>>>(1.0, cyc, out);
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  printf("dependent latency (cycles): DFMA %lld  DMUL %lld  rsqrt(double)+DADD %lld  SHFL+DADD %lld\n", hc[0], hc[1],
         hc[2], hc[3]);
  const int nsteps = 1600;   // converging matrix: later steps may skip (nrot == 0) -> refresh input each run
  const char* names[] = {"real step", "rotation from table (no rsqrt chain)", "no barrier (__syncwarp)",
                         "rotations by 16 threads + smem broadcast (2 barriers)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k_steps<0><<<1, NT>>>(a, 16, cyc, out);
      if (mode == 1) k_steps<1><<<1, NT>>>(a, 16, cyc, out);
      if (mode == 2) k_steps<2><<<1, NT>>>(a, 16, cyc, out);
      if (mode == 3) k_steps<3><<<1, NT>>>(a, 16, cyc, out);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%-55s %6.0f cycles/step (16 steps, first sweep: every pair rotates)\n", names[mode], hc[0] / 16.0);
  }
  for (int rep = 0; rep < 2; ++rep) k_steps_f<<<1, NT>>>(a, cyc, out);
  cudaDeviceSynchronize();
  cudaMemcpy(hc, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
  printf("%-55s %6.0f cycles/step\n", "FP32 real step", hc[0] / 16.0);
  (void)nsteps;
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
