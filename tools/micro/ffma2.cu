// FFMA vs FFMA2 (fma.rn.f32x2) vs IMAD issue throughput on sm_100a: 8 independent chains per
// thread, 148×8 blocks of 256 threads; prints Gop/s and ops/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
__global__ void k_ffma(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av), B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 t = make_float2(threadIdx.x + i, i); x[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
  float s = 0; for (int i = 0; i < 8; ++i) { float2 t = *reinterpret_cast<float2*>(&x[i]); s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imad(float* out, uint32_t a, uint32_t b) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void k_mix(float* out, float a, float b, uint32_t c, uint32_t d) {   // 1 FFMA2 : 1 IMAD
  unsigned long long x[4]; uint32_t y[4];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long*>(&av), B = *reinterpret_cast<unsigned long long*>(&bv);
#pragma unroll
  for (int i = 0; i < 4; ++i) { float2 t = make_float2(threadIdx.x + i, i); x[i] = *reinterpret_cast<unsigned long long*>(&t); y[i] = threadIdx.x * i; }
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[i]) : "r"(c), "r"(d));
    }
  float s = 0; for (int i = 0; i < 4; ++i) { float2 t = *reinterpret_cast<float2*>(&x[i]); s += t.x + t.y + y[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms = 0, clk = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 8 * 256 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double insts = (double)sms * 8 * 256 * ITERS * 8;   // per-thread instruction count × threads
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma<<<sms * 8, 256>>>(out, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("FFMA : %.1f G thread-instr/s\n", insts / ms / 1e6);
    cudaEventRecord(e0); k_ffma2<<<sms * 8, 256>>>(out, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("FFMA2: %.1f G thread-instr/s (x2 flops)\n", insts / ms / 1e6);
    cudaEventRecord(e0); k_imad<<<sms * 8, 256>>>(out, 3u, 7u); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("IMAD : %.1f G thread-instr/s\n", insts / ms / 1e6);
    cudaEventRecord(e0); k_mix<<<sms * 8, 256>>>(out, 1.0001f, 0.5f, 3u, 7u); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("FFMA2+IMAD mix: %.1f G thread-instr/s\n", insts / ms / 1e6);
  }
  printf("SMs %d, max clock %d kHz; 1 warp-instr/clk/SMSP = %.1f G thread-instr/s at max clock\n", sms, clk,
         sms * 4.0 * 32 * clk / 1e6);
  return 0;
}
