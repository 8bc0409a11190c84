// Shared device helpers for the B200 (sm_100a) randomized PSD-projection kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PSD_DEVINL __device__ __forceinline__

namespace psd {

constexpr int kWarp = 32;

PSD_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

PSD_DEVINL double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Non-negative doubles order like their bit patterns, so a u64 atomicMax is a
// deterministic max for them.
PSD_DEVINL void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ---- cp.async (LDGSTS) with zero-fill -------------------------------------
PSD_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PSD_DEVINL void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}

PSD_DEVINL void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}

PSD_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
PSD_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- FP64 tensor core: mma.sync m8n8k4 → SASS DMMA.8x8x4 -------------------
// A fragment: A[g][t]; B fragment: B[k=t][n=g]; C: C[g][2t], C[g][2t+1]
// with g = lane>>2, t = lane&3.
PSD_DEVINL void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

}  // namespace psd
