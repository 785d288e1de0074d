// Tensor-pipe rate of the MMA shapes the attention kernel issues, one CTA per SM:
//   SS  : D[128x128] += A[128x16] (smem, K-major) * B[128x16]^T (smem, K-major)   (Q.K^T step)
//   TS  : D[128x128] += A[128x16] (TMEM)           * B (smem, MN-major V)          (P.V step)
//   SS256: M=128, N=256 (the GEMM's per-SM shape)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2605_02953_b200/csrc tools/mma_rate.cu -o /tmp/mma_rate -lcuda
// Prints SM clocks per MMA instruction and the implied dense FLOP/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tf_ptx.cuh"

using namespace tf;

__device__ __forceinline__ uint64_t desc_mn(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128) rate_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t id128 = umma_idesc_bf16(128, 128);
    constexpr uint32_t id256 = umma_idesc_bf16(128, 256);
    constexpr uint32_t idpv = umma_idesc_bf16(128, 128) | (1u << 16);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0)
          umma_bf16(tmem, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), id128, 1);
        else if (MODE == 1)
          mma_ts(tmem + 256, tmem + kk * 8, desc_mn(b + kk * 2048, 16384), idpv, 1);
        else
          umma_bf16(tmem, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), id256, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait_spin(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  const int iters = 4096;
  const char* names[3] = {"SS M128 N128 K16", "TS M128 N128 K16 (A in TMEM, B MN-major)", "SS M128 N256 K16"};
  const double flop[3] = {2.0 * 128 * 128 * 16, 2.0 * 128 * 128 * 16, 2.0 * 128 * 256 * 16};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      long long cyc = 0;
      const size_t sm = 65536 + 1024;
      if (mode == 0) { cudaFuncSetAttribute(rate_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); rate_kernel<0><<<148, 128, sm>>>(iters, d); }
      if (mode == 1) { cudaFuncSetAttribute(rate_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); rate_kernel<1><<<148, 128, sm>>>(iters, d); }
      if (mode == 2) { cudaFuncSetAttribute(rate_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); rate_kernel<2><<<148, 128, sm>>>(iters, d); }
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      const double per = static_cast<double>(cyc) / (iters * 8.0);
      printf("%-44s %s: %.1f clk/MMA -> %.0f FLOP/clk/SM\n", names[mode], cudaGetErrorString(e), per, flop[mode] / per);
    }
  }
  return 0;
}
