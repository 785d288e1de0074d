// Tensor-pipe rate of cta_group::2 MMA shapes (the pair attention kernel's and the
// pair GEMM's), one 2-CTA cluster per SM pair, the leader issues:
//   0 SS  M=256 N=128 : D += A(smem) B(smem, K-major)^T     (Q.K^T with Q in smem)
//   1 TS  M=256 N=128 : D += A(TMEM) B(smem, K-major)^T     (Q.K^T with Q in TMEM)
//   2 TS  M=256 N=128 : D += A(TMEM) B(smem, MN-major)      (P.V)
//   3 SS  M=256 N=256 : the GEMM's pair shape
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include
//        -I paper_2605_02953_b200/csrc tools/mma_rate_pair.cu -o tools/mma_rate_pair.bin
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

__device__ __forceinline__ void mma_ts_pair(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) rate_pair_kernel(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t cta = cluster_ctarank();
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (cta == 0 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t id128 = umma_idesc_bf16(256, 128);
    constexpr uint32_t id256 = umma_idesc_bf16(256, 256);
    constexpr uint32_t idpv = umma_idesc_bf16(256, 128) | (1u << 16);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0)
          umma_bf16_pair(tmem, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), id128, 1);
        else if (MODE == 1)
          mma_ts_pair(tmem, tmem + 384 + kk * 8, umma_desc_k_sw128(b + kk * 32), id128, 1);
        else if (MODE == 2)
          mma_ts_pair(tmem + 256, tmem + kk * 8, desc_mn(b + kk * 2048, 16384), idpv, 1);
        else
          umma_bf16_pair(tmem, umma_desc_k_sw128(a + kk * 32), umma_desc_k_sw128(b + kk * 32), id256, 1);
      }
    }
    umma_commit_pair_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[MODE] = t1 - t0;
  } else if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_pair(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int iters = 2000;
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[4] = {"pair SS M256 N128 (QK^T, Q smem)", "pair TS M256 N128 (QK^T, Q TMEM)",
                          "pair TS M256 N128 MN-major B (PV)", "pair SS M256 N256 (GEMM)"};
  const int ns[4] = {128, 128, 128, 256};
  auto run = [&](auto kern, int mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    kern<<<nsm & ~1, 128, 65536 + 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[8];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double per = static_cast<double>(h[mode]) / (iters * 8.0);
    const double flop_sm = 2.0 * 128 * ns[mode] * 16;  // per SM per instruction (its 128 rows)
    printf("%-36s %s  %7.1f clk/MMA  %6.0f FLOP/clk/SM\n", names[mode], cudaGetErrorString(e), per, flop_sm / per);
  };
  run(rate_pair_kernel<0>, 0);
  run(rate_pair_kernel<1>, 1);
  run(rate_pair_kernel<2>, 2);
  run(rate_pair_kernel<3>, 3);
  return 0;
}
