// Operand preparation for the reference's float32 contract.
//
// The reference computes in float32 (numpy/BLAS, ovs/kernels/oracles.py:12-27) and
// its tests pin unordered float paths to a norm-relative error of 1e-5
// (tests/test_kernels.py:365-381).  The tensor cores here take bf16 (8 significant
// bits), so a float32 operand x is split exactly-enough into three bf16 terms
//     x = x0 + x1 + x2,  x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1)
// (24 significant bits in all), and the product a*b is expanded into the six
// terms with i + j <= 2: a0b0, a0b1, a1b0, a0b2, a1b1, a2b0 (the dropped terms
// are ~2^-24 relative).  The six products are laid out along K so the unchanged
// GEMM (and every fused protocol around it: the AllGather of A rows, the K-sharded
// ReduceScatter, the AllReduce) computes sum_k sum_terms in fp32 accumulation:
//     A' = [a0 | a0 | a1 | a0 | a1 | a2]      (role 0, 6*kp columns)
//     B' = [b0 | b1 | b0 | b2 | b1 | b0]      (role 1)
// Integer-lattice inputs are exact in x0 alone (x1 = x2 = 0), so the reference's
// bitwise float tests stay bitwise.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tf_internal.h"

namespace tf {
namespace {

__constant__ int kTermA[6] = {0, 0, 1, 0, 1, 2};
__constant__ int kTermB[6] = {0, 1, 0, 2, 1, 0};

// one thread per (row, 4 source columns); writes 6 x 4 bf16
__global__ void split3_kernel(const float* __restrict__ src, int64_t rows, int64_t k, int64_t ld_src,
                              __nv_bfloat16* __restrict__ dst, int64_t kp, int role) {
  const int64_t groups = (kp + 3) / 4;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * groups) return;
  const int64_t r = idx / groups, c0 = (idx % groups) * 4;
  __nv_bfloat16 t[3][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t c = c0 + j;
    const float x = (c < k) ? src[r * ld_src + c] : 0.f;
    const __nv_bfloat16 x0 = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(x0);
    const __nv_bfloat16 x1 = __float2bfloat16_rn(r1);
    const __nv_bfloat16 x2 = __float2bfloat16_rn(r1 - __bfloat162float(x1));
    t[0][j] = x0; t[1][j] = x1; t[2][j] = x2;
  }
  const int* term = role == 0 ? kTermA : kTermB;
  __nv_bfloat16* row = dst + r * 6 * kp;
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    const int w = term[s];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (c0 + j < kp) row[s * kp + c0 + j] = t[w][j];
  }
}

}  // namespace
}  // namespace tf

extern "C" {

int tf_split_f32_bf16x3(const float* src, int64_t rows, int64_t k, int64_t ld_src, void* dst, int64_t kp,
                        int role, void* stream) {
  if (rows < 0 || k < 0 || kp < k || ld_src < k) return tf::fail(TF_ERR_INVALID, "bad split shape");
  if (role != 0 && role != 1) return tf::fail(TF_ERR_INVALID, "role must be 0 (A) or 1 (B)");
  if (rows == 0 || kp == 0) return TF_OK;
  if (!src || !dst) return tf::fail(TF_ERR_INVALID, "NULL operand");
  const int64_t total = rows * ((kp + 3) / 4);
  const unsigned blocks = static_cast<unsigned>((total + 255) / 256);
  tf::split3_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, rows, k, ld_src, static_cast<__nv_bfloat16*>(dst), kp, role);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

}  // extern "C"
