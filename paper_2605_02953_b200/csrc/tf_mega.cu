// Task-level megakernel executor (ovs/megakernel/runner.py:120-195).
//
// One persistent launch co-schedules every rank of a local team: CTA b serves
// rank b / num_sms, queue b % num_sms.  Each CTA drains its static queue
// ([slot][sm][30] int32 records, encoding.py:127-166): fetch the record,
// acquire-wait the dependency flags (scoreboard slot = task * max_tiles + tile,
// scoreboard.py:33-48; allreduce tasks wait on every peer's copy), run the task,
// release its flag (.sys, so peers can poll it).
//   linear     y[tile] = x[rows] . w[cols]^T, a tcgen05 kind::tf32 tile: fp32
//              operands staged into 128-byte-swizzled smem, fp32 TMEM accumulator
//              (exact for the reference's integer-valued "exact mode" data)
//   add        y[rows] = a[rows] + b[rows]
//   allreduce  y[rows] = sum over ranks (ascending) of x_rank[rows], read over
//              P2P -- the multimem_ld_reduce of runner.py:173-188
// Tensors are fp32 [rows, cols] at their io-slot byte offsets in each PE's heap.
#include <cuda_runtime.h>

#include <string>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

constexpr int kIntPerTask = 30;
constexpr int kIoOff = 6;
constexpr int kIoSlot = 6;
constexpr int kMegaThreads = 128;
constexpr int kKB = 32;  // fp32 per 128-byte row

struct MegaParams {
  const int32_t* queues;
  const int32_t* counts;
  const int32_t* deps;
  const int32_t* layer_cfg;  // [layers][4]: op, block_m, block_n, block_rows
  int num_sms, max_tiles;
  uint64_t flag_base;
  unsigned long long epoch;
  unsigned long long timeout_ns;
  int world;
  uint8_t* base[kMaxWorld];
  uint64_t* sig[kMaxWorld];
  unsigned long long* err[kMaxWorld];
};

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__host__ __device__ constexpr uint32_t umma_idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// stage rows [r0, r0 + nrows) x k-cols [k0, k0 + 32) of a fp32 [rows, cols] tensor into
// a 128-byte-swizzled K-major tile (row r at r*128, 16-byte chunk j at (j ^ r%8) * 16),
// zero outside [valid_rows) x [cols)
__device__ __forceinline__ void stage_tile(uint8_t* dst, const float* src, int rows, int cols,
                                           int r0, int nrows, int valid_rows, int k0) {
  for (int i = threadIdx.x; i < nrows * 8; i += blockDim.x) {
    const int r = i >> 3, j = i & 7;
    const int gr = r0 + r, gc = k0 + j * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < valid_rows && gr < rows) {
      const float* p = src + static_cast<long long>(gr) * cols + gc;
      if (gc < cols) v.x = p[0];
      if (gc + 1 < cols) v.y = p[1];
      if (gc + 2 < cols) v.z = p[2];
      if (gc + 3 < cols) v.w = p[3];
    }
    *reinterpret_cast<float4*>(dst + r * 128 + ((j ^ (r & 7)) << 4)) = v;
  }
}

constexpr int kMegaSmem = 1024 + 128 * 128 + 256 * 128;

__global__ void __launch_bounds__(kMegaThreads, 1) megakernel(const __grid_constant__ MegaParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sa = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));  // A: 128 x 32 fp32
  uint8_t* sb = sa + 128 * 128;                                                       // B: <= 256 x 32 fp32
  __shared__ uint64_t mma_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t task[kIntPerTask];
  const int rank = blockIdx.x / p.num_sms;
  const int sm = blockIdx.x % p.num_sms;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&mma_bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  uint32_t mma_phase = 0;
  uint64_t* flags = p.sig[rank] + p.flag_base;
  const int n_tasks = p.counts[sm];

  for (int idx = 0; idx < n_tasks; ++idx) {
    if (threadIdx.x < kIntPerTask)
      task[threadIdx.x] = p.queues[(static_cast<long long>(idx) * p.num_sms + sm) * kIntPerTask + threadIdx.x];
    __syncthreads();
    const int task_id = task[2], tile = task[3];
    const int* cfg = p.layer_cfg + task_id * 4;
    const int op = cfg[0];
    // ---- wait dependencies (allreduce: on every rank's scoreboard)
    const int npe = op == 2 ? p.world : 1;
    for (int row = task[4]; row < task[5]; ++row) {
      const int prod = p.deps[row * 3], lo = p.deps[row * 3 + 1], hi = p.deps[row * 3 + 2];
      for (int i = threadIdx.x; i < (hi - lo) * npe; i += blockDim.x) {
        const int t = lo + i / npe;
        const int pe = npe == 1 ? rank : i % npe;
        const uint64_t slot = static_cast<uint64_t>(prod) * p.max_tiles + t;
        wait_geq_sys(p.sig[pe] + p.flag_base + slot, p.epoch, p.timeout_ns, p.err[rank],
                     0x8000000ull | slot);
      }
    }
    __syncthreads();
    // ---- io slots
    auto io_ptr = [&](int i, int pe) -> float* {
      return reinterpret_cast<float*>(p.base[pe] + task[kIoOff + i * kIoSlot]);
    };
    auto io_dim = [&](int i, int d) { return task[kIoOff + i * kIoSlot + 2 + d]; };
    if (op == 0) {  // ---------------------------------------------------- linear
      const float* x = io_ptr(0, rank);
      const float* w = io_ptr(1, rank);
      float* y = io_ptr(2, rank);
      const int m = io_dim(0, 0), k = io_dim(0, 1), n = io_dim(1, 0);
      const int bm = cfg[1], bn = cfg[2];
      const int ntn = (n + bn - 1) / bn;
      const int r0 = (tile / ntn) * bm, c0 = (tile % ntn) * bn;
      const int npad = ((bn + 15) / 16) * 16;
      const uint32_t idesc = umma_idesc_tf32(128, npad);
      for (int k0 = 0; k0 < k; k0 += kKB) {
        stage_tile(sa, x, m, k, r0, 128, bm, k0);
        stage_tile(sb, w, n, k, c0, npad, bn, k0);
        fence_proxy_async_shared();
        __syncthreads();
        if (threadIdx.x == 0) {
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < kKB / 8; ++kk)  // kind::tf32: K = 8 per instruction (32 B)
            umma_tf32(tmem, umma_desc_k_sw128(smem_u32(sa) + kk * 32),
                      umma_desc_k_sw128(smem_u32(sb) + kk * 32), idesc, (k0 | kk) != 0);
          umma_commit(&mma_bar);
        }
        mbar_wait(&mma_bar, mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
      }
      // epilogue: TMEM lane = tile row, column = tile col
      const int row = warp * 32 + lane;
      for (int cc = 0; cc < npad; cc += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cc, v);
        tmem_ld_wait();
        if (row < bm && r0 + row < m)
          for (int j = 0; j < 32; ++j) {
            const int c = cc + j;
            if (c < bn && c0 + c < n)
              y[static_cast<long long>(r0 + row) * n + c0 + c] = __uint_as_float(v[j]);
          }
      }
      tc_fence_before();
    } else {  // ------------------------------------------------------- add / allreduce
      const int br = cfg[3];
      const int rows = io_dim(0, 0), cols = io_dim(0, 1);
      const int r0 = tile * br, r1 = min(r0 + br, rows);
      const long long lo = static_cast<long long>(r0) * cols, hi = static_cast<long long>(r1) * cols;
      if (op == 1) {
        const float* a = io_ptr(0, rank);
        const float* b = io_ptr(1, rank);
        float* y = io_ptr(2, rank);
        for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) y[i] = a[i] + b[i];
      } else {
        float* y = io_ptr(1, rank);
        for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
          float acc = 0.f;
          for (int pe = 0; pe < p.world; ++pe) acc += io_ptr(0, pe)[i];  // ascending team rank
          y[i] = acc;
        }
      }
    }
    // ---- release (scoreboard.py:50-56): double release is a protocol error
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t slot = static_cast<uint64_t>(task_id) * p.max_tiles + tile;
      if (ld_acquire_sys(flags + slot) >= p.epoch) atomicCAS(p.err[rank], 0ull, 0x9000000ull | slot);
      fence_sys();
      st_release_sys(flags + slot, p.epoch);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace
}  // namespace tf

using tf::fail;

extern "C" int tf_megakernel_run(tf_team* t, const tf_mega_args* a, void* stream) {
  if (!t || !a) return fail(TF_ERR_INVALID, "NULL argument");
  if (t->ipc) return fail(TF_ERR_CONFIG, "tf_megakernel_run drives a local team (all ranks co-resident)");
  if (a->num_sms < 1) return fail(TF_ERR_INVALID, "num_sms must be >= 1");
  for (int pe = 1; pe < t->world; ++pe)
    if (t->pes[pe].device != t->pes[0].device)
      return fail(TF_ERR_CONFIG, "the co-scheduled megakernel needs every PE on one device");
  const int grid = t->world * a->num_sms;
  if (grid > tf::num_sms_of_current_device())
    return fail(TF_ERR_CONFIG, "world * num_sms CTAs must be co-resident (<= SM count)");
  tf::MegaParams p{};
  p.queues = a->queues;
  p.counts = a->counts;
  p.deps = a->deps;
  p.layer_cfg = a->layer_cfg;
  p.num_sms = a->num_sms;
  p.max_tiles = a->max_tiles;
  p.flag_base = a->flag_base;
  p.epoch = a->epoch ? a->epoch : 1;
  p.timeout_ns = a->timeout_ns ? a->timeout_ns : t->timeout_ns;
  p.world = t->world;
  for (int pe = 0; pe < t->world; ++pe) {
    p.base[pe] = t->pes[pe].base;
    p.sig[pe] = t->pes[pe].sig;
    p.err[pe] = t->err_word(pe);
  }
  static uint64_t attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    TF_CUDA_TRY(cudaFuncSetAttribute(tf::megakernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tf::kMegaSmem));
    attr_done |= 1ull << dev;
  }
  tf::megakernel<<<grid, tf::kMegaThreads, tf::kMegaSmem, static_cast<cudaStream_t>(stream)>>>(p);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}
