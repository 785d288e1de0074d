// Internal declarations shared by the CUDA translation units of libtilefuse.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/tilefuse.h"

namespace tf {

constexpr int kMaxWorld = TF_MAX_WORLD;

// Thread-local error text returned by tf_last_error().
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
#define TF_CUDA_TRY(expr)                                                             \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return ::tf::fail(TF_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// One launch of the persistent sm_100a GEMM (see tf_gemm.cu).
struct GemmLaunch {
  // operands: A [M, K] row-major (lda elems), B [N, K] row-major (ldb elems), bf16
  const void* a = nullptr;
  const void* b = nullptr;
  int64_t m = 0, n = 0, k = 0, lda = 0, ldb = 0;
  // tiling / order (reference WorkloadContext semantics, ovs/kernels/context.py:18-54)
  int block_m = 128;                 // 128 = one CTA per tile, 256 = CTA pair (cta_group::2)
  int block_n = 256;
  int group_m = 8;
  int num_sms = 0;                   // persistent CTAs (reference num_gemm_sms); 0 = all SMs
  const int32_t* tile_map = nullptr; // device [num_pid_m] permutation or nullptr
  // epilogue
  int epilogue = 0;                  // 0 = store C, 1 = scatter row-slices to owners
  int out_f32 = 0;                   // 1: fp32 output, 0: bf16 output
  void* c = nullptr;
  int64_t ldc = 0;
  // AllGather consumer waits (chunk_flags[c] >= epoch before reading rows of chunk c)
  const uint64_t* chunk_flags = nullptr;
  uint64_t epoch = 0;
  int64_t rows_per_chunk = 0;
  int chunks_per_rank = 1;           // flags per source rank (sub-chunked pulls)
  // ReduceScatter producer (scatter epilogue)
  int rank = 0, world = 1;
  int64_t rows_per_rank = 0;
  void* peer_slots[kMaxWorld] = {};     // owner's slot buffer base, [world*rows_per_rank, slot_ld]
  uint64_t* peer_counts[kMaxWorld] = {};// owner's per-row-tile arrival counters
  int64_t slot_ld = 0;
  unsigned long long* err = nullptr;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  bool no_tail_split = false;        // disable the split-K tail (e.g. inside fused protocols)
  bool wait_on_b = false;            // chunk flags guard B rows (gathered N-side operand)
  const int32_t* tile_map_n = nullptr; // device [num_pid_n] permutation or nullptr
  int trace_rank = 0;                // rank tag for device trace events
  // grouped (MoE) mode: a = gathered rows [m, k], b = stacked experts [n_experts * n, k]
  const void* moe_tab = nullptr;     // device int4 [moe_slots] {expert, row0, rows, segs}
  int moe_slots = 0;
  int n_experts = 0;
  const uint64_t* src_flags = nullptr;
  uint64_t src_target = 0;
  int comm_ctas = 0;                 // pull-engine CTAs in front of the GEMM CTAs
  const uint8_t* peer_ws[kMaxWorld] = {};
  uint8_t* own_ws = nullptr;
  const int32_t* irb = nullptr;
  const int32_t* dstb = nullptr;
  int64_t row_bytes = 0;
  uint64_t* own_flags = nullptr;
};

int launch_gemm(const GemmLaunch& g, cudaStream_t stream);
void layer_release_team(const tf_team* t);
int num_sms_of_current_device();
// device trace ring of `device` (tf_trace_enable) and its capacity, or 0 / nullptr
int trace_buffer(int device, unsigned long long** buf);
// SM -> die table (tf_topo.cu): device [256] die ids by %smid plus a per-launch counter
// slot (a ring of kDieCtrSlots self-resetting counters), or nullptr without two dies
constexpr int kDieCtrSlots = 64;
const uint8_t* sm_die_table(int dev, unsigned long long** ctr_slot);

}  // namespace tf
