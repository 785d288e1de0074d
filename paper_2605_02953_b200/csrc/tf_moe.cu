// Expert-parallel MoE: routing, counts/offsets, dispatch and combine.
//
// The reference has no all-to-all -- its MoE path is AllGather +
// grouped GEMM (ovs/kernels/ag_moe.py:20-158).  What it pins, and what this
// file keeps bit-exact, is the layout:
//   * routing counts are a [world, E] matrix, entry (s, e) = rows source rank s
//     sends to expert e (ag_moe.py:28-33);
//   * a rank's chunk is grouped by expert, then keeps source order
//     (ag_moe.py:_pull_engine, oracles.py:38-50);
//   * the receive side is expert-major, then source rank, then source order
//     (gather_tokens_by_expert, oracles.py:38-50).
// Rank d owns experts [d*E/w, (d+1)*E/w).
//
// Kernels
//   topk_kernel        warp per token: k rounds of warp argmax (ties -> lower id)
//   count_fused_kernel deterministic stable send order in one launch: chunk CTAs
//                      build per-warp histograms (__match_any_sync), publish the
//                      chunk histogram with a release flag, wait for all chunks,
//                      then derive totals, expert bases, chunk offsets and ranks --
//                      no atomic decides a position, so counts, offsets and layout
//                      are bit-exact (hist / scan / rank kernels when there are
//                      more chunks than SMs)
//   layout_kernel      per-expert destination segment base on the owner
//   scatter_kernel     warp per (token, <= 8 KB row piece): TMA bulk copy into smem,
//                      bulk stores to the destination rows this rank owns, 16-byte
//                      P2P stores over NVLink to the rows peers own
//   combine_kernel     warp per token: pulls the k expert rows (16-byte loads,
//                      k loads in flight per lane), fp32 weighted sum in slot
//                      order, bf16 out
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

constexpr int kChunk = 1024;  // (token, slot) entries per ranking chunk

// ---------------------------------------------------------------- routing
// Order-preserving float -> u32 (larger float => larger key); 0 marks "taken".
__device__ __forceinline__ uint32_t f2key(float f) {
  const uint32_t b = __float_as_uint(f + 0.0f);  // -0 -> +0: equal logits tie on the id
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// Warp per token.  Each lane keeps its best remaining logit (first index on
// ties); a round is two warp reductions on the integer pipe (`redux.sync`: max
// key, then min expert id among lanes holding it), so picks are identical to a
// stable sort by (-logit, expert id).
// Lane j < k returns slot j's (expert, weight) of the token whose logits are `row`.
template <int VPL>  // logits per lane (E <= 32 * VPL)
__device__ __forceinline__ void topk_warp_scan(const float* __restrict__ row, int E, int k, int lane,
                                               int& out_idx, float& out_w) {
  uint32_t key[VPL];
#pragma unroll
  for (int c = 0; c < VPL; ++c) {  // coalesced: lane + 32c
    const int e = lane + 32 * c;
    key[c] = e < E ? f2key(row[e]) : 0u;
  }
  auto lane_best = [&](uint32_t& bk, uint32_t& bi) {
    bk = key[0];
    bi = lane;
#pragma unroll
    for (int c = 1; c < VPL; ++c)
      if (key[c] > bk) { bk = key[c]; bi = lane + 32 * c; }  // strict: first index wins
  };
  uint32_t bk, bi;
  lane_best(bk, bi);
  float sel0 = 0.f, z = 0.f, my_val = 0.f;
  int my_idx = 0;
  for (int r = 0; r < k; ++r) {
    const uint32_t m = __reduce_max_sync(0xffffffffu, bk);
    const uint32_t wi = __reduce_min_sync(0xffffffffu, bk == m ? bi : 0xFFFFFFFFu);
    if ((wi & 31) == static_cast<uint32_t>(lane)) {
#pragma unroll
      for (int c = 0; c < VPL; ++c)
        if (c == static_cast<int>(wi >> 5)) key[c] = 0u;  // taken
      lane_best(bk, bi);
    }
    const float best = key2f(m);
    if (r == 0) sel0 = best;
    const float ez = __expf(best - sel0);
    z += ez;
    if (lane == r) { my_val = ez; my_idx = static_cast<int>(wi); }
  }
  out_idx = my_idx;
  out_w = my_val / z;
}

// Same picks with each lane's keys pre-sorted (odd-even transposition, stable: equal
// keys keep the lower expert id first), so a round is one max reduction, a ballot of
// the lanes whose head holds it (a second reduction only on a cross-lane tie) and a
// register shift in the winning lane -- instead of two reductions and a rescan.
template <int VPL>
__device__ __forceinline__ void topk_warp_sorted(const float* __restrict__ row, int E, int k, int lane,
                                                 int& out_idx, float& out_w) {
  uint32_t key[VPL], id[VPL];
#pragma unroll
  for (int c = 0; c < VPL; ++c) {  // coalesced: lane + 32c
    const int e = lane + 32 * c;
    key[c] = e < E ? f2key(row[e]) : 0u;
    id[c] = static_cast<uint32_t>(e);
  }
#pragma unroll
  for (int rnd = 0; rnd < VPL; ++rnd)
#pragma unroll
    for (int a = rnd & 1; a + 1 < VPL; a += 2) {
      const bool sw = key[a + 1] > key[a];  // strict: stable
      const uint32_t k0 = sw ? key[a + 1] : key[a], k1 = sw ? key[a] : key[a + 1];
      const uint32_t i0 = sw ? id[a + 1] : id[a], i1 = sw ? id[a] : id[a + 1];
      key[a] = k0; key[a + 1] = k1; id[a] = i0; id[a + 1] = i1;
    }
  float sel0 = 0.f, z = 0.f, my_val = 0.f;
  int my_idx = 0;
  for (int r = 0; r < k; ++r) {
    const uint32_t m = __reduce_max_sync(0xffffffffu, key[0]);
    const unsigned hold = __ballot_sync(0xffffffffu, key[0] == m);
    uint32_t wi;
    if (__popc(hold) == 1) wi = __shfl_sync(0xffffffffu, id[0], __ffs(hold) - 1);
    else wi = __reduce_min_sync(0xffffffffu, key[0] == m ? id[0] : 0xFFFFFFFFu);
    if ((wi & 31) == static_cast<uint32_t>(lane)) {  // pop the head
#pragma unroll
      for (int c = 0; c + 1 < VPL; ++c) { key[c] = key[c + 1]; id[c] = id[c + 1]; }
      key[VPL - 1] = 0u;
    }
    const float best = key2f(m);
    if (r == 0) sel0 = best;
    const float ez = __expf(best - sel0);
    z += ez;
    if (lane == r) { my_val = ez; my_idx = static_cast<int>(wi); }
  }
  out_idx = my_idx;
  out_w = my_val / z;
}

#ifndef TF_MOE_TOPK_SORTED
#define TF_MOE_TOPK_SORTED 1
#endif
template <int VPL>
__device__ __forceinline__ void topk_warp(const float* __restrict__ row, int E, int k, int lane,
                                          int& out_idx, float& out_w) {
  if constexpr (TF_MOE_TOPK_SORTED && VPL <= 8) topk_warp_sorted<VPL>(row, E, k, lane, out_idx, out_w);
  else topk_warp_scan<VPL>(row, E, k, lane, out_idx, out_w);
}

template <int VPL>
__global__ void topk_kernel(const float* __restrict__ logits, int64_t tokens, int E, int k,
                            int32_t* __restrict__ idx, float* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= tokens) return;
  int my_idx;
  float my_w;
  topk_warp<VPL>(logits + t * E, E, k, lane, my_idx, my_w);
  if (lane < k) {
    idx[t * k + lane] = my_idx;
    w[t * k + lane] = my_w;
  }
}

// ---------------------------------------------------------------- stable counting
__global__ void hist_kernel(const int32_t* __restrict__ idx, int64_t entries, int E,
                            int32_t* __restrict__ chunk_hist /* [nchunks][E] */) {
  extern __shared__ int32_t h[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kChunk;
  for (int i = threadIdx.x; i < kChunk; i += blockDim.x) {
    const int64_t g = base + i;
    if (g < entries) {
      const int e = idx[g];
      if (e >= 0 && e < E) atomicAdd(&h[e], 1);  // order-independent count
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    chunk_hist[static_cast<int64_t>(blockIdx.x) * E + e] = h[e];
}

// block-wide exclusive scan of n (<= 1024 * 4) ints in smem, 1024 threads
__device__ void block_exclusive_scan(int32_t* data, int n) {
  __shared__ int32_t warp_tot[32];
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(lo + per, n);
  int32_t local = 0;
  for (int i = lo; i < hi; ++i) local += data[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x / 32;
    int32_t x = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t o = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += o;
    }
    if (lane < nw) warp_tot[lane] = x;  // inclusive over warps
  }
  __syncthreads();
  int32_t run = incl - local + (warp > 0 ? warp_tot[warp - 1] : 0);
  for (int i = lo; i < hi; ++i) {
    const int32_t v = data[i];
    data[i] = run;
    run += v;
  }
  __syncthreads();
}

// one block of 1024: per-expert exclusive scan over chunks, totals, expert bases
__global__ void __launch_bounds__(1024) scan_kernel(int32_t* __restrict__ chunk_hist, int nchunks,
                                                    int E, int32_t* __restrict__ counts,
                                                    int32_t* __restrict__ expert_base) {
  extern __shared__ int32_t tot[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t run = 0;
    for (int c0 = 0; c0 < nchunks; c0 += 16) {  // 16 independent loads in flight
      int32_t v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        v[u] = c0 + u < nchunks ? chunk_hist[static_cast<int64_t>(c0 + u) * E + e] : 0;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (c0 + u < nchunks) {
          chunk_hist[static_cast<int64_t>(c0 + u) * E + e] = run;
          run += v[u];
        }
    }
    tot[e] = run;
    counts[e] = run;
  }
  __syncthreads();
  block_exclusive_scan(tot, E);
  for (int e = threadIdx.x; e < E; e += blockDim.x) expert_base[e] = tot[e];
}

// 1024 threads: entry i of the chunk; rank among same-expert entries before it.
__global__ void __launch_bounds__(kChunk) rank_kernel(const int32_t* __restrict__ idx,
                                                      int64_t entries, int E,
                                                      const int32_t* __restrict__ chunk_off,
                                                      const int32_t* __restrict__ expert_base,
                                                      int32_t* __restrict__ sorted_pos) {
  extern __shared__ int32_t wc[];  // [32 warps][E]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  const int64_t g = static_cast<int64_t>(blockIdx.x) * kChunk + threadIdx.x;
  const int e = g < entries ? idx[g] : -1;
  const unsigned same = __match_any_sync(0xffffffffu, e);
  const int in_warp = __popc(same & ((1u << lane) - 1));
  if (e >= 0 && in_warp == 0) wc[warp * E + e] = __popc(same);
  __syncthreads();
  if (e >= 0) {
    int before = 0;
    for (int w2 = 0; w2 < warp; ++w2) before += wc[w2 * E + e];
    sorted_pos[g] = expert_base[e] + chunk_off[static_cast<int64_t>(blockIdx.x) * E + e] + before +
                    in_warp;
  }
}


// Single-pass stable counting (hist + scan + rank in one launch): every chunk CTA
// (1024 entries) builds its per-warp and chunk histograms, publishes the chunk
// histogram with a release flag, waits until every chunk has published (all chunk
// CTAs are co-resident), then derives the totals, the expert bases and its own
// chunk offsets and writes the stable send positions.  Same arithmetic as the
// three-kernel path, so positions are identical.
__global__ void __launch_bounds__(kChunk) count_fused_kernel(
    const int32_t* __restrict__ idx, int64_t entries, int E, int nchunks, int32_t* chunk_hist,
    unsigned long long* flags, unsigned long long epoch, unsigned long long timeout_ns,
    unsigned long long* err, int32_t* __restrict__ counts, int32_t* __restrict__ expert_base,
    int32_t* __restrict__ sorted_pos) {
  extern __shared__ int32_t fsm[];
  const int parts = max(1, kChunk / E);  // threads per expert for the cross-chunk sums
  int32_t* wc = fsm;                // [32 warps][E] -> exclusive prefix over warps
  int32_t* tot = fsm + 32 * E;      // [E]
  int32_t* off = tot + E;           // [E]
  int32_t* part_t = off + E;        // [parts][E]
  int32_t* part_o = part_t + parts * E;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) wc[i] = 0;
  __syncthreads();
  const int64_t g = static_cast<int64_t>(c) * kChunk + threadIdx.x;
  const int e = g < entries ? idx[g] : -1;
  const unsigned same = __match_any_sync(0xffffffffu, e);
  const int in_warp = __popc(same & ((1u << lane) - 1));
  if (e >= 0 && in_warp == 0) wc[warp * E + e] = __popc(same);
  __syncthreads();
  for (int x = threadIdx.x; x < E; x += blockDim.x) {
    int32_t sum = 0;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {  // in place: per-warp counts -> exclusive prefix
      const int32_t v = wc[w * E + x];
      wc[w * E + x] = sum;
      sum += v;
    }
    chunk_hist[static_cast<int64_t>(c) * E + x] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flags + c), "l"(epoch) : "memory");
  }
  for (int x = threadIdx.x; x < nchunks; x += blockDim.x) {
    uint64_t v;
    const uint64_t t0 = globaltimer_ns();
    while (true) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + x) : "memory");
      if (v >= epoch) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        if (err) atomicCAS(err, 0ull, 0x5200000ull | static_cast<unsigned>(x));
        break;
      }
    }
  }
  __syncthreads();
  // totals and this chunk's offsets: `parts` threads per expert, strided chunks
  for (int i = threadIdx.x; i < parts * E; i += blockDim.x) {
    const int x = i % E, part = i / E;
    int32_t t = 0, o = 0;
#pragma unroll 8
    for (int cc = part; cc < nchunks; cc += parts) {
      const int32_t v = __ldcg(chunk_hist + static_cast<int64_t>(cc) * E + x);
      o += cc < c ? v : 0;
      t += v;
    }
    part_t[part * E + x] = t;
    part_o[part * E + x] = o;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < E; x += blockDim.x) {
    int32_t t = 0, o = 0;
    for (int part = 0; part < parts; ++part) {
      t += part_t[part * E + x];
      o += part_o[part * E + x];
    }
    tot[x] = t;
    off[x] = o;
  }
  __syncthreads();
  if (c == 0)
    for (int x = threadIdx.x; x < E; x += blockDim.x) counts[x] = tot[x];
  block_exclusive_scan(tot, E);  // expert bases (ends with __syncthreads)
  if (c == 0)
    for (int x = threadIdx.x; x < E; x += blockDim.x) expert_base[x] = tot[x];
  if (e >= 0) sorted_pos[g] = tot[e] + off[e] + wc[warp * E + e] + in_warp;
}

// ---------------------------------------------------------------- exchange / layout
struct PeerPtrs {
  void* p[kMaxWorld];
};
struct PeerSig {
  uint64_t* p[kMaxWorld];
};

// push this rank's count row into every peer's matrix, then release its flag
__global__ void push_counts_kernel(const int32_t* __restrict__ row, int E, PeerPtrs mats,
                                   PeerSig flags, int world, int rank, uint64_t epoch) {
  for (int p = 0; p < world; ++p) {
    int32_t* dst = static_cast<int32_t*>(mats.p[p]) + static_cast<int64_t>(rank) * E;
    for (int e = threadIdx.x; e < E; e += blockDim.x) dst[e] = row[e];
  }
  __syncthreads();
  if (threadIdx.x < world) {
    fence_sys();
    st_release_sys(flags.p[threadIdx.x] + rank, epoch);
  }
}

__global__ void wait_flags_kernel(const uint64_t* flags, int n, uint64_t epoch, uint64_t timeout_ns,
                                  unsigned long long* err, unsigned long long tag) {
  const int i = threadIdx.x;
  if (i < n) wait_geq_sys(flags + i, epoch, timeout_ns, err, tag | i);
  __syncthreads();
}

// seg_base[e] = start row, on e's owner, of the segment (expert e, source `rank`):
// exclusive scan of expert totals inside each owner's expert range, plus the rows
// of lower source ranks for the same expert.  One block of 1024 threads.
__global__ void __launch_bounds__(1024) layout_kernel(const int32_t* __restrict__ mat, int world,
                                                      int E, int rank,
                                                      int32_t* __restrict__ seg_base,
                                                      int32_t* __restrict__ counts_out,
                                                      int64_t* __restrict__ recv_rows) {
  extern __shared__ int32_t tot[];  // [E]
  const int epr = E / world;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int32_t t = 0;
    for (int s = 0; s < world; ++s) t += mat[s * E + e];
    tot[e] = t;
  }
  for (int i = threadIdx.x; i < world * E; i += blockDim.x) counts_out[i] = mat[i];
  __syncthreads();
  __shared__ int32_t last_tot;
  if (threadIdx.x == 0) last_tot = tot[(rank + 1) * epr - 1];
  block_exclusive_scan(tot, E);  // global exclusive prefix over experts
  if (threadIdx.x == 0) *recv_rows = static_cast<int64_t>(tot[(rank + 1) * epr - 1]) + last_tot -
                                     tot[rank * epr];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int owner_first = (e / epr) * epr;
    int32_t base = tot[e] - tot[owner_first];  // rows of lower experts on the same owner
    for (int s = 0; s < rank; ++s) base += mat[s * E + e];
    seg_base[e] = base;
  }
}

// warp per (token, piece of <= 8 KB of the row): one bulk copy (TMA engine) brings the
// piece of x[t] into this warp's smem buffer; destination rows on this rank are
// written by bulk stores, rows owned by peers by the warp's 16-byte P2P stores over
// NVLink.  Lane j < k resolves slot j's destination row.
constexpr int kScatterWarps = 8;
constexpr int kScatterBuf = 8192;  // bytes per warp (>= half a row, 16-byte multiple)

__global__ void __launch_bounds__(32 * kScatterWarps) scatter_kernel(
    const uint4* __restrict__ x, int64_t tokens, int64_t vec_per_row, int k, int E, int world,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ sorted_pos,
    const int32_t* __restrict__ expert_base, const int32_t* __restrict__ seg_base,
    int32_t* __restrict__ dest_row, PeerPtrs recv, int64_t max_recv, unsigned long long* err, int rank) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ uint64_t bar[kScatterWarps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* buf = sbuf + wib * kScatterBuf;
  if (lane == 0) {
    mbar_init(&bar[wib], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t phase = 0;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int epr = E / world;
  constexpr int64_t kPiece = kScatterBuf / 16;  // uint4 per piece
  const int64_t npieces = (vec_per_row + kPiece - 1) / kPiece;
  for (int64_t wi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       wi < tokens * npieces; wi += nwarps) {
    const int64_t t = wi / npieces, piece = wi % npieces;
    const int64_t v0 = piece * kPiece, v1 = min(v0 + kPiece, vec_per_row);
    const uint32_t bytes = static_cast<uint32_t>((v1 - v0) * 16);
    uint4* my_dst = nullptr;
    int my_remote = 0;
    if (lane < k) {
      const int64_t slot = t * k + lane;
      const int e = idx[slot];
      const int64_t row = static_cast<int64_t>(seg_base[e]) + (sorted_pos[slot] - expert_base[e]);
      if (piece == 0) dest_row[slot] = static_cast<int32_t>(row);
      if (row < max_recv) my_dst = static_cast<uint4*>(recv.p[e / epr]) + row * vec_per_row + v0;
      else if (err) atomicCAS(err, 0ull, 0x5000000ull | 0xFFFFFFull);
      my_remote = (e / epr) != rank;
    }
    uint4* dsts[16];
#pragma unroll
    for (int j = 0; j < 16; ++j)
      dsts[j] = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_dst), j));
    const unsigned remote = __ballot_sync(0xffffffffu, my_remote != 0 && my_dst != nullptr);
    if (lane == 0) {
      // the previous half row's stores must have finished reading the buffer
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_arrive_expect_tx(&bar[wib], bytes);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(buf)),
          "l"(x + t * vec_per_row + v0), "r"(bytes), "r"(smem_u32(&bar[wib]))
          : "memory");
    }
    mbar_wait(&bar[wib], phase);  // every lane: the bulk load's bytes are visible
    if (lane == 0) {
      // local owner: bulk store straight from smem on the TMA engine
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < k && dsts[j] != nullptr && !((remote >> j) & 1))
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dsts[j]),
                       "r"(smem_u32(buf)), "r"(bytes)
                       : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // remote owners: 16-byte P2P stores over NVLink from the staged row piece
    for (int j = 0; j < k; ++j) {
      if (!((remote >> j) & 1)) continue;
      const uint4* sb = reinterpret_cast<const uint4*>(buf);
      for (int v = lane; v < static_cast<int>(bytes / 16); v += 32) dsts[j][v] = sb[v];
    }
    phase ^= 1;
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores globally done
}

// Persistent, double-buffered variant: each warp walks (token, piece) tasks with a
// grid stride and keeps two row pieces in shared memory, so the bulk load of task
// i+1 is in flight while task i's bulk / P2P stores drain.
constexpr int kScatter2Warps = 4;
constexpr int kScatter2Buf = 8192;  // bytes per buffer, two buffers per warp

__global__ void __launch_bounds__(32 * kScatter2Warps) scatter2_kernel(
    const uint4* __restrict__ x, int64_t tokens, int64_t vec_per_row, int k, int E, int world,
    const int32_t* __restrict__ idx, const int32_t* __restrict__ sorted_pos,
    const int32_t* __restrict__ expert_base, const int32_t* __restrict__ seg_base,
    int32_t* __restrict__ dest_row, PeerPtrs recv, int64_t max_recv, unsigned long long* err, int rank) {
  extern __shared__ __align__(128) uint8_t sbuf[];
  __shared__ uint64_t bar[2 * kScatter2Warps];
  __shared__ uint4* sdst[kScatter2Warps][16];  // this task's destinations (lane j -> slot j)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* const buf0 = sbuf + (2 * wib) * kScatter2Buf;  // buffer b at buf0 + b * kScatter2Buf
  uint64_t* bars = bar + 2 * wib;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
  }
  __syncwarp();
  uint32_t phases = 0;  // bit b: parity of buffer b's barrier
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int epr = E / world;
  constexpr int64_t kPiece = kScatter2Buf / 16;  // uint4 per piece
  const int64_t npieces = (vec_per_row + kPiece - 1) / kPiece;
  const int64_t ntasks = tokens * npieces;
  auto piece_bytes = [&](int64_t wi) {
    const int64_t v0 = (wi % npieces) * kPiece;
    return static_cast<uint32_t>((min(v0 + kPiece, vec_per_row) - v0) * 16);
  };
  auto issue_load = [&](int64_t wi, int b) {  // lane 0 only
    const int64_t t = wi / npieces, v0 = (wi % npieces) * kPiece;
    const uint32_t bytes = piece_bytes(wi);
    mbar_arrive_expect_tx(&bars[b], bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf0 + b * kScatter2Buf)),
        "l"(x + t * vec_per_row + v0), "r"(bytes), "r"(smem_u32(&bars[b]))
        : "memory");
  };
  int64_t wi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (lane == 0 && wi < ntasks) issue_load(wi, 0);
  for (int b = 0; wi < ntasks; wi += nwarps, b ^= 1) {
    const int64_t t = wi / npieces, piece = wi % npieces;
    const int64_t v0 = piece * kPiece;
    const uint32_t bytes = piece_bytes(wi);
    uint4* my_dst = nullptr;
    int my_remote = 0;
    if (lane < k) {
      const int64_t slot = t * k + lane;
      const int e = idx[slot];
      const int64_t row = static_cast<int64_t>(seg_base[e]) + (sorted_pos[slot] - expert_base[e]);
      if (piece == 0) dest_row[slot] = static_cast<int32_t>(row);
      if (row < max_recv) my_dst = static_cast<uint4*>(recv.p[e / epr]) + row * vec_per_row + v0;
      else if (err) atomicCAS(err, 0ull, 0x5000000ull | 0xFFFFFFull);
      my_remote = (e / epr) != rank;
    }
    if (lane < k) sdst[wib][lane] = my_dst;
    __syncwarp();
    const unsigned remote = __ballot_sync(0xffffffffu, my_remote != 0 && my_dst != nullptr);
    mbar_wait(&bars[b], (phases >> b) & 1);  // task wi's piece is in buffer b
    phases ^= 1u << b;
    if (lane == 0) {
      // the other buffer's stores (task wi - nwarps) must have finished reading it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (wi + nwarps < ntasks) issue_load(wi + nwarps, b ^ 1);
      for (int j = 0; j < k; ++j)
        if (sdst[wib][j] != nullptr && !((remote >> j) & 1))
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst[wib][j]),
                       "r"(smem_u32(buf0 + b * kScatter2Buf)), "r"(bytes)
                       : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (int j = 0; j < k; ++j) {
      if (!((remote >> j) & 1)) continue;
      uint4* d = reinterpret_cast<uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_dst), j));
      const uint4* sb = reinterpret_cast<const uint4*>(buf0 + b * kScatter2Buf);
      for (int v = lane; v < static_cast<int>(bytes / 16); v += 32) d[v] = sb[v];
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores globally done
}

// after the scatter kernel (stream order): release "source `rank` delivered" on every owner
__global__ void release_kernel(PeerSig flags, int world, int rank, uint64_t epoch) {
  if (threadIdx.x < world) {
    fence_sys();
    st_release_sys(flags.p[threadIdx.x] + rank, epoch);
  }
}

// ---------------------------------------------------------------- fused dispatch
// One persistent launch per rank replaces topk + count + push + wait + layout +
// scatter + release: CTA c owns tokens [c*tpc, (c+1)*tpc).
//   PRE   (top-k of its tokens when logits are given) -> stable per-expert ranks of
//         its (token, slot) entries in token order -> chunk histogram published
//         with a release flag -> grid-wide wait -> totals, expert bases and this
//         chunk's offsets (same arithmetic as count_fused_kernel, so send positions
//         are bit-identical) -> CTA 0 pushes the count row to every peer's matrix.
//   MAIN  wait for every source's count row -> destination segment bases
//         (layout_kernel's arithmetic) -> double-buffered scatter of its own tokens
//         (bulk copy in, bulk stores to local rows, 16-byte P2P stores to peers) ->
//         the last CTA to finish releases "source `rank` delivered" on every owner.
// The first row pieces are already loading while PRE runs (x does not depend on
// the routing).  All CTAs must be co-resident (grid <= SMs x occupancy).
constexpr int kFdWarps = 12;
constexpr int kFdBuf = 8192;            // bytes per row piece buffer (two per warp)
constexpr int kFdEntCap = 1024;         // (token, slot) entries per CTA
constexpr int kFdDoneSlot = 1023;
constexpr int kFdMaxNb = 4;             // most row-piece buffers per warp
constexpr int kFdReadyBase = 1024;      // gflags[1024 + c]: CTA c's destination rows are in dest_row
constexpr int kFdTicket = 2048;         // gflags[2048]: next (token, piece) ticket of the launch
constexpr int kFdRedBase = 2064;        // gflags[2064 + q]: column reducer q published
constexpr int kFdFlagWords = 2368;
constexpr int64_t kFdHistInts = 1023LL * 1024;  // chunk_hist [G][Ep]; then the prefixes, then the totals       // gflags[1023]: CTAs done scattering (grid <= 1023)

struct FusedDispatch {
  const uint4* x;
  const float* logits;                  // nullptr: routing given in idx
  int64_t tokens, vec_per_row, max_recv;
  int k, E, world, rank, tpc, mode;     // mode: bit 0 PRE, bit 1 MAIN
  int32_t* idx;
  float* w;
  int32_t* sorted_pos;
  int32_t* dest_row;
  int32_t* ebase;                       // [E] expert bases of the send order
  int32_t* seg_base;                    // [E]
  int32_t* counts_out;                  // [world][E]
  int64_t* recv_rows;
  int32_t* mat;                         // this rank's [world][E] count matrix
  PeerPtrs mats, recv;
  PeerSig count_flags, deliver_flags;
  const uint64_t* own_count_flags;      // [world] on this rank
  unsigned long long epoch;             // MoE call epoch
  int32_t* chunk_hist;                  // [grid][E]
  unsigned long long* gflags;           // [grid] barrier flags, then the done counter
  unsigned long long gepoch;
  unsigned long long* err;
  unsigned long long timeout_ns;
  int dbg;                              // timing experiments only (TF_MOE_FD_DEBUG): 1 no scatter, 2 no grid wait
  int nb;                               // row piece buffers per warp (2..4), sharing the warp's 2 * kFdBuf bytes
  int dyn;                              // 1: pieces handed out by a grid-wide ticket counter (PRE+MAIN launches)
  int reduce;                           // 1: column-reducer CTAs publish the chunk prefixes (else every CTA sums)
  int lhist;                            // 1: every CTA counts every entry of p.idx (no histogram exchange)
};

__device__ __forceinline__ uint64_t ld_acquire_gpu(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// chunk histograms are stored with the expert stride rounded up to 4 (16-byte rows)
__host__ __device__ __forceinline__ int fd_stride(int E) { return (E + 3) & ~3; }

// wc [nw][E] and the cross-chunk partial sums [2][4 * blockDim] share one region
__host__ __device__ __forceinline__ int fd_wc_ints(int E) {
  return kFdWarps * E > 8 * 32 * kFdWarps ? kFdWarps * E : 8 * 32 * kFdWarps;
}

size_t fused_dispatch_smem(int E) {
  return static_cast<size_t>(2) * kFdWarps * kFdBuf +
         (static_cast<size_t>(fd_wc_ints(E)) + 4 * static_cast<size_t>(E) + 2 * kFdEntCap) * 4;
}

template <int VPL>  // VPL 0: routing given
__global__ void __launch_bounds__(32 * kFdWarps, 1) dispatch_fused_kernel(const FusedDispatch p) {
  extern __shared__ __align__(128) uint8_t fsm_raw[];
  __shared__ uint64_t bars[kFdMaxNb * kFdWarps];  // [warp][buffer]: row piece landed
  __shared__ uint64_t rbars[kFdWarps];            // [warp]: logits rows landed (routing)
  __shared__ uint4* sdst[kFdWarps][16];
  __shared__ int32_t last_tot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nw = kFdWarps;
  const int E = p.E, k = p.k, G = gridDim.x, c = blockIdx.x;
  uint8_t* bufs = fsm_raw;                                     // [nw][2 * kFdBuf]
  int32_t* wc = reinterpret_cast<int32_t*>(fsm_raw + 2 * nw * kFdBuf);  // [nw][E]
  int32_t* cnt = wc + fd_wc_ints(E);                           // [E]
  int32_t* tot = cnt + E;                                      // [E]
  int32_t* off = tot + E;                                      // [E]
  int32_t* seg = off + E;                                      // [E]
  int32_t* idx_s = seg + E;                                    // [kFdEntCap]
  int32_t* pos_s = idx_s + kFdEntCap;                          // [kFdEntCap] rank inside the expert's send segment
  int32_t* part = wc;                                          // [2][4 * blockDim] cross-chunk partial sums (after wc)
  const int Ep = fd_stride(E);
  const int64_t t0 = static_cast<int64_t>(c) * p.tpc;
  const int64_t t_end = t0 + p.tpc < p.tokens ? t0 + p.tpc : p.tokens;
  const int nt = t_end > t0 ? static_cast<int>(t_end - t0) : 0;
  const int ent = nt * k;
  const int epr = E / p.world;
  // the warp's 2 * kFdBuf bytes hold NB row-piece buffers; rows split into equal
  // 16-byte-multiple pieces that fit one buffer
  // dynamic pieces: every launch that runs PRE and MAIN (gepoch is fresh) and scatters
  const bool dyn = p.dyn && (p.mode & 3) == 3 && !(p.dbg & 1);
  const int NB = dyn ? 2 : p.nb < 2 ? 2 : p.nb > kFdMaxNb ? kFdMaxNb : p.nb;
  const uint32_t buf_bytes = (2u * kFdBuf / NB) & ~15u;
  const int64_t npieces = (p.vec_per_row + buf_bytes / 16 - 1) / (buf_bytes / 16);
  const int64_t kPiece = (p.vec_per_row + npieces - 1) / npieces;  // vectors per piece
  const int ntasks = (p.dbg & 1) ? 0 : static_cast<int>(nt * npieces);
  uint8_t* wbuf = bufs + static_cast<size_t>(warp) * 2 * kFdBuf;
  // TF_MOE_FD_DEBUG bit 3: every CTA prints its SM, phase clocks and %globaltimer at
  // start / histogram published / counts released / exit (tools/moe_stamps.py)
  const uint64_t g_start = (p.dbg & 8) ? globaltimer_ns() : 0;
  uint64_t g_arrive = 0, g_release = 0;
  const long long stamp_all0 = clock64();
  long long stamp_all_mid = 0;
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bars[kFdMaxNb * warp + b], 1);
    mbar_init(&rbars[warp], 1);
    fence_barrier_init();
  }
  __syncwarp();
  auto piece_bytes = [&](int64_t ti) {
    const int64_t v0 = (ti % npieces) * kPiece;
    return static_cast<uint32_t>((min(v0 + kPiece, p.vec_per_row) - v0) * 16);
  };
  const int64_t dyn_total = p.tokens * npieces;  // tickets of the launch (dyn)
  auto issue_load = [&](int64_t ti, int b) {  // lane 0 only; ti: CTA-local task, or a global ticket (dyn)
    const int64_t t = (dyn ? 0 : t0) + ti / npieces, v0 = (ti % npieces) * kPiece;
    const uint32_t bytes = piece_bytes(ti);
    mbar_arrive_expect_tx(&bars[kFdMaxNb * warp + b], bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(wbuf + b * buf_bytes)),
        "l"(p.x + t * p.vec_per_row + v0), "r"(bytes), "r"(smem_u32(&bars[kFdMaxNb * warp + b]))
        : "memory");
  };
  // buffer 0 (the first buffer_bytes <= kFdBuf of the warp's region) loads under PRE;
  // the routing below stages logits in the region's second half
  int64_t cur = 0;  // dyn: this warp's current ticket (drawn before PRE, its row loads under PRE)
  if (dyn) {
    if (lane == 0) {
      cur = static_cast<int64_t>(atomicAdd(p.gflags + kFdTicket, 1ull));
      if (cur < dyn_total) issue_load(cur, 0);
      // every warp draws exactly one ticket past the end; the last such draw resets the
      // counter for the next launch (stream-ordered after this one)
      else if (cur == dyn_total + static_cast<int64_t>(G) * nw - 1) p.gflags[kFdTicket] = 0;
    }
    cur = __shfl_sync(0xffffffffu, cur, 0);
  } else if ((p.mode & 2) && lane == 0 && warp < ntasks) {
    issue_load(warp, 0);
  }

  if (p.mode & 1) {
    // ---- routing of this CTA's tokens
    if constexpr (VPL > 0) {
      // this warp's tokens tt = warp + j*nw: their logits rows come in with one bulk
      // copy each (one DRAM latency per round, not per token) into the warp's second
      // row buffer, which the scatter does not use before its second task
      const uint32_t rb = static_cast<uint32_t>(E) * 4;
      const bool bulk = (rb % 16) == 0 && (reinterpret_cast<uintptr_t>(p.logits) % 16) == 0;
      const int per_round = bulk ? static_cast<int>(kFdBuf / rb) : 1;
      const float* lbuf = reinterpret_cast<const float*>(wbuf + kFdBuf);
      uint32_t rph = 0;
      for (int j0 = 0; warp + j0 * nw < nt; j0 += per_round) {
        const int nr = min(per_round, (nt - warp + nw - 1) / nw - j0);
        if (bulk) {
          if (lane == 0) {
            mbar_arrive_expect_tx(&rbars[warp], rb * nr);
            for (int j = 0; j < nr; ++j)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      smem_u32(lbuf) + j * rb),
                  "l"(p.logits + (t0 + warp + (j0 + j) * nw) * E), "r"(rb), "r"(smem_u32(&rbars[warp]))
                  : "memory");
          }
          mbar_wait(&rbars[warp], rph);
          rph ^= 1;
        }
        for (int j = 0; j < nr; ++j) {
          const int tt = warp + (j0 + j) * nw;
          int my_idx;
          float my_w;
          topk_warp<VPL>(bulk ? lbuf + j * E : p.logits + (t0 + tt) * E, E, k, lane, my_idx, my_w);
          if (lane < k) {
            idx_s[tt * k + lane] = my_idx;
            p.idx[(t0 + tt) * k + lane] = my_idx;
            p.w[(t0 + tt) * k + lane] = my_w;
          }
        }
        __syncwarp();
      }
    } else {
      for (int i = tid; i < ent; i += blockDim.x) idx_s[i] = p.idx[t0 * k + i];
    }
    for (int x = tid; x < E; x += blockDim.x) cnt[x] = 0;
    // ---- stable ranks: entries in token order, blockDim at a time
    for (int base = 0; base < ent; base += blockDim.x) {
      for (int i = tid; i < nw * E; i += blockDim.x) wc[i] = 0;
      __syncthreads();
      const int i = base + tid;
      int e = i < ent ? idx_s[i] : -1;
      if (e >= E || e < -1) {
        if (p.err) atomicCAS(p.err, 0ull, 0x5300000ull | static_cast<unsigned>(i & 0xFFFFF));
        e = -1;
      }
      const unsigned same = __match_any_sync(0xffffffffu, e);
      const int in_warp = __popc(same & ((1u << lane) - 1));
      if (e >= 0 && in_warp == 0) wc[warp * E + e] = __popc(same);
      __syncthreads();
      for (int x = tid; x < E; x += blockDim.x) {
        int32_t run = cnt[x];
#pragma unroll
        for (int ww = 0; ww < nw; ++ww) {
          const int32_t v = wc[ww * E + x];
          wc[ww * E + x] = run;
          run += v;
        }
        cnt[x] = run;
      }
      __syncthreads();
      if (i < ent) pos_s[i] = e >= 0 ? wc[warp * E + e] + in_warp : -1;
      __syncthreads();
    }
    __syncthreads();
    auto wait_flags = [&](const unsigned long long* f, int n, unsigned long long code) {
      for (int x = tid; x < n; x += blockDim.x) {
        if (ld_acquire_gpu(f + x) >= p.gepoch) continue;
        const uint64_t ts = globaltimer_ns();
        while (ld_acquire_gpu(f + x) < p.gepoch) {
          if (globaltimer_ns() - ts > p.timeout_ns) {
            if (p.err) atomicCAS(p.err, 0ull, code | static_cast<unsigned>(x));
            break;
          }
        }
      }
    };
    if (p.lhist) {
      // ---- every CTA counts every entry itself (the routing is in p.idx: the input, or
      // published by each CTA's routing behind its arrival flag): totals, and the
      // entries of the chunks below this one -- no histogram exchange
      if (VPL > 0) {
        if (tid == 0) {
          if (p.dbg & 8) g_arrive = globaltimer_ns();
          __threadfence();
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.gflags + c), "l"(p.gepoch) : "memory");
        }
        if (!(p.dbg & 2)) wait_flags(p.gflags, G, 0x5400000ull);
        __syncthreads();
      }
      int32_t* hrest = wc;  // entries of this and higher chunks
      int32_t* hbelow = wc + E;
      for (int x = tid; x < 2 * E; x += blockDim.x) wc[x] = 0;
      __syncthreads();
      const int64_t nent = p.tokens * k, below_end = t0 * k;
      auto count = [&](int e, int64_t i) {  // one shared-memory atomic per entry
        if (e >= 0 && e < E) atomicAdd(i < below_end ? &hbelow[e] : &hrest[e], 1);
      };
      if ((reinterpret_cast<uintptr_t>(p.idx) & 15) == 0) {
        const int4* idx4 = reinterpret_cast<const int4*>(p.idx);
        // every CTA reads the same 16-byte vectors: start each CTA at its own slice so
        // the 148 readers of a line are spread in time (no L2 hot spot)
        const int64_t n4 = nent / 4, rot = n4 * c / G;
        constexpr int kBatch = 8;  // independent 16-byte loads in flight per thread before counting
        for (int64_t base = tid; base < n4; base += kBatch * blockDim.x) {
          int4 v[kBatch];
          int64_t q[kBatch];
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            const int64_t qq = base + static_cast<int64_t>(u) * blockDim.x;
            q[u] = qq + rot < n4 ? qq + rot : qq + rot - n4;
            v[u] = qq < n4 ? __ldcg(idx4 + q[u]) : make_int4(-1, -1, -1, -1);
          }
#pragma unroll
          for (int u = 0; u < kBatch; ++u) {
            count(v[u].x, 4 * q[u]);
            count(v[u].y, 4 * q[u] + 1);
            count(v[u].z, 4 * q[u] + 2);
            count(v[u].w, 4 * q[u] + 3);
          }
        }
        for (int64_t i = (nent / 4) * 4 + tid; i < nent; i += blockDim.x) count(__ldcg(p.idx + i), i);
      } else {
        for (int64_t i = tid; i < nent; i += blockDim.x) count(__ldcg(p.idx + i), i);
      }
      __syncthreads();
      if ((p.dbg & 8) && tid == 0) g_release = globaltimer_ns();
      for (int x = tid; x < E; x += blockDim.x) {
        const int32_t t = hrest[x] + hbelow[x];
        tot[x] = t;
        off[x] = hbelow[x];
        cnt[x] = t;  // this rank's count row (tot becomes the expert bases below)
      }
    } else {
    // ---- publish the chunk histogram
    for (int x = tid; x < Ep; x += blockDim.x) p.chunk_hist[static_cast<int64_t>(c) * Ep + x] = x < E ? cnt[x] : 0;
    __syncthreads();
    if (tid == 0) {
      if (p.dbg & 8) g_arrive = globaltimer_ns();
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.gflags + c), "l"(p.gepoch) : "memory");
    }
    const int Q = Ep / 4;
    if (p.reduce && G <= static_cast<int>(blockDim.x) && Q <= G && !(p.dbg & 2)) {
      // ---- column reducers: CTA q < Q owns experts [4q, 4q + 4): waits for every chunk,
      // scans its column over the chunks (one int4 per thread) and publishes every
      // chunk's exclusive prefix and the totals; the other CTAs read one prefix row.
      int32_t* pfx = p.chunk_hist + kFdHistInts;  // [G][Ep]
      int32_t* totg = pfx + kFdHistInts;          // [Ep]
      if (c < Q) {
        __shared__ int4 wsum[kFdWarps];
        wait_flags(p.gflags, G, 0x5400000ull);
        __syncthreads();
        const int4 v = tid < G ? __ldcg(reinterpret_cast<const int4*>(p.chunk_hist) + static_cast<int64_t>(tid) * Q + c)
                               : make_int4(0, 0, 0, 0);
        int4 inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int ax = __shfl_up_sync(0xffffffffu, inc.x, o), ay = __shfl_up_sync(0xffffffffu, inc.y, o);
          const int az = __shfl_up_sync(0xffffffffu, inc.z, o), aw = __shfl_up_sync(0xffffffffu, inc.w, o);
          if (lane >= o) { inc.x += ax; inc.y += ay; inc.z += az; inc.w += aw; }
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        int4 below = make_int4(0, 0, 0, 0);
        for (int ww = 0; ww < warp; ++ww) {
          const int4 u = wsum[ww];
          below.x += u.x; below.y += u.y; below.z += u.z; below.w += u.w;
        }
        if (tid < G) {
          const int4 ex = make_int4(below.x + inc.x - v.x, below.y + inc.y - v.y, below.z + inc.z - v.z,
                                    below.w + inc.w - v.w);
          reinterpret_cast<int4*>(pfx)[static_cast<int64_t>(tid) * Q + c] = ex;
          if (tid == G - 1)
            reinterpret_cast<int4*>(totg)[c] = make_int4(ex.x + v.x, ex.y + v.y, ex.z + v.z, ex.w + v.w);
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.gflags + kFdRedBase + c), "l"(p.gepoch)
                       : "memory");
        }
      }
      wait_flags(p.gflags + kFdRedBase, Q, 0x5600000ull);
      __syncthreads();
      if ((p.dbg & 8) && tid == 0) g_release = globaltimer_ns();
      for (int x = tid; x < E; x += blockDim.x) {
        const int32_t t = __ldcg(totg + x);
        off[x] = __ldcg(pfx + static_cast<int64_t>(c) * Ep + x);
        tot[x] = t;
        cnt[x] = t;  // this rank's count row (tot becomes the expert bases below)
      }
    } else {
    // ---- every CTA waits for every chunk and sums the columns itself
    if (!(p.dbg & 2)) wait_flags(p.gflags, G, 0x5400000ull);
    __syncthreads();
    if ((p.dbg & 8) && tid == 0) g_release = globaltimer_ns();
    // ---- totals and this chunk's offsets: thread = (4-expert quad, chunk group), one
    // 16-byte load per chunk, all chunk groups' loads independent
    {
      const int quads = Ep / 4;
      const int groups = max(1, static_cast<int>(blockDim.x) / quads);
      int4* part_t = reinterpret_cast<int4*>(part);
      int4* part_o = reinterpret_cast<int4*>(part + 4 * blockDim.x);
      for (int i = tid; i < quads * groups; i += blockDim.x) {
        const int q = i % quads, g = i / quads;
        int4 t = make_int4(0, 0, 0, 0), o = make_int4(0, 0, 0, 0);
        const int4* col = reinterpret_cast<const int4*>(p.chunk_hist) + q;
#pragma unroll 16
        for (int c0 = g; c0 < G; c0 += groups) {
          const int cc = c0 + c < G ? c0 + c : c0 + c - G;  // rotated start: spread the readers of a row
          const int4 v = __ldcg(col + static_cast<int64_t>(cc) * quads);
          t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
          if (cc < c) { o.x += v.x; o.y += v.y; o.z += v.z; o.w += v.w; }
        }
        part_t[g * quads + q] = t;
        part_o[g * quads + q] = o;
      }
      __syncthreads();
      for (int x = tid; x < E; x += blockDim.x) {
        int32_t t = 0, o = 0;
        for (int g = 0; g < groups; ++g) {
          t += part[4 * (g * quads) + x];
          o += part[4 * blockDim.x + 4 * (g * quads) + x];
        }
        tot[x] = t;
        off[x] = o;
        cnt[x] = t;  // this rank's count row (tot becomes the expert bases below)
      }
    }
    }
    }  // histogram exchange
    __syncthreads();
    block_exclusive_scan(tot, E);  // ends with __syncthreads
    if (c == 0)
      for (int x = tid; x < E; x += blockDim.x) {
        p.ebase[x] = tot[x];
        p.mat[static_cast<int64_t>(p.rank) * E + x] = cnt[x];
      }
    for (int i = tid; i < ent; i += blockDim.x) {
      if (pos_s[i] < 0) continue;
      const int e = idx_s[i];
      pos_s[i] += off[e];
      p.sorted_pos[t0 * k + i] = tot[e] + pos_s[i];
    }
    if (c == 0 && p.world > 1) {  // count row -> every peer's matrix, then its flag
      for (int q = 0; q < p.world; ++q) {
        int32_t* dst = static_cast<int32_t*>(p.mats.p[q]) + static_cast<int64_t>(p.rank) * E;
        for (int x = tid; x < E; x += blockDim.x) dst[x] = cnt[x];
      }
      __syncthreads();
      if (tid < p.world) {
        fence_sys();
        st_release_sys(p.count_flags.p[tid] + p.rank, p.epoch);
      }
    }
    __syncthreads();
  } else {
    // MAIN only: the PRE launch left idx / sorted_pos / ebase in global memory
    for (int x = tid; x < E; x += blockDim.x) tot[x] = __ldcg(p.ebase + x);
    __syncthreads();
    for (int i = tid; i < ent; i += blockDim.x) {
      const int e = __ldcg(p.idx + t0 * k + i);
      idx_s[i] = e;
      pos_s[i] = (e >= 0 && e < E) ? __ldcg(p.sorted_pos + t0 * k + i) - tot[e] : -1;
    }
    __syncthreads();
  }
  if (!(p.mode & 2)) return;

  // ---- destination segment bases (layout_kernel's arithmetic)
  if (p.world > 1) {
    if (tid < p.world)
      wait_geq_sys(p.own_count_flags + tid, p.epoch, p.timeout_ns, p.err, 0x5000000ull | tid);
    __syncthreads();
  }
  for (int x = tid; x < E; x += blockDim.x) {
    int32_t t = 0, below = 0;
    for (int s = 0; s < p.world; ++s) {
      // own row: from smem when PRE ran in this launch (CTA 0 may not have stored it yet)
      const int32_t v = (s == p.rank && (p.mode & 1)) ? cnt[x] : __ldcg(p.mat + s * E + x);
      t += v;
      below += s < p.rank ? v : 0;
    }
    seg[x] = t;
    off[x] = below;  // rows of lower source ranks for the same expert
  }
  __syncthreads();
  if (tid == 0) last_tot = seg[(p.rank + 1) * epr - 1];
  block_exclusive_scan(seg, E);
  for (int x = tid; x < E; x += blockDim.x) {
    const int owner_first = (x / epr) * epr;
    off[x] += seg[x] - seg[owner_first];
  }
  __syncthreads();
  if (c == 0) {
    if (tid == 0)
      *p.recv_rows = static_cast<int64_t>(seg[(p.rank + 1) * epr - 1]) + last_tot - seg[p.rank * epr];
    for (int x = tid; x < E; x += blockDim.x) p.seg_base[x] = off[x];
    for (int i = tid; i < p.world * E; i += blockDim.x)
      p.counts_out[i] = (i / E == p.rank && (p.mode & 1)) ? cnt[i % E] : __ldcg(p.mat + i);
  }

  stamp_all_mid = clock64();
  if (dyn) {
    // ---- dynamic scatter: publish this CTA's destination rows, then every warp takes
    // (token, piece) tickets from the grid-wide counter until they run out, so SMs that
    // drain their stores faster take more pieces.  A ticket's row load only needs the
    // token; its stores wait for the owner CTA's "rows published" flag.
    for (int i = tid; i < ent; i += blockDim.x)
      if (pos_s[i] >= 0) p.dest_row[t0 * k + i] = off[idx_s[i]] + pos_s[i];
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.gflags + kFdReadyBase + c), "l"(p.gepoch) : "memory");
    }
    uint32_t phases = 0;
    const int64_t vpr = p.vec_per_row;
    int b = 0;
    while (cur < dyn_total) {
      int64_t nxt = 0;
      if (lane == 0) {
        nxt = static_cast<int64_t>(atomicAdd(p.gflags + kFdTicket, 1ull));
        if (nxt == dyn_total + static_cast<int64_t>(G) * nw - 1) p.gflags[kFdTicket] = 0;  // last draw of the launch
      }
      nxt = __shfl_sync(0xffffffffu, nxt, 0);
      const int64_t t = cur / npieces;
      const int64_t v0 = (cur % npieces) * kPiece;
      const uint32_t bytes = piece_bytes(cur);
      uint4* my_dst = nullptr;
      int my_remote = 0;
      if (lane < k) {
        const unsigned long long* rf = p.gflags + kFdReadyBase + t / p.tpc;
        if (ld_acquire_gpu(rf) < p.gepoch) {
          const uint64_t ts = globaltimer_ns();
          while (ld_acquire_gpu(rf) < p.gepoch)
            if (globaltimer_ns() - ts > p.timeout_ns) {
              if (p.err) atomicCAS(p.err, 0ull, 0x5500000ull | static_cast<unsigned>(t / p.tpc));
              break;
            }
        }
        const int e = __ldcg(p.idx + t * k + lane);
        if (e >= 0 && e < E) {
          const int64_t row = __ldcg(p.dest_row + t * k + lane);
          if (row < p.max_recv) my_dst = static_cast<uint4*>(p.recv.p[e / epr]) + row * vpr + v0;
          else if (p.err) atomicCAS(p.err, 0ull, 0x5000000ull | 0xFFFFFFull);
          my_remote = (e / epr) != p.rank;
        }
      }
      if (lane < k) sdst[warp][lane] = my_dst;
      __syncwarp();
      const unsigned remote = __ballot_sync(0xffffffffu, my_remote != 0 && my_dst != nullptr);
      mbar_wait(&bars[kFdMaxNb * warp + b], (phases >> b) & 1);
      phases ^= 1u << b;
      uint8_t* buf = wbuf + b * buf_bytes;
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // buffer b ^ 1 free
        if (nxt < dyn_total) issue_load(nxt, b ^ 1);
        for (int j = 0; j < k; ++j)
          if (sdst[warp][j] != nullptr && !((remote >> j) & 1))
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst[warp][j]),
                         "r"(smem_u32(buf)), "r"(bytes)
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      for (int j = 0; j < k; ++j) {
        if (!((remote >> j) & 1)) continue;
        uint4* d = sdst[warp][j];
        const uint4* sb = reinterpret_cast<const uint4*>(buf);
        for (int v = lane; v < static_cast<int>(bytes / 16); v += 32) d[v] = sb[v];
      }
      __syncwarp();
      cur = nxt;
      b ^= 1;
    }
  } else {
  // ---- scatter this CTA's tokens: task j of this warp is piece (warp + j * nw),
  // buffer j % NB; the load of task j + NB - 1 goes out once task j - 1's stores
  // have read their buffer, so NB - 1 loads are in flight under the stores
  if (lane == 0)
    for (int b = 1; b < NB - 1; ++b)
      if (warp + b * nw < ntasks) issue_load(warp + b * nw, b);
  uint32_t phases = 0;
  const int64_t vpr = p.vec_per_row;
  int b = 0;
  for (int ti = warp; ti < ntasks; ti += nw, b = (b + 1 == NB) ? 0 : b + 1) {
    const int tt = static_cast<int>(ti / npieces);
    const int64_t v0 = (ti % npieces) * kPiece;
    const uint32_t bytes = piece_bytes(ti);
    uint4* my_dst = nullptr;
    int my_remote = 0;
    if (lane < k) {
      const int slot = tt * k + lane;
      const int e = idx_s[slot];
      if (pos_s[slot] >= 0) {
        const int64_t row = static_cast<int64_t>(off[e]) + pos_s[slot];
        if (v0 == 0) p.dest_row[t0 * k + slot] = static_cast<int32_t>(row);
        if (row < p.max_recv) my_dst = static_cast<uint4*>(p.recv.p[e / epr]) + row * vpr + v0;
        else if (p.err) atomicCAS(p.err, 0ull, 0x5000000ull | 0xFFFFFFull);
        my_remote = (e / epr) != p.rank;
      }
    }
    if (lane < k) sdst[warp][lane] = my_dst;
    __syncwarp();
    const unsigned remote = __ballot_sync(0xffffffffu, my_remote != 0 && my_dst != nullptr);
    mbar_wait(&bars[kFdMaxNb * warp + b], (phases >> b) & 1);
    phases ^= 1u << b;
    uint8_t* buf = wbuf + b * buf_bytes;
    if (lane == 0) {
      for (int j = 0; j < k; ++j)
        if (sdst[warp][j] != nullptr && !((remote >> j) & 1))
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(sdst[warp][j]),
                       "r"(smem_u32(buf)), "r"(bytes)
                       : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    for (int j = 0; j < k; ++j) {
      if (!((remote >> j) & 1)) continue;
      uint4* d = sdst[warp][j];
      const uint4* sb = reinterpret_cast<const uint4*>(buf);
      for (int v = lane; v < static_cast<int>(bytes / 16); v += 32) d[v] = sb[v];
    }
    __syncwarp();  // the lanes' remote stores have read the buffer
    if (lane == 0 && ti + (NB - 1) * nw < ntasks) {
      // refill buffer (b + NB - 1) % NB, last used by the previous task: its stores
      // are the second most recent bulk group
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue_load(ti + (NB - 1) * nw, b == 0 ? NB - 1 : b - 1);
    }
  }
  }  // static scatter
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores performed
  if ((p.dbg & 8) && tid == 0)
    printf("fdsm cta %d sm %u pre_layout %lld scatter %lld clk t %llu %llu %llu %llu\n", c, smid_u32(),
           stamp_all_mid - stamp_all0, clock64() - stamp_all_mid, static_cast<unsigned long long>(g_start),
           static_cast<unsigned long long>(g_arrive), static_cast<unsigned long long>(g_release),
           static_cast<unsigned long long>(globaltimer_ns()));
  if (p.world > 1) {
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_global();
      fence_sys();
      unsigned long long* done = p.gflags + kFdDoneSlot;
      const unsigned long long old = atomicAdd(done, 1ull);
      if (old == static_cast<unsigned long long>(G - 1)) {  // last CTA: every row of this rank landed
        fence_sys();
        *done = 0;  // the next launch on this device is stream-ordered after this one
        for (int q = 0; q < p.world; ++q) st_release_sys(p.deliver_flags.p[q] + p.rank, p.epoch);
      }
    }
  }
}

// warp per token; hidden in 256-element chunks (8 bf16 = 16 bytes per lane)
__global__ void __launch_bounds__(256) combine_kernel(
    int64_t tokens, int64_t vec_per_row, int k, int E, int world,
    const int32_t* __restrict__ idx, const float* __restrict__ w,
    const int32_t* __restrict__ dest_row, PeerPtrs yout, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int epr = E / world;
  for (int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < tokens;
       t += nwarps) {
    const uint4* rows[16];
    float wt[16];
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      rows[j] = static_cast<const uint4*>(yout.p[e / epr]) +
                static_cast<int64_t>(dest_row[t * k + j]) * vec_per_row;
      wt[j] = w[t * k + j];
    }
    for (int64_t v = lane; v < vec_per_row; v += 32) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint4 val[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < k) val[j] = rows[j][v];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < k) {
          const uint32_t u[4] = {val[j].x, val[j].y, val[j].z, val[j].w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[2 * q] = fmaf(wt[j], __uint_as_float(u[q] << 16), acc[2 * q]);
            acc[2 * q + 1] = fmaf(wt[j], __uint_as_float(u[q] & 0xFFFF0000u), acc[2 * q + 1]);
          }
        }
      }
      out[t * vec_per_row + v] =
          make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                     pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
    }
  }
}

// k <= 8: U hidden vectors per lane per iteration, so a warp keeps U*k 16-byte
// loads in flight (read-once rows: no L1 allocation).
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <int U>
__global__ void __launch_bounds__(256) combine8_kernel(
    int64_t tokens, int64_t vec_per_row, int k, int E, int world,
    const int32_t* __restrict__ idx, const float* __restrict__ w,
    const int32_t* __restrict__ dest_row, PeerPtrs yout, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int epr = E / world;
  for (int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < tokens;
       t += nwarps) {
    // lane j < k resolves slot j, then the warp shares it
    const uint4* my_row = nullptr;
    float my_w = 0.f;
    if (lane < k) {
      const int e = idx[t * k + lane];
      my_row = static_cast<const uint4*>(yout.p[e / epr]) +
               static_cast<int64_t>(dest_row[t * k + lane]) * vec_per_row;
      my_w = w[t * k + lane];
    }
    const uint4* rows[8];
    float wt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      rows[j] = reinterpret_cast<const uint4*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(my_row), j));
      wt[j] = __shfl_sync(0xffffffffu, my_w, j);
    }
    for (int64_t v0 = lane; v0 < vec_per_row; v0 += 32 * U) {
      uint4 val[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j < k && v0 + 32 * u < vec_per_row) val[u][j] = ld_stream(rows[j] + v0 + 32 * u);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (v0 + 32 * u >= vec_per_row) break;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < k) {
            const uint32_t q4[4] = {val[u][j].x, val[u][j].y, val[u][j].z, val[u][j].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[2 * q] = fmaf(wt[j], __uint_as_float(q4[q] << 16), acc[2 * q]);
              acc[2 * q + 1] = fmaf(wt[j], __uint_as_float(q4[q] & 0xFFFF0000u), acc[2 * q + 1]);
            }
          }
        }
        out[t * vec_per_row + v0 + 32 * u] =
            make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                       pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
      }
    }
  }
}

int64_t count_scratch_bytes(int64_t entries, int E) {
  const int64_t nchunks = (entries + kChunk - 1) / kChunk;
  return (std::max<int64_t>(nchunks, 1) * E + E) * 4 + 256;
}

// counts[e], ebase[e] (exclusive scan of counts) and the stable send positions
int run_count(const int32_t* idx, int64_t entries, int E, int32_t* counts, int32_t* sorted_pos,
              void* scratch, int32_t* ebase, cudaStream_t s) {
  const int nchunks = static_cast<int>(std::max<int64_t>((entries + kChunk - 1) / kChunk, 1));
  int32_t* chunk = static_cast<int32_t*>(scratch);
  if (!ebase) ebase = chunk + static_cast<int64_t>(nchunks) * E;
  if (static_cast<size_t>(32) * E * 4 > 227 * 1024) return fail(TF_ERR_CONFIG, "too many experts");
  {
    // single-pass path when every chunk CTA can be co-resident
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t fsm = (static_cast<size_t>(34) * E + 2 * static_cast<size_t>(std::max(1, kChunk / E)) * E) * 4;
    static std::map<int, unsigned long long*> flag_bufs;
    static std::map<int, unsigned long long> epochs;
    static std::mutex mu;
    if (entries > 0 && nchunks <= num_sms_of_current_device() && fsm <= 200 * 1024) {
      unsigned long long* flags = nullptr;
      unsigned long long ep = 0;
      {
        std::lock_guard<std::mutex> lk(mu);
        auto it = flag_bufs.find(dev);
        if (it == flag_bufs.end()) {
          TF_CUDA_TRY(cudaMalloc(&flags, 1024 * sizeof(unsigned long long)));
          TF_CUDA_TRY(cudaMemset(flags, 0, 1024 * sizeof(unsigned long long)));
          flag_bufs[dev] = flags;
          TF_CUDA_TRY(cudaFuncSetAttribute(count_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           200 * 1024));
        } else {
          flags = it->second;
        }
        ep = ++epochs[dev];
      }
      count_fused_kernel<<<nchunks, kChunk, fsm, s>>>(idx, entries, E, nchunks, chunk, flags, ep,
                                                      20ull * 1000 * 1000 * 1000, nullptr, counts, ebase,
                                                      sorted_pos);
      TF_CUDA_TRY(cudaGetLastError());
      return TF_OK;
    }
  }
  hist_kernel<<<nchunks, 256, E * 4, s>>>(idx, entries, E, chunk);
  scan_kernel<<<1, 1024, E * 4, s>>>(chunk, nchunks, E, counts, ebase);  // E <= 1024*4 ints
  if (entries > 0) {
    const size_t sm = static_cast<size_t>(32) * E * 4;
    static bool attr = false;
    if (!attr && sm > 48 * 1024) {
      TF_CUDA_TRY(cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       227 * 1024));
      attr = true;
    }
    rank_kernel<<<nchunks, kChunk, sm, s>>>(idx, entries, E, chunk, ebase, sorted_pos);
  }
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

// Per-PE workspace: count matrix [w][E] (peers write their rows), this PE's
// expert bases [E] and destination segment bases [E], receive buffer and
// expert-output buffer ([max_recv][H] bf16 each).
struct MoeWs {
  Workspace* ws;
  size_t mat_off, ebase_off, seg_off, recv_off, yout_off;
};

int moe_workspace(tf_team* t, const tf_moe_args* a, MoeWs* out) {
  const int w = t->world;
  const size_t mat = (static_cast<size_t>(w) * a->n_experts * 4 + 1023) / 1024 * 1024;
  const size_t vec = (static_cast<size_t>(a->n_experts) * 4 + 1023) / 1024 * 1024;
  const size_t buf = (static_cast<size_t>(a->max_recv) * a->hidden * 2 + 1023) / 1024 * 1024;
  const std::string key = "moe:" + std::to_string(a->n_experts) + "x" + std::to_string(a->hidden) +
                          "x" + std::to_string(a->max_recv);
  int rc = TF_OK;
  Workspace* ws = t->workspace(key, mat + 2 * vec + 2 * buf, 3 * static_cast<size_t>(w), &rc);
  if (!ws) return rc;
  out->ws = ws;
  out->mat_off = ws->data_off;
  out->ebase_off = ws->data_off + mat;
  out->seg_off = out->ebase_off + vec;
  out->recv_off = out->seg_off + vec;
  out->yout_off = out->recv_off + buf;
  return TF_OK;
}

int check_moe(tf_team* t, int rank, const tf_moe_args* a) {
  if (!t || !a) return fail(TF_ERR_INVALID, "NULL argument");
  if (rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  if (a->n_experts < 1 || a->n_experts % t->world)
    return fail(TF_ERR_INVALID, "n_experts must be >= 1 and divisible by world");
  if (a->k < 1 || a->k > 16 || a->k > a->n_experts) return fail(TF_ERR_INVALID, "need 1 <= k <= min(16, E)");
  if (a->hidden < 8 || a->hidden % 8) return fail(TF_ERR_INVALID, "hidden must be a positive multiple of 8");
  if (a->tokens < 0 || a->max_recv < 0) return fail(TF_ERR_INVALID, "negative size");
  return TF_OK;
}


// Fused dispatch launch (mode 1 PRE, 2 MAIN, 3 both).  Returns TF_ERR_CONFIG (no
// launch) when the shape does not fit the fused kernel; the caller then runs the
// multi-kernel path.
int launch_fused_dispatch(FusedDispatch p, cudaStream_t s, bool* launched) {
  *launched = false;
  static const bool enabled = [] {
    const char* e = getenv("TF_MOE_FUSED");
    return !e || atoi(e) != 0;
  }();
  if (!enabled || p.E > 1024) return TF_OK;
  int dev = 0;
  TF_CUDA_TRY(cudaGetDevice(&dev));
  const size_t smem = fused_dispatch_smem(p.E);
  if (smem > 225 * 1024) return TF_OK;
  const int vpl = !p.logits ? 0 : p.E <= 64 ? 2 : p.E <= 256 ? 8 : 32;
  const void* fn = vpl == 0 ? reinterpret_cast<const void*>(dispatch_fused_kernel<0>)
                 : vpl == 2 ? reinterpret_cast<const void*>(dispatch_fused_kernel<2>)
                 : vpl == 8 ? reinterpret_cast<const void*>(dispatch_fused_kernel<8>)
                            : reinterpret_cast<const void*>(dispatch_fused_kernel<32>);
  static std::mutex mu;
  static std::map<int, unsigned long long*> flag_bufs;
  static std::map<int, unsigned long long> epochs;
  static std::map<std::pair<int, const void*>, int> occ;
  unsigned long long* flags = nullptr;
  unsigned long long ge = 0;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = flag_bufs.find(dev);
    if (it == flag_bufs.end()) {
      TF_CUDA_TRY(cudaMalloc(&flags, kFdFlagWords * sizeof(unsigned long long)));
      TF_CUDA_TRY(cudaMemset(flags, 0, kFdFlagWords * sizeof(unsigned long long)));
      flag_bufs[dev] = flags;
    } else {
      flags = it->second;
    }
    auto key = std::make_pair(dev, fn);
    auto oi = occ.find(key);
    if (oi == occ.end()) {
      cudaFuncAttributes fa{};
      TF_CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
      int optin = 0;
      TF_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      const int dyn_max = optin - static_cast<int>(fa.sharedSizeBytes);
      if (dyn_max < static_cast<int>(smem)) return TF_OK;  // multi-kernel path
      TF_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
      TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kFdWarps, smem));
      occ[key] = per_sm;
    } else {
      per_sm = oi->second;
    }
    if (p.mode & 1) ge = ++epochs[dev];
  }
  if (per_sm < 1) return TF_OK;
  const int64_t cap = std::min<int64_t>(static_cast<int64_t>(num_sms_of_current_device()) * per_sm, kFdDoneSlot);
  const int64_t T = p.tokens;
  int64_t G = std::max<int64_t>(1, std::min<int64_t>(cap, T));
  const int64_t tpc = T > 0 ? (T + G - 1) / G : 1;
  G = T > 0 ? (T + tpc - 1) / tpc : 1;
  if (tpc * p.k > kFdEntCap) return TF_OK;
  p.tpc = static_cast<int>(tpc);
  p.gflags = flags;
  p.gepoch = ge;
  // the chunk histogram scratch [G][E] (G <= 1023, E <= 1024): one 4 MB buffer per device
  void* hist = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    static std::map<int, void*> hist_bufs;
    auto it = hist_bufs.find(dev);
    if (it == hist_bufs.end()) {
      TF_CUDA_TRY(cudaMalloc(&hist, (2 * static_cast<size_t>(kFdHistInts) + 1024) * 4));
      hist_bufs[dev] = hist;
    } else {
      hist = it->second;
    }
  }
  p.chunk_hist = static_cast<int32_t*>(hist);
  static const int dbg = [] {
    const char* e = getenv("TF_MOE_FD_DEBUG");
    return e ? atoi(e) : 0;
  }();
  p.dbg = dbg;
  static const int nb = [] {
    const char* e = getenv("TF_MOE_FD_NB");
    return e ? atoi(e) : 2;
  }();
  p.nb = nb;
  static const int dyn = [] {
    const char* e = getenv("TF_MOE_FD_DYN");
    return e ? atoi(e) : 1;
  }();
  p.dyn = dyn;
  static const int reduce = [] {  // measured neutral (profiles/r02_moe_dispatch_s3.txt): opt-in
    const char* e = getenv("TF_MOE_FD_REDUCE");
    return e ? atoi(e) : 0;
  }();
  p.reduce = reduce;
  // local counting: measured 104.4 vs 109.5 us with the routing given, 117.8-118.8 vs
  // 115.6-116.7 us when the launch routes (profiles/r02_moe_dispatch_s3.txt), so by
  // default only for given routing (TF_MOE_FD_LHIST: 0 never, 1 given routing, 2 always)
  static const int lhist = [] {
    const char* e = getenv("TF_MOE_FD_LHIST");
    return e ? atoi(e) : 1;
  }();
  p.lhist = lhist == 2 || (lhist == 1 && !p.logits);
  void* args[] = {&p};
  TF_CUDA_TRY(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(G)), dim3(32 * kFdWarps), args, smem, s));
  *launched = true;
  return TF_OK;
}

int grid_for(int64_t warps) {
  int64_t blocks = (warps * 32 + 255) / 256;
  const int cap = num_sms_of_current_device() * 8;
  if (blocks > cap) blocks = cap;
  return static_cast<int>(std::max<int64_t>(blocks, 1));
}

}  // namespace
}  // namespace tf

using tf::fail;

extern "C" {

int tf_moe_topk(const float* logits, int64_t tokens, int n_experts, int k, int32_t* topk_idx,
                float* topk_w, void* stream) {
  if (n_experts < 1 || n_experts > 1024) return fail(TF_ERR_INVALID, "1 <= n_experts <= 1024");
  if (k < 1 || k > 16 || k > n_experts) return fail(TF_ERR_INVALID, "need 1 <= k <= min(16, E)");
  if (tokens <= 0) return TF_OK;
  const int64_t threads = tokens * 32;
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  auto s = static_cast<cudaStream_t>(stream);
  if (n_experts <= 64) tf::topk_kernel<2><<<grid, 256, 0, s>>>(logits, tokens, n_experts, k, topk_idx, topk_w);
  else if (n_experts <= 256) tf::topk_kernel<8><<<grid, 256, 0, s>>>(logits, tokens, n_experts, k, topk_idx, topk_w);
  else tf::topk_kernel<32><<<grid, 256, 0, s>>>(logits, tokens, n_experts, k, topk_idx, topk_w);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}

int64_t tf_moe_count_scratch_bytes(int64_t entries, int n_experts) {
  return tf::count_scratch_bytes(entries, n_experts);
}

int tf_moe_count(const int32_t* topk_idx, int64_t tokens, int k, int n_experts, int32_t* counts,
                 int32_t* sorted_pos, void* scratch, void* stream) {
  if (n_experts < 1) return fail(TF_ERR_INVALID, "n_experts must be >= 1");
  if (tokens < 0 || k < 1) return fail(TF_ERR_INVALID, "bad tokens/k");
  if (!scratch) return fail(TF_ERR_INVALID, "scratch is NULL");
  return tf::run_count(topk_idx, tokens * k, n_experts, counts, sorted_pos, scratch, nullptr,
                       static_cast<cudaStream_t>(stream));
}

int tf_moe_buffers(tf_team* t, int rank, const tf_moe_args* a, void** recv, void** expert_out) {
  int rc = tf::check_moe(t, rank, a);
  if (rc) return rc;
  tf::MoeWs m;
  rc = tf::moe_workspace(t, a, &m);
  if (rc) return rc;
  if (recv) *recv = t->pes[rank].base + m.recv_off;
  if (expert_out) *expert_out = t->pes[rank].base + m.yout_off;
  return TF_OK;
}

int tf_moe_dispatch(tf_team* t, int rank, const tf_moe_args* a, int phase, void* stream) {
  int rc = tf::check_moe(t, rank, a);
  if (rc) return rc;
  tf::MoeWs m;
  rc = tf::moe_workspace(t, a, &m);
  if (rc) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  const int w = t->world, E = a->n_experts;
  const int64_t entries = a->tokens * a->k;
  const size_t sig = m.ws->sig_base;  // [0,w) counts ready, [w,2w) delivered, [2w,3w) outputs ready
  const int dev = t->pes[rank].device;
  int32_t* ebase = reinterpret_cast<int32_t*>(t->pes[rank].base + m.ebase_off);
  int32_t* seg_base = reinterpret_cast<int32_t*>(t->pes[rank].base + m.seg_off);
  if (a->logits && (!a->topk_idx || !a->topk_w))
    return fail(TF_ERR_INVALID, "routing from logits needs topk_idx and topk_w outputs");
  const int fmode = ((phase & TF_PHASE_PRE) ? 1 : 0) | ((phase & TF_PHASE_MAIN) ? 2 : 0);
  bool fused = false;
  if (fmode) {
    // one launch per phase group (PRE+MAIN in one when the caller drives both)
    tf::FusedDispatch p{};
    p.x = static_cast<const uint4*>(a->x);
    p.logits = a->logits;
    p.tokens = a->tokens;
    p.vec_per_row = a->hidden / 8;
    p.max_recv = a->max_recv;
    p.k = a->k;
    p.E = E;
    p.world = w;
    p.rank = rank;
    p.mode = fmode;
    p.idx = const_cast<int32_t*>(a->topk_idx);
    p.w = const_cast<float*>(a->topk_w);
    p.sorted_pos = a->sorted_pos;
    p.dest_row = a->dest_row;
    p.ebase = ebase;
    p.seg_base = seg_base;
    p.counts_out = a->counts;
    p.recv_rows = a->recv_rows;
    p.mat = reinterpret_cast<int32_t*>(t->pes[rank].base + m.mat_off);
    for (int q = 0; q < w; ++q) {
      p.mats.p[q] = t->pes[q].base + m.mat_off;
      p.recv.p[q] = t->pes[q].base + m.recv_off;
      p.count_flags.p[q] = t->pes[q].sig + sig;
      p.deliver_flags.p[q] = t->pes[q].sig + sig + w;
    }
    p.own_count_flags = t->pes[rank].sig + sig;
    p.epoch = m.ws->epoch[rank] + ((fmode & 1) ? 1 : 0);
    p.err = t->err_word(rank);
    p.timeout_ns = t->timeout_ns;
    rc = tf::launch_fused_dispatch(p, s, &fused);
    if (rc) return rc;
    if (fused && (fmode & 1)) m.ws->epoch[rank] = p.epoch;
  }
  if ((phase & TF_PHASE_PRE) && !fused) {
    if (a->logits) {
      rc = tf_moe_topk(a->logits, a->tokens, E, a->k, const_cast<int32_t*>(a->topk_idx),
                       const_cast<float*>(a->topk_w), stream);
      if (rc) return rc;
    }
    const uint64_t e = ++m.ws->epoch[rank];
    // count into this rank's own row of its local matrix, then push the row to all peers
    int32_t* own_row = reinterpret_cast<int32_t*>(t->pes[rank].base + m.mat_off) +
                       static_cast<int64_t>(rank) * E;
    void* chunk = t->scratch(dev, tf::count_scratch_bytes(entries, E));
    if (!chunk) return fail(TF_ERR_ALLOC, "cannot allocate MoE count scratch");
    rc = tf::run_count(a->topk_idx, entries, E, own_row, a->sorted_pos, chunk, ebase, s);
    if (rc) return rc;
    tf::PeerPtrs mats{};
    tf::PeerSig flags{};
    for (int p = 0; p < w; ++p) {
      mats.p[p] = t->pes[p].base + m.mat_off;
      flags.p[p] = t->pes[p].sig + sig;
    }
    if (w > 1) tf::push_counts_kernel<<<1, 256, 0, s>>>(own_row, E, mats, flags, w, rank, e);
    TF_CUDA_TRY(cudaGetLastError());
  }
  if ((phase & TF_PHASE_MAIN) && !fused) {
    const uint64_t e = m.ws->epoch[rank];
    if (w > 1)
      tf::wait_flags_kernel<<<1, 32 * ((w + 31) / 32), 0, s>>>(t->pes[rank].sig + sig, w, e,
                                                               t->timeout_ns, t->err_word(rank),
                                                               0x5000000ull);
    const int32_t* mat = reinterpret_cast<const int32_t*>(t->pes[rank].base + m.mat_off);
    tf::layout_kernel<<<1, 1024, E * 4, s>>>(mat, w, E, rank, seg_base, a->counts, a->recv_rows);
    tf::PeerPtrs recv{};
    tf::PeerSig flags{};
    for (int p = 0; p < w; ++p) {
      recv.p[p] = t->pes[p].base + m.recv_off;
      flags.p[p] = t->pes[p].sig + sig + w;
    }
    static uint64_t attr_done = 0;
    if (!(attr_done & (1ull << dev))) {
      TF_CUDA_TRY(cudaFuncSetAttribute(tf::scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tf::kScatterWarps * tf::kScatterBuf));
      attr_done |= 1ull << dev;
    }
    if (entries > 0)
    {
      static const int sv = [] {
        const char* e = getenv("TF_MOE_SCATTER");
        return e ? atoi(e) : 2;
      }();
      if (sv == 2) {
        static uint64_t attr2 = 0;
        constexpr int smem2 = 2 * tf::kScatter2Warps * tf::kScatter2Buf;
        if (!(attr2 & (1ull << dev))) {
          TF_CUDA_TRY(cudaFuncSetAttribute(tf::scatter2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           smem2));
          attr2 |= 1ull << dev;
        }
        int per_sm = 0;
        TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tf::scatter2_kernel,
                                                                  32 * tf::kScatter2Warps, smem2));
        const int64_t tasks = a->tokens * ((a->hidden / 8 + tf::kScatter2Buf / 16 - 1) / (tf::kScatter2Buf / 16));
        const int64_t cap = static_cast<int64_t>(tf::num_sms_of_current_device()) * std::max(per_sm, 1);
        const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, (tasks + tf::kScatter2Warps - 1) /
                                                                                        tf::kScatter2Warps)));
        tf::scatter2_kernel<<<grid, 32 * tf::kScatter2Warps, smem2, s>>>(
            static_cast<const uint4*>(a->x), a->tokens, a->hidden / 8, a->k, E, w, a->topk_idx,
            a->sorted_pos, ebase, seg_base, a->dest_row, recv, a->max_recv, t->err_word(rank), rank);
      } else {
        tf::scatter_kernel<<<tf::grid_for(a->tokens * ((a->hidden / 8 + 511) / 512)), 32 * tf::kScatterWarps,
                             tf::kScatterWarps * tf::kScatterBuf, s>>>(
            static_cast<const uint4*>(a->x), a->tokens, a->hidden / 8, a->k, E, w, a->topk_idx,
            a->sorted_pos, ebase, seg_base, a->dest_row, recv, a->max_recv, t->err_word(rank), rank);
      }
    }
    if (w > 1) tf::release_kernel<<<1, 32 * ((w + 31) / 32), 0, s>>>(flags, w, rank, e);
    TF_CUDA_TRY(cudaGetLastError());
  }
  if ((phase & TF_PHASE_POST) && w > 1) {
    const uint64_t e = m.ws->epoch[rank];
    tf::wait_flags_kernel<<<1, 32 * ((w + 31) / 32), 0, s>>>(t->pes[rank].sig + sig + w, w, e,
                                                             t->timeout_ns, t->err_word(rank),
                                                             0x5100000ull);
    TF_CUDA_TRY(cudaGetLastError());
  }
  return TF_OK;
}

int tf_moe_combine(tf_team* t, int rank, const tf_moe_args* a, int phase, void* stream) {
  int rc = tf::check_moe(t, rank, a);
  if (rc) return rc;
  tf::MoeWs m;
  rc = tf::moe_workspace(t, a, &m);
  if (rc) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  const int w = t->world;
  const size_t sig = m.ws->sig_base + 2 * w;
  const uint64_t e = m.ws->epoch[rank];  // same epoch as the dispatch it answers
  if ((phase & TF_PHASE_PRE) && w > 1) {
    tf::PeerSig flags{};
    for (int p = 0; p < w; ++p) flags.p[p] = t->pes[p].sig + sig;
    tf::release_kernel<<<1, 32 * ((w + 31) / 32), 0, s>>>(flags, w, rank, e);
    TF_CUDA_TRY(cudaGetLastError());
  }
  if (phase & TF_PHASE_MAIN) {
    if (w > 1)
      tf::wait_flags_kernel<<<1, 32 * ((w + 31) / 32), 0, s>>>(t->pes[rank].sig + sig, w, e,
                                                               t->timeout_ns, t->err_word(rank),
                                                               0x5200000ull);
    tf::PeerPtrs y{};
    for (int p = 0; p < w; ++p) y.p[p] = t->pes[p].base + m.yout_off;
    if (a->tokens > 0)
    {
      static const int cv = [] {
        const char* e = getenv("TF_MOE_COMBINE_U");
        return e ? atoi(e) : 2;
      }();
      if (a->k <= 8 && cv == 2)
        tf::combine8_kernel<2><<<tf::grid_for(a->tokens), 256, 0, s>>>(
            a->tokens, a->hidden / 8, a->k, a->n_experts, w, a->topk_idx, a->topk_w, a->dest_row, y,
            static_cast<uint4*>(a->out));
      else if (a->k <= 8 && cv == 4)
        tf::combine8_kernel<4><<<tf::grid_for(a->tokens), 256, 0, s>>>(
            a->tokens, a->hidden / 8, a->k, a->n_experts, w, a->topk_idx, a->topk_w, a->dest_row, y,
            static_cast<uint4*>(a->out));
      else if (a->k <= 8 && cv == 1)
        tf::combine8_kernel<1><<<tf::grid_for(a->tokens), 256, 0, s>>>(
            a->tokens, a->hidden / 8, a->k, a->n_experts, w, a->topk_idx, a->topk_w, a->dest_row, y,
            static_cast<uint4*>(a->out));
      else
        tf::combine_kernel<<<tf::grid_for(a->tokens), 256, 0, s>>>(
            a->tokens, a->hidden / 8, a->k, a->n_experts, w, a->topk_idx, a->topk_w, a->dest_row, y,
            static_cast<uint4*>(a->out));
    }
    TF_CUDA_TRY(cudaGetLastError());
  }
  return TF_OK;
}

}  // extern "C"

