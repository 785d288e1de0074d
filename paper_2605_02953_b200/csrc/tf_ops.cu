// Fused collective operators: AllGather+GEMM and GEMM+ReduceScatter.
//
// tf_ag_gemm  <- ovs/kernels/ag_gemm.py:20-94
//   PRE : local A shard -> own workspace slot [rank] (D2D copy fusion), own
//         arrival flag := epoch, barrier arrive              (ag_gemm.py:59-62)
//   MAIN: barrier wait; on comm_stream the pull engine copies chunk
//         (rank+i)%w from the peer's workspace (copy engine over NVLink) and
//         then stores arrival[src] := epoch (ag_gemm.py:64-69); on `stream`
//         the persistent tcgen05 GEMM runs the gather-swizzled tile order and
//         acquire-waits per tile on the covering chunks (ag_gemm.py:72-94).
//   The workspace is double-buffered by epoch parity so one barrier per call
//   is enough (a peer can be at most one call behind).
//
// tf_gemm_rs  <- ovs/kernels/gemm_rs.py:31-338
//   fused   : epilogue stores each tile's row slices into the owners' slot
//             [rank] (gemm_rs.py:135-162) and release-adds the owner's
//             per-row-tile counter; the owner reduces its `world` slots in fp32
//             in ascending or ring order once a row tile's counter reaches
//             world * num_pid_n (gemm_rs.py:325-338).
//   unfused : tiles land in the producer's own gemm_out; the same counters
//             (gemm_rs.py:107-132) release the owner's pull-reduce, which
//             reads the peers' rows directly over NVLink (gemm_rs.py:177-196).
//   Counters are reset by their owner after the reduce (gemm_rs.py:168-174);
//   the barrier at the start of the next call orders the reset before any
//   peer's next increment.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

constexpr int kBM = 128;

struct ReduceSrc {
  const void* src[kMaxWorld];  // row 0 of this owner's block in each source's buffer
};

// Owner-side reduction of `world` partial row blocks.  Work item = (row tile,
// 2048-column chunk); waits on the row tile's arrival counter, then sums the
// sources in `order` in fp32 with 16-byte vector loads.
template <bool IN_F32>
__global__ void __launch_bounds__(256) rs_reduce_kernel(
    ReduceSrc srcs, long long src_ld, int world, int nnodes, int intra_ring, int inter_ring, int owner, void* out,
    long long out_ld, int out_f32, int out_vec, long long rows, long long n, long long row0_global,
    const uint64_t* counters, unsigned long long expected, int first_tile, int ntiles,
    int col_chunks, unsigned long long timeout_ns, unsigned long long* err,
    unsigned long long* trace, int trace_cap) {
  const int items = ntiles * col_chunks;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int t = item / col_chunks;
    const int cc = item - t * col_chunks;
    const int pid_m = first_tile + t;
    if (counters) {
      if (threadIdx.x == 0) {
        wait_geq_sys(counters + pid_m, expected, timeout_ns, err, 0x4000000ull | pid_m);
        if (trace) {  // the row block's "segment ready" moment, seen by its owner
          const unsigned long long now = globaltimer_ns();
          trace_push(trace, trace_cap, 5, owner, pid_m, now, now,
                     (static_cast<unsigned long long>(owner) << 32) |
                         static_cast<unsigned>(ld_relaxed_sys(counters + pid_m)));
        }
      }
      __syncthreads();
    }
    // rows of this owner covered by global row tile pid_m
    const long long g0 = max(static_cast<long long>(pid_m) * kBM, row0_global);
    const long long g1 = min(static_cast<long long>(pid_m + 1) * kBM, row0_global + rows);
    const long long c0 = static_cast<long long>(cc) * 2048;
    const long long c1 = min(c0 + 2048, n);
    const long long width = c1 - c0;
    const long long vec_per_row = (width + 7) / 8;
    const long long total = (g1 - g0) * vec_per_row;
    for (long long v = threadIdx.x; v < total; v += blockDim.x) {
      const long long r = g0 - row0_global + v / vec_per_row;
      const long long c = c0 + (v % vec_per_row) * 8;
      // The reference's summation tree (gemm_rs.py:199-319): node partials are left
      // folds over the node's ranks in the intra-node order (reduce_visit_order, or the
      // neighbour ring when links are not a full mesh), then a left fold of the node
      // partials in the inter-node order.  One node: a flat fold.
      float acc[8], part[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
      const bool full = c + 8 <= n;
      const int lws = world / nnodes;
      const int onode = owner / lws, olocal = owner % lws;
      for (int a = 0; a < nnodes; ++a) {
        const int nd = inter_ring ? (onode + 1 + a) % nnodes : a;
#pragma unroll
        for (int j = 0; j < 8; ++j) part[j] = 0.f;
        for (int b = 0; b < lws; ++b) {
          const int s = nd * lws + (intra_ring ? (olocal + 1 + b) % lws : b);
          if constexpr (IN_F32) {
            const float* p = static_cast<const float*>(srcs.src[s]) + r * src_ld + c;
            if (full) {
              const float4 x0 = *reinterpret_cast<const float4*>(p);
              const float4 x1 = *reinterpret_cast<const float4*>(p + 4);
              part[0] += x0.x; part[1] += x0.y; part[2] += x0.z; part[3] += x0.w;
              part[4] += x1.x; part[5] += x1.y; part[6] += x1.z; part[7] += x1.w;
            } else {
              for (int j = 0; j < 8 && c + j < n; ++j) part[j] += p[j];
            }
          } else {
            const uint16_t* p = static_cast<const uint16_t*>(srcs.src[s]) + r * src_ld + c;
            if (full) {
              const uint4 x = *reinterpret_cast<const uint4*>(p);
              const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                part[2 * j] += __uint_as_float(w[j] << 16);
                part[2 * j + 1] += __uint_as_float(w[j] & 0xFFFF0000u);
              }
            } else {
              for (int j = 0; j < 8 && c + j < n; ++j)
                part[j] += __uint_as_float(static_cast<uint32_t>(p[j]) << 16);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += part[j];
      }
      if (out_f32) {
        float* o = static_cast<float*>(out) + r * out_ld + c;
        if (full && out_vec) {
          *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
          *reinterpret_cast<float4*>(o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
        } else {
          for (int j = 0; j < 8 && c + j < n; ++j) o[j] = acc[j];
        }
      } else {
        uint16_t* o = static_cast<uint16_t*>(out) + r * out_ld + c;
        if (full && out_vec) {
          *reinterpret_cast<uint4*>(o) =
              make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                         pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
        } else {
          for (int j = 0; j < 8 && c + j < n; ++j)
            o[j] = static_cast<uint16_t>(pack_bf16x2(acc[j], 0.f) & 0xFFFF);
        }
      }
    }
    __syncthreads();
  }
}

struct PeerBase {
  const void* p[kMaxWorld];
};
struct PeerCnt {
  const uint64_t* p[kMaxWorld];
};
struct PeerOut {
  void* p[kMaxWorld];
};
struct PeerFlag {
  uint64_t* p[kMaxWorld];
};

// GEMM+AllReduce reduction.  Work item = (128-row block b, 2048-column chunk).
// one-shot (bcast == 0): reduce every block into `out` (local).
// two-shot (bcast == 1): reduce only blocks b % world == rank, store the result
// into every peer's result buffer and release flag[b] on each peer.
template <bool IN_F32>
__global__ void __launch_bounds__(256) ar_reduce_kernel(
    PeerBase parts, long long ld, int world, int rank, int bcast, void* out, long long out_ld,
    int out_f32, int out_vec, PeerOut results, PeerFlag flags, long long m, long long n,
    PeerCnt counters, unsigned long long expected, int col_chunks, unsigned long long epoch,
    unsigned long long timeout_ns, unsigned long long* err) {
  const int nblocks = static_cast<int>((m + 127) / 128);
  const int my_blocks = bcast ? (nblocks - rank + world - 1) / world : nblocks;
  const int items = my_blocks * col_chunks;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int bi = item / col_chunks;
    const int cc = item - bi * col_chunks;
    const int b = bcast ? rank + bi * world : bi;
    if (threadIdx.x < world)
      wait_geq_sys(counters.p[threadIdx.x] + b, expected, timeout_ns, err, 0x4000000ull | b);
    __syncthreads();
    const long long r0 = static_cast<long long>(b) * 128;
    const long long r1 = min(r0 + 128, m);
    const long long c0 = static_cast<long long>(cc) * 2048;
    const long long c1 = min(c0 + 2048, n);
    const long long vec_per_row = (c1 - c0 + 7) / 8;
    const long long total = (r1 - r0) * vec_per_row;
    for (long long v = threadIdx.x; v < total; v += blockDim.x) {
      const long long r = r0 + v / vec_per_row;
      const long long c = c0 + (v % vec_per_row) * 8;
      const bool full = c + 8 <= n;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      for (int s = 0; s < world; ++s) {  // ascending rank order: deterministic
        if constexpr (IN_F32) {
          const float* p = static_cast<const float*>(parts.p[s]) + r * ld + c;
          if (full) {
            const float4 x0 = *reinterpret_cast<const float4*>(p);
            const float4 x1 = *reinterpret_cast<const float4*>(p + 4);
            acc[0] += x0.x; acc[1] += x0.y; acc[2] += x0.z; acc[3] += x0.w;
            acc[4] += x1.x; acc[5] += x1.y; acc[6] += x1.z; acc[7] += x1.w;
          } else {
            for (int j = 0; j < 8 && c + j < n; ++j) acc[j] += p[j];
          }
        } else {
          const uint16_t* p = static_cast<const uint16_t*>(parts.p[s]) + r * ld + c;
          if (full) {
            const uint4 x = *reinterpret_cast<const uint4*>(p);
            const uint32_t w4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[2 * j] += __uint_as_float(w4[j] << 16);
              acc[2 * j + 1] += __uint_as_float(w4[j] & 0xFFFF0000u);
            }
          } else {
            for (int j = 0; j < 8 && c + j < n; ++j)
              acc[j] += __uint_as_float(static_cast<uint32_t>(p[j]) << 16);
          }
        }
      }
      const int ndst = bcast ? world : 1;
      for (int d = 0; d < ndst; ++d) {
        void* base = bcast ? results.p[d] : out;
        const long long oll = bcast ? ld : out_ld;
        const bool vec = full && (bcast ? true : out_vec);
        if (out_f32) {
          float* o = static_cast<float*>(base) + r * oll + c;
          if (vec) {
            *reinterpret_cast<float4*>(o) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            *reinterpret_cast<float4*>(o + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
          } else {
            for (int j = 0; j < 8 && c + j < n; ++j) o[j] = acc[j];
          }
        } else {
          uint16_t* o = static_cast<uint16_t*>(base) + r * oll + c;
          if (vec) {
            *reinterpret_cast<uint4*>(o) =
                make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]),
                           pack_bf16x2(acc[4], acc[5]), pack_bf16x2(acc[6], acc[7]));
          } else {
            for (int j = 0; j < 8 && c + j < n; ++j)
              o[j] = static_cast<uint16_t>(pack_bf16x2(acc[j], 0.f) & 0xFFFF);
          }
        }
      }
    }
    if (bcast) {
      // publish the block's chunk: stores visible system-wide, then flag every peer
      fence_sys();
      __syncthreads();
      if (threadIdx.x < world) red_add_release_sys(flags.p[threadIdx.x] + b, 1);
    }
    __syncthreads();
  }
}

// Two-shot GEMM+AllReduce over NVLS (the reference's multimem_ld_reduce +
// multimem_st pair, gemm_ar.py:103-133): the partials live in the team's
// multicast region; for each owned block the owner issues multimem.ld_reduce on
// the multicast address (the NVSwitch sums every rank's copy) and multimem.st of
// the sum (the switch writes it into every rank's result copy), 16 bytes per
// instruction, then release-flags the block on every peer.  Requires
// ld * esz % 16 == 0 (ld is n rounded up to 8).
template <bool F32>
__global__ void __launch_bounds__(256) ar_nvls_kernel(
    const uint8_t* mc_parts, uint8_t* mc_res, long long ld, int world, int rank, long long m,
    long long n, PeerCnt counters, unsigned long long expected, PeerFlag flags, int col_chunks,
    unsigned long long timeout_ns, unsigned long long* err) {
  constexpr int esz = F32 ? 4 : 2;
  constexpr int per_vec = 16 / esz;
  const int nblocks = static_cast<int>((m + 127) / 128);
  const int my_blocks = (nblocks - rank + world - 1) / world;
  const int items = my_blocks * col_chunks;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int bi = item / col_chunks;
    const int cc = item - bi * col_chunks;
    const int b = rank + bi * world;
    if (threadIdx.x < world)
      wait_geq_sys(counters.p[threadIdx.x] + b, expected, timeout_ns, err, 0x4000000ull | b);
    __syncthreads();
    // partials were written through the unicast alias; read them through the multicast one
    asm volatile("fence.proxy.alias;" ::: "memory");
    const long long r0 = static_cast<long long>(b) * 128, r1 = min(r0 + 128, m);
    const long long c0 = static_cast<long long>(cc) * 2048, c1 = min(c0 + 2048, ld);
    const long long vec_per_row = (c1 - c0) / per_vec;
    const long long total = (r1 - r0) * vec_per_row;
    for (long long v = threadIdx.x; v < total; v += blockDim.x) {
      const long long r = r0 + v / vec_per_row;
      const long long c = c0 + (v % vec_per_row) * per_vec;
      const long long off = (r * ld + c) * esz;
      uint32_t q0, q1, q2, q3;
      if constexpr (F32)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q0), "=r"(q1), "=r"(q2), "=r"(q3) : "l"(mc_parts + off) : "memory");
      else
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q0), "=r"(q1), "=r"(q2), "=r"(q3) : "l"(mc_parts + off) : "memory");
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc_res + off),
                   "f"(__uint_as_float(q0)), "f"(__uint_as_float(q1)), "f"(__uint_as_float(q2)),
                   "f"(__uint_as_float(q3))
                   : "memory");
    }
    asm volatile("fence.proxy.alias;" ::: "memory");
    fence_sys();
    __syncthreads();
    if (threadIdx.x < world) red_add_release_sys(flags.p[threadIdx.x] + b, 1);
    __syncthreads();
  }
}

// two-shot tail: wait until every block's column chunks have been flagged
// (target = epoch * col_chunks), then copy the result buffer into `out`.
__global__ void ar_gather_kernel(const void* result, long long ld, void* out, long long out_ld,
                                 int esz, long long m, long long n, const uint64_t* flags,
                                 unsigned long long target, unsigned long long timeout_ns,
                                 unsigned long long* err) {
  const int nblocks = static_cast<int>((m + 127) / 128);
  for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
    if (threadIdx.x == 0) wait_geq_sys(flags + b, target, timeout_ns, err, 0x4800000ull | b);
    __syncthreads();
    asm volatile("fence.proxy.alias;" ::: "memory");  // NVLS: results arrived through the multicast alias
    const long long r0 = static_cast<long long>(b) * 128, r1 = min(r0 + 128, m);
    const long long row_bytes = n * esz;
    for (long long r = r0; r < r1; ++r) {
      const uint8_t* src = static_cast<const uint8_t*>(result) + r * ld * esz;
      uint8_t* dst = static_cast<uint8_t*>(out) + r * out_ld * esz;
      for (long long i = threadIdx.x; i < row_bytes; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
  }
}

struct StreamJoin {
  // fork `side` from `main` and join back; no-ops when they are the same stream
  static int fork(cudaStream_t main, cudaStream_t side) {
    if (main == side) return TF_OK;
    cudaEvent_t e;
    TF_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TF_CUDA_TRY(cudaEventRecord(e, main));
    TF_CUDA_TRY(cudaStreamWaitEvent(side, e, 0));
    cudaEventDestroy(e);
    return TF_OK;
  }
};

int check_gemm_args(const tf_gemm_args* a) {
  if (!a) return fail(TF_ERR_INVALID, "args is NULL");
  if (a->m < 0 || a->n < 0 || a->k < 1) return fail(TF_ERR_INVALID, "bad GEMM shape");
  if (a->block_m != 0 && a->block_m != 128 && a->block_m != 256 && a->block_m != 512)
    return fail(TF_ERR_CONFIG, "block_m must be 128 (one CTA), 256 or 512 (CTA pair)");
  if (a->block_n != 0 && a->block_n != 128 && a->block_n != 256)
    return fail(TF_ERR_CONFIG, "block_n must be 128 or 256");
  if (a->block_k != 0 && a->block_k != 64) return fail(TF_ERR_CONFIG, "block_k must be 64");
  if (a->out_dtype != TF_DTYPE_BF16 && a->out_dtype != TF_DTYPE_F32)
    return fail(TF_ERR_INVALID, "out_dtype must be TF_DTYPE_BF16 or TF_DTYPE_F32");
  if (a->num_gemm_sms < 0 || a->num_comm_sms < 0) return fail(TF_ERR_CONFIG, "negative SM count");
  return TF_OK;
}

GemmLaunch base_launch(const tf_gemm_args* a) {
  GemmLaunch g;
  g.a = a->a;
  g.b = a->b;
  g.m = a->m;
  g.n = a->n;
  g.k = a->k;
  g.lda = a->lda ? a->lda : a->k;
  g.ldb = a->ldb ? a->ldb : a->k;
  g.block_m = a->block_m ? a->block_m : 128;
  g.block_n = a->block_n ? a->block_n : 256;
  g.group_m = a->group_m > 0 ? a->group_m : 8;
  g.tile_map = a->swizzle ? a->tile_map : nullptr;
  g.out_f32 = a->out_dtype == TF_DTYPE_F32;
  g.c = a->c;
  g.ldc = a->ldc ? a->ldc : a->n;
  return g;
}

int gemm_grid(const tf_gemm_args* a) {
  // comm / reduce CTAs are small and co-reside with the 1-CTA/SM GEMM, so the
  // GEMM keeps every SM unless num_gemm_sms pins it (reference semantics)
  const int sms = num_sms_of_current_device();
  int g = a->num_gemm_sms > 0 ? a->num_gemm_sms : sms;
  if (g < 1) g = 1;
  if (g > sms) g = sms;
  return g;
}

}  // namespace
}  // namespace tf

using tf::fail;

extern "C" {

int tf_gemm(const tf_gemm_args* args, void* stream) {
  int rc = tf::check_gemm_args(args);
  if (rc) return rc;
  tf::GemmLaunch g = tf::base_launch(args);
  g.num_sms = tf::gemm_grid(args);
  return tf::launch_gemm(g, static_cast<cudaStream_t>(stream));
}

int tf_ag_gemm(tf_team* t, int rank, const tf_gemm_args* args, int phase, void* stream,
               void* comm_stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  int rc = tf::check_gemm_args(args);
  if (rc) return rc;
  const int w = t->world;
  if (args->m % w) return fail(TF_ERR_INVALID, "gathered M must divide evenly across ranks");
  if ((args->k * 2) % 16) return fail(TF_ERR_INVALID, "K must be a multiple of 8 (16-byte rows)");
  const int64_t mpr = args->m / w;
  if (w == 1) {
    // no exchange: the local GEMM straight from the caller's A (no workspace copy)
    if (!(phase & TF_PHASE_MAIN)) return TF_OK;
    tf::GemmLaunch g = tf::base_launch(args);
    g.num_sms = tf::gemm_grid(args);
    return tf::launch_gemm(g, static_cast<cudaStream_t>(stream));
  }
  const size_t chunk_bytes = static_cast<size_t>(mpr) * args->k * 2;
  // Each peer chunk is pulled as `sub` row slices with their own flags, so the first
  // wave of tiles waits for the first slice of a chunk, not the whole chunk (a TP8
  // chunk of config 2 is 16.8 MB: ~22 us at 770 GB/s).  Slices are whole 128-row
  // blocks; at most 64 flags per parity.
  constexpr int kMaxSub = 4;
  int sub = 1;
  for (int c = kMaxSub; c > 1; c /= 2)
    if (mpr % (128 * c) == 0 && w * c <= 64) { sub = c; break; }
  if (const char* e = getenv("TF_AG_SUBCHUNKS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= kMaxSub && mpr % v == 0 && w * v <= 64) sub = v;
  }
  const int fstride = w * kMaxSub;  // flags per call parity
  const int64_t rows_sub = mpr / sub;
  const size_t sub_bytes = chunk_bytes / sub;
  const int nflags = w * sub;
  const std::string key = "ag:" + std::to_string(args->m) + "x" + std::to_string(args->k);
  tf::Workspace* ws = t->workspace(key, 2 * chunk_bytes * w, 2 * fstride, &rc);
  if (!ws) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  auto cs = comm_stream ? static_cast<cudaStream_t>(comm_stream) : s;

  if (phase & TF_PHASE_PRE) {
    const uint64_t e = ++t->op_epoch[rank];
    const int par = static_cast<int>(e & 1);
    uint8_t* own = t->pes[rank].base + ws->data_off + par * chunk_bytes * w;
    const int64_t lda = args->lda ? args->lda : args->k;
    TF_CUDA_TRY(cudaMemcpy2DAsync(own + rank * chunk_bytes, args->k * 2, args->a, lda * 2,
                                  args->k * 2, mpr, cudaMemcpyDefault, s));
    for (int j = 0; j < sub; ++j) {
      rc = tf::stream_signal_set(t, rank, ws->sig_base + par * fstride + rank * sub + j, e, s);
      if (rc) return rc;
    }
    rc = tf::team_barrier_arrive(t, rank, s);
    if (rc) return rc;
  }
  if (phase & TF_PHASE_MAIN) {
    const uint64_t e = t->op_epoch[rank];
    const int par = static_cast<int>(e & 1);
    const size_t buf_off = ws->data_off + par * chunk_bytes * w;
    uint8_t* own = t->pes[rank].base + buf_off;
    rc = tf::team_barrier_wait(t, rank, s);
    if (rc) return rc;
    rc = tf::StreamJoin::fork(s, cs);
    if (rc) return rc;
    for (int i = 1; i < w; ++i) {
      const int src = (rank + i) % w;  // pull order of ag_gemm.py:64-69
      for (int j = 0; j < sub; ++j) {
        const size_t off = src * chunk_bytes + j * sub_bytes;
        TF_CUDA_TRY(cudaMemcpyAsync(own + off, t->pes[src].base + buf_off + off, sub_bytes,
                                    cudaMemcpyDefault, cs));
        rc = tf::stream_signal_set(t, rank, ws->sig_base + par * fstride + src * sub + j, e, cs);
        if (rc) return rc;
      }
    }
    (void)nflags;
    tf::GemmLaunch g = tf::base_launch(args);
    g.a = own;
    g.lda = args->k;
    g.num_sms = tf::gemm_grid(args);
    g.chunk_flags = t->pes[rank].sig + ws->sig_base + par * fstride;
    g.epoch = e;
    g.rows_per_chunk = rows_sub;
    g.chunks_per_rank = sub;
    g.trace_rank = rank;
    g.err = t->err_word(rank);
    g.timeout_ns = t->timeout_ns;
    rc = tf::launch_gemm(g, s);
    if (rc) return rc;
    rc = tf::StreamJoin::fork(cs, s);  // join: next call's comm is ordered after this GEMM
    if (rc) return rc;
  }
  if (phase & TF_PHASE_POST) {
    // epoch flags need no reset; nothing to do
  }
  return TF_OK;
}

int tf_gemm_rs(tf_team* t, int rank, const tf_gemm_args* args, int phase, void* stream,
               void* comm_stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  int rc = tf::check_gemm_args(args);
  if (rc) return rc;
  const int w = t->world;
  if (args->m % w) return fail(TF_ERR_INVALID, "M must divide evenly across ranks");
  const int64_t mpr = args->m / w;
  const int64_t n = args->n;
  if (w == 1) {
    // no exchange: rows of the only rank are the whole GEMM (tests/test_kernels.py:203-207)
    if (!(phase & TF_PHASE_MAIN)) return TF_OK;
    tf::GemmLaunch g = tf::base_launch(args);
    g.num_sms = tf::gemm_grid(args);
    return tf::launch_gemm(g, static_cast<cudaStream_t>(stream));
  }
  const bool f32 = args->out_dtype == TF_DTYPE_F32;
  const int esz = f32 ? 4 : 2;
  const int64_t ld = (n + 7) / 8 * 8;  // 16-byte aligned slot rows
  const int64_t num_pid_m = (args->m + tf::kBM - 1) / tf::kBM;
  const int bn = args->block_n ? args->block_n : 256;
  const int64_t num_pid_n = (n + bn - 1) / bn;
  const bool fused = args->fuse_scatter != 0;
  // fused: [world][mpr][ld] slots; unfused: gemm_out [m][ld] (same size)
  const size_t bytes = static_cast<size_t>(args->m) * ld * esz;
  const std::string key = std::string(fused ? "rsf:" : "rsu:") + std::to_string(args->m) + "x" +
                          std::to_string(n) + (f32 ? "f" : "h") + ":" + std::to_string(bn);
  tf::Workspace* ws = t->workspace(key, bytes, static_cast<size_t>(num_pid_m), &rc);
  if (!ws) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  auto cs = comm_stream ? static_cast<cudaStream_t>(comm_stream) : s;
  // the reduce may overlap the GEMM only when no other rank shares this device
  const bool overlap = t->distinct_devices && cs != s;

  auto launch_reduce = [&](cudaStream_t rs) -> int {
    tf::ReduceSrc srcs{};
    for (int src = 0; src < w; ++src) {
      if (fused)
        srcs.src[src] = t->pes[rank].base + ws->data_off + static_cast<size_t>(src) * mpr * ld * esz;
      else
        srcs.src[src] = t->pes[src].base + ws->data_off + static_cast<size_t>(rank) * mpr * ld * esz;
    }
    const int64_t first_tile = rank * mpr / tf::kBM;
    const int64_t last_tile = ((rank + 1) * mpr - 1) / tf::kBM;
    const int ntiles = static_cast<int>(last_tile - first_tile + 1);
    const int col_chunks = static_cast<int>((n + 2047) / 2048);
    const int ldc = static_cast<int>(args->ldc ? args->ldc : n);
    // overlapped: a few co-resident CTAs (they fit beside the 1-CTA/SM GEMM);
    // serialised: the whole GPU
    int grid = overlap ? (args->num_comm_sms > 0 ? args->num_comm_sms * 2 : 16)
                       : tf::num_sms_of_current_device();
    const int items = ntiles * col_chunks;
    if (grid > items) grid = items;
    if (grid < 1) grid = 1;
    const unsigned long long expected = static_cast<unsigned long long>(w) * num_pid_n;
    const uint64_t* cnt = t->pes[rank].sig + ws->sig_base;
    const int out_vec = ((static_cast<int64_t>(ldc) * esz) % 16 == 0) &&
                        (reinterpret_cast<uintptr_t>(args->c) % 16 == 0);
    // summation tree: fused = one flat fold over the world (_fused_reducer); unfused =
    // the hierarchical reducer with the neighbour ring inside a node when the links are
    // not a full mesh (_hier_reducer / _scatter_ring)
    const int ring = args->reduce_order == TF_REDUCE_RING;
    const int nn = (!fused && args->nnodes > 1 && w % args->nnodes == 0) ? args->nnodes : 1;
    const int intra = (!fused && args->ring_links && w / nn > 1) ? 1 : ring;
    int dev = 0;
    cudaGetDevice(&dev);
    unsigned long long* tr = nullptr;
    const int tcap = tf::trace_buffer(dev, &tr);
    if (f32)
      tf::rs_reduce_kernel<true><<<grid, 256, 0, rs>>>(
          srcs, ld, w, nn, intra, ring, rank, args->c, ldc, 1, out_vec, mpr, n,
          rank * mpr, cnt, expected, static_cast<int>(first_tile), ntiles, col_chunks,
          t->timeout_ns, t->err_word(rank), tr, tcap);
    else
      tf::rs_reduce_kernel<false><<<grid, 256, 0, rs>>>(
          srcs, ld, w, nn, intra, ring, rank, args->c, ldc, 0, out_vec, mpr, n,
          rank * mpr, cnt, expected, static_cast<int>(first_tile), ntiles, col_chunks,
          t->timeout_ns, t->err_word(rank), tr, tcap);
    TF_CUDA_TRY(cudaGetLastError());
    // owner resets its counters once consumed (gemm_rs.py:168-174)
    TF_CUDA_TRY(cudaMemsetAsync(t->pes[rank].sig + ws->sig_base, 0, num_pid_m * sizeof(uint64_t), rs));
    return TF_OK;
  };

  if (phase & TF_PHASE_PRE) {
    rc = tf::team_barrier_arrive(t, rank, s);
    if (rc) return rc;
  }
  if (phase & TF_PHASE_MAIN) {
    rc = tf::team_barrier_wait(t, rank, s);
    if (rc) return rc;
    tf::GemmLaunch g = tf::base_launch(args);
    g.num_sms = tf::gemm_grid(args);
    g.trace_rank = rank;
    g.epilogue = 1;
    g.rank = rank;
    g.world = w;
    g.rows_per_rank = mpr;
    g.slot_ld = ld;
    g.out_f32 = f32;
    for (int o = 0; o < w; ++o) {
      uint8_t* slots_o = t->pes[o].base + ws->data_off;
      if (fused) {
        g.peer_slots[o] = slots_o;
      } else {
        // own gemm_out, biased so that row = o*mpr + orow lands at its natural place
        uint8_t* own = t->pes[rank].base + ws->data_off;
        g.peer_slots[o] = own + (static_cast<int64_t>(o) - rank) * mpr * ld * esz;
      }
      g.peer_counts[o] = t->pes[o].sig + ws->sig_base;
    }
    g.err = t->err_word(rank);
    g.timeout_ns = t->timeout_ns;
    // The GEMM is enqueued first and the reduce only waits on the pre-GEMM
    // point of `stream`: whatever the streams' blocking semantics, the spinning
    // reduce can never sit in front of the producer it waits for.
    cudaEvent_t pre = nullptr;
    if (overlap) {
      TF_CUDA_TRY(cudaEventCreateWithFlags(&pre, cudaEventDisableTiming));
      TF_CUDA_TRY(cudaEventRecord(pre, s));
    }
    rc = tf::launch_gemm(g, s);
    if (rc) return rc;
    if (overlap) {
      TF_CUDA_TRY(cudaStreamWaitEvent(cs, pre, 0));
      cudaEventDestroy(pre);
      rc = launch_reduce(cs);
      if (rc) return rc;
      rc = tf::StreamJoin::fork(cs, s);
      if (rc) return rc;
    }
  }
  if (phase & TF_PHASE_POST) {
    if (!overlap) {
      rc = launch_reduce(s);
      if (rc) return rc;
    }
  }
  return TF_OK;
}

int tf_gemm_ar(tf_team* t, int rank, const tf_gemm_args* args, int two_shot, int phase,
               void* stream, void* comm_stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  int rc = tf::check_gemm_args(args);
  if (rc) return rc;
  const int w = t->world;
  const int64_t m = args->m, n = args->n;
  const bool f32 = args->out_dtype == TF_DTYPE_F32;
  const int esz = f32 ? 4 : 2;
  const int64_t ld = (n + 7) / 8 * 8;
  const int bn = args->block_n ? args->block_n : 256;
  const int64_t num_pid_n = (n + bn - 1) / bn;
  const int64_t nblocks = (m + 127) / 128;
  const int col_chunks = static_cast<int>((n + 2047) / 2048);
  const size_t bytes = static_cast<size_t>(m) * ld * esz;
  // one workspace per protocol: the broadcast flags only advance in two-shot calls,
  // so their epoch must not be shared with one-shot calls
  const std::string key = std::string(two_shot ? "ar2:" : "ar1:") + std::to_string(m) + "x" +
                          std::to_string(n) + (f32 ? "f" : "h") + ":" + std::to_string(bn);
  // data: partial [m][ld] + result [m][ld]; signals: counters [nblocks] + flags [nblocks]
  tf::Workspace* ws = t->workspace(key, 2 * bytes, 2 * static_cast<size_t>(nblocks), &rc);
  if (!ws) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  auto cs = comm_stream ? static_cast<cudaStream_t>(comm_stream) : s;
  const bool overlap = t->distinct_devices && cs != s && w > 1;
  if (phase & TF_PHASE_PRE) {
    ++ws->epoch[rank];
    rc = tf::team_barrier_arrive(t, rank, s);
    if (rc) return rc;
  }
  const uint64_t e = ws->epoch[rank];
  // NVLS two-shot: partials and results in the team's multicast region
  size_t nv_off = 0;
  const bool nvls = two_shot && w > 1 && t->distinct_devices && (ld * esz) % 16 == 0 &&
                    tf::nvls_workspace(t, key, 2 * bytes, &nv_off);
  auto launch_reduce = [&](cudaStream_t rs) -> int {
    if (nvls) {
      tf::PeerCnt cnt{};
      tf::PeerFlag flg{};
      for (int p = 0; p < w; ++p) {
        cnt.p[p] = t->pes[p].sig + ws->sig_base;
        flg.p[p] = t->pes[p].sig + ws->sig_base + nblocks;
      }
      const int64_t my_blocks = (nblocks - rank + w - 1) / w;
      int grid = overlap ? (args->num_comm_sms > 0 ? args->num_comm_sms * 2 : 16)
                         : tf::num_sms_of_current_device();
      if (grid > my_blocks * col_chunks) grid = static_cast<int>(my_blocks * col_chunks);
      if (grid < 1) grid = 1;
      const unsigned long long expected = e * static_cast<unsigned long long>(num_pid_n);
      const uint8_t* mp = t->nvls_mc + nv_off;
      uint8_t* mr = t->nvls_mc + nv_off + bytes;
      if (f32)
        tf::ar_nvls_kernel<true><<<grid, 256, 0, rs>>>(mp, mr, ld, w, rank, m, n, cnt, expected, flg,
                                                       col_chunks, t->timeout_ns, t->err_word(rank));
      else
        tf::ar_nvls_kernel<false><<<grid, 256, 0, rs>>>(mp, mr, ld, w, rank, m, n, cnt, expected, flg,
                                                        col_chunks, t->timeout_ns, t->err_word(rank));
      TF_CUDA_TRY(cudaGetLastError());
      return TF_OK;
    }
    tf::PeerBase parts{};
    tf::PeerCnt cnt{};
    tf::PeerOut res{};
    tf::PeerFlag flg{};
    for (int p = 0; p < w; ++p) {
      parts.p[p] = t->pes[p].base + ws->data_off;
      cnt.p[p] = t->pes[p].sig + ws->sig_base;
      res.p[p] = t->pes[p].base + ws->data_off + bytes;
      flg.p[p] = t->pes[p].sig + ws->sig_base + nblocks;
    }
    const int64_t ldc = args->ldc ? args->ldc : n;
    const int out_vec = ((ldc * esz) % 16 == 0) && (reinterpret_cast<uintptr_t>(args->c) % 16 == 0);
    int grid = overlap ? (args->num_comm_sms > 0 ? args->num_comm_sms * 2 : 16)
                       : tf::num_sms_of_current_device();
    const int64_t my_blocks = two_shot ? (nblocks - rank + w - 1) / w : nblocks;
    if (grid > my_blocks * col_chunks) grid = static_cast<int>(my_blocks * col_chunks);
    if (grid < 1) grid = 1;
    const unsigned long long expected = e * static_cast<unsigned long long>(num_pid_n);
    if (f32)
      tf::ar_reduce_kernel<true><<<grid, 256, 0, rs>>>(
          parts, ld, w, rank, two_shot, args->c, ldc, 1, out_vec, res, flg, m, n, cnt, expected,
          col_chunks, e, t->timeout_ns, t->err_word(rank));
    else
      tf::ar_reduce_kernel<false><<<grid, 256, 0, rs>>>(
          parts, ld, w, rank, two_shot, args->c, ldc, 0, out_vec, res, flg, m, n, cnt, expected,
          col_chunks, e, t->timeout_ns, t->err_word(rank));
    TF_CUDA_TRY(cudaGetLastError());
    return TF_OK;
  };
  auto launch_gather = [&](cudaStream_t gs) -> int {
    const int64_t ldc = args->ldc ? args->ldc : n;
    int grid = static_cast<int>(std::min<int64_t>(nblocks, tf::num_sms_of_current_device()));
    const uint8_t* res = nvls ? t->nvls_uc[rank] + nv_off + bytes : t->pes[rank].base + ws->data_off + bytes;
    tf::ar_gather_kernel<<<std::max(grid, 1), 256, 0, gs>>>(
        res, ld, args->c, ldc, esz, m, n,
        t->pes[rank].sig + ws->sig_base + nblocks, e * static_cast<unsigned long long>(col_chunks),
        t->timeout_ns, t->err_word(rank));
    TF_CUDA_TRY(cudaGetLastError());
    return TF_OK;
  };
  if (phase & TF_PHASE_MAIN) {
    rc = tf::team_barrier_wait(t, rank, s);
    if (rc) return rc;
    tf::GemmLaunch g = tf::base_launch(args);
    g.num_sms = tf::gemm_grid(args);
    g.epilogue = 1;  // own partial buffer + own counters (single "owner")
    g.rank = 0;
    g.world = 1;
    g.rows_per_rank = m;
    g.slot_ld = ld;
    g.out_f32 = f32;
    g.peer_slots[0] = nvls ? static_cast<void*>(t->nvls_uc[rank] + nv_off)
                           : static_cast<void*>(t->pes[rank].base + ws->data_off);
    g.peer_counts[0] = t->pes[rank].sig + ws->sig_base;
    g.err = t->err_word(rank);
    g.timeout_ns = t->timeout_ns;
    cudaEvent_t pre = nullptr;
    if (overlap) {
      TF_CUDA_TRY(cudaEventCreateWithFlags(&pre, cudaEventDisableTiming));
      TF_CUDA_TRY(cudaEventRecord(pre, s));
    }
    rc = tf::launch_gemm(g, s);
    if (rc) return rc;
    if (overlap) {
      TF_CUDA_TRY(cudaStreamWaitEvent(cs, pre, 0));
      cudaEventDestroy(pre);
      rc = launch_reduce(cs);
      if (rc) return rc;
      if (two_shot) {
        rc = launch_gather(cs);
        if (rc) return rc;
      }
      rc = tf::StreamJoin::fork(cs, s);
      if (rc) return rc;
    }
  }
  if (phase & TF_PHASE_POST) {
    if (!overlap) {
      rc = launch_reduce(s);
      if (rc) return rc;
    }
  }
  // two-shot results are only complete once every owner has broadcast: with shared
  // devices the gather must follow every rank's POST, so it runs as a 4th phase bit
  if ((phase & 8) && two_shot && !overlap) {
    rc = launch_gather(s);
    if (rc) return rc;
  }
  return TF_OK;
}

int tf_ag_kv_scores(tf_team* t, int rank, const tf_attn_args* a, int phase, void* stream,
                    void* comm_stream) {
  if (!t || !a || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "bad team/rank/args");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  if (a->s_local < 0 || a->hq < 1 || a->hkv < 1 || a->hq % a->hkv)
    return fail(TF_ERR_INVALID, "need hq % hkv == 0 and positive head counts");
  if (a->d < 8 || a->d % 8) return fail(TF_ERR_INVALID, "head dim must be a positive multiple of 8");
  if (a->out_dtype != TF_DTYPE_BF16 && a->out_dtype != TF_DTYPE_F32)
    return fail(TF_ERR_INVALID, "out_dtype must be TF_DTYPE_BF16 or TF_DTYPE_F32");
  const int w = t->world;
  const int64_t sl = a->s_local, st = sl * w;
  const int64_t krow = a->hkv * a->d;  // one key row: all kv heads
  const size_t chunk_bytes = static_cast<size_t>(sl) * krow * 2;
  auto s = static_cast<cudaStream_t>(stream);
  auto cs = comm_stream ? static_cast<cudaStream_t>(comm_stream) : s;
  int rc = TF_OK;
  const std::string key = "agkv:" + std::to_string(st) + "x" + std::to_string(krow);
  tf::Workspace* ws = t->workspace(key, 2 * chunk_bytes * w, 2 * w, &rc);
  if (!ws) return rc;
  if (phase & TF_PHASE_PRE) {
    const uint64_t e = ++ws->epoch[rank];
    const int par = static_cast<int>(e & 1);
    uint8_t* own = t->pes[rank].base + ws->data_off + par * chunk_bytes * w;
    if (chunk_bytes)
      TF_CUDA_TRY(cudaMemcpyAsync(own + rank * chunk_bytes, a->k, chunk_bytes, cudaMemcpyDefault, s));
    rc = tf::stream_signal_set(t, rank, ws->sig_base + par * w + rank, e, s);
    if (rc) return rc;
    if (w > 1) {
      rc = tf::team_barrier_arrive(t, rank, s);
      if (rc) return rc;
    }
  }
  if (phase & TF_PHASE_MAIN) {
    const uint64_t e = ws->epoch[rank];
    const int par = static_cast<int>(e & 1);
    const size_t buf_off = ws->data_off + par * chunk_bytes * w;
    uint8_t* own = t->pes[rank].base + buf_off;
    if (w > 1) {
      rc = tf::team_barrier_wait(t, rank, s);
      if (rc) return rc;
      rc = tf::StreamJoin::fork(s, cs);
      if (rc) return rc;
      for (int i = 1; i < w; ++i) {
        const int src = (rank + i) % w;  // pull order of ag_gemm.py:64-69
        TF_CUDA_TRY(cudaMemcpyAsync(own + src * chunk_bytes,
                                    t->pes[src].base + buf_off + src * chunk_bytes, chunk_bytes,
                                    cudaMemcpyDefault, cs));
        rc = tf::stream_signal_set(t, rank, ws->sig_base + par * w + src, e, cs);
        if (rc) return rc;
      }
    }
    const int64_t group = a->hq / a->hkv;
    const int esz = a->out_dtype == TF_DTYPE_F32 ? 4 : 2;
    for (int64_t h = 0; h < a->hq && sl > 0; ++h) {
      tf::GemmLaunch g;
      g.a = static_cast<const uint8_t*>(a->q) + h * a->d * 2;  // Q_h: rows stride hq*d
      g.lda = a->hq * a->d;
      g.b = own + (h / group) * a->d * 2;                        // K_g: rows stride hkv*d
      g.ldb = krow;
      g.m = sl;
      g.n = st;
      g.k = a->d;
      g.block_m = a->block_m ? a->block_m : 256;
      g.block_n = a->block_n ? a->block_n : 256;
      g.group_m = a->group_m > 0 ? a->group_m : 8;
      g.num_sms = a->num_gemm_sms > 0 ? a->num_gemm_sms : tf::num_sms_of_current_device();
      g.tile_map_n = a->swizzle ? a->key_tile_map : nullptr;
      g.out_f32 = a->out_dtype == TF_DTYPE_F32;
      g.c = static_cast<uint8_t*>(a->scores) + static_cast<size_t>(h) * sl * st * esz;
      g.ldc = st;
      g.chunk_flags = t->pes[rank].sig + ws->sig_base + par * w;
      g.epoch = e;
      g.rows_per_chunk = sl;
      g.wait_on_b = true;
      g.no_tail_split = true;
      g.trace_rank = rank;
      g.err = t->err_word(rank);
      g.timeout_ns = t->timeout_ns;
      rc = tf::launch_gemm(g, s);
      if (rc) return rc;
    }
    if (w > 1) {
      rc = tf::StreamJoin::fork(cs, s);
      if (rc) return rc;
    }
  }
  return TF_OK;
}

}  // extern "C"
