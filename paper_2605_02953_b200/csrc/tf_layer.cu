// Task-level megakernel for a fused transformer layer in bf16 (BASELINE config 5;
// SURVEY §8(f) #1).  Same wire contract as the reference's executor
// (ovs/megakernel/encoding.py:20-166, builders.py:105-162, scoreboard.py:33-56,
// runner.py:120-195): 30-word task records in [slot][sm] queues, dependency rows
// (producer task, first tile, one-past-last tile), scoreboard slot
// task * max_tiles + tile, release-stored with the call epoch.
//
// One persistent launch, one CTA per SM, 256 threads with fixed roles; every role
// walks the CTA's queue in order and does its share of each task:
//
//   task          warp 0 (TMA)            warp 1 (MMA, one lane)     warps 2-5 (128 thr)
//   linear        wait deps, A (2 x 128   tcgen05 128x256x16 per     TMEM -> epilogue (plain |
//   (256 x 256)   rows) + B (256 rows)    M-half into TMEM [0,256)   RoPE | SiLU*up) -> bf16
//                 boxes, 3-stage ring     and [256,512); half 1      per half, release the
//                                         lags 2 k-blocks at tile    tile flag
//                                         edges (drain overlaps)
//   attention     wait deps, Q of two    per head: S = Q K^T, then  online softmax per head
//   (2 heads of   heads once, K/V tiles  O += P V (P from TMEM,     (causal mask, lazy
//   a KV group)   through a 4-slot ring  V MN-major) and the next   rescale), P -> TMEM;
//                                        S in the same columns      one head's softmax
//                                                                   overlaps the other's MMAs
//   rmsnorm       -                       -                          - (warps 6-7: wait deps,
//                                                                      y = x*rstd*g)
//   allreduce_    -                       -                          - (warps 6-7: wait deps on
//   residual                                                           every PE, y = sum x_pe + res)
//
// The linear ring (3 x 64 KB) and the attention buffers (Q, 5 K/V slots) alias the
// same 192 KB of shared memory and TMEM columns [0, 512); when consecutive tensor
// tasks of a CTA change class, all six warps meet at a named barrier first, by
// which point every TMA load has been consumed and every MMA has retired.
// Elementwise tasks run on two dedicated warps (6-7), so the tensor roles keep
// streaming GEMM tiles while a norm or allreduce of the same CTA is in flight.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

constexpr int kLThreads = 256;      // warps 0-5 tensor roles, warps 6-7 elementwise tasks
constexpr int kTensorThreads = 192;
constexpr int kRing = 3;
constexpr int kHalfBox = 16384;               // 128 rows x 128 B
constexpr int kAStage = 2 * 128 * 64 * 2;     // two 128-row A blocks, 32 KB
constexpr int kBStage = 256 * 64 * 2;         // 32 KB
constexpr int kStage = kAStage + kBStage;     // 64 KB
constexpr int kRegion = kRing * kStage;       // 192 KB
constexpr int kLag = 2;                       // k-blocks the second M-half trails at tile edges
constexpr int kQOff = 0;                      // attention aliases: Q of up to 2 heads (64 KB)
constexpr int kKVOff = 4 * kHalfBox;          // ring of 4 K-or-V slots (32 KB each)
constexpr int kKVSlot = 2 * kHalfBox;
constexpr int kKVSlots = 4;                   // P lives in TMEM (over its S buffer), not smem
constexpr float kLazyRescale = 8.0f;          // log2 units the running max may lag before O is rescaled
constexpr int kLayerSmem = 1024 + kRegion + 512;
constexpr int kCfgInts = 16;
constexpr int kThrottleTasks = 64;
constexpr int kIntPerTask = 30;

enum { OP_RMSNORM = 1, OP_LINEAR = 2, OP_ATTENTION = 3, OP_ALLREDUCE_RES = 4 };
enum { EPI_NONE = 0, EPI_ROPE = 1, EPI_SILU_MUL = 2 };
enum { CLS_ELEM = 0, CLS_LINEAR = 1, CLS_ATTN = 2 };

struct LayerParams {
  const int32_t* queues;
  const int32_t* counts;
  const int32_t* deps;
  const int32_t* cfg;        // [layers][16]
  const CUtensorMap* maps;   // [ranks in launch][num_maps]
  int num_maps;
  int num_sms, max_tiles;
  int fixed_rank;            // IPC: this process's rank; local team: -1 (rank = cta / num_sms)
  const uint8_t* sm_die;     // die-ranked queues (one rank per launch): SM -> die table
  unsigned long long* die_ctr;  // and this launch's self-resetting counter, or nullptr
  // linear-tile wave throttle (TF_LAYER_THROTTLE): [ranks in launch][kThrottleTasks] tiles
  // started per task, zeroed before the launch; a CTA starts its k-th tile of a linear
  // task only once k * num_sms - num_sms / 2 tiles of it have started, so the round-robin
  // waves stay within ~1.5 waves of each other and their operand panels stay in L2
  unsigned* lin_started;
  int world;
  uint64_t flag_base;
  unsigned long long epoch;
  unsigned long long timeout_ns;
  uint8_t* base[kMaxWorld];
  uint64_t* sig[kMaxWorld];
  unsigned long long* err[kMaxWorld];
  unsigned long long* trace;  // [ctas][slots][4] or nullptr
  int slots;
};

struct Rec {
  int task_id, tile, dep0, dep1;
  long long off[4];  // bytes; tag bits 8-11 = shift of the encoded offset (heaps > 2 GiB)
  int d0[4], d1[4];
};

__device__ __forceinline__ void load_rec(const LayerParams& p, int idx, int sm, Rec& r) {
  const int32_t* q = p.queues + (static_cast<long long>(idx) * p.num_sms + sm) * kIntPerTask;
  r.task_id = __ldg(q + 2);
  r.tile = __ldg(q + 3);
  r.dep0 = __ldg(q + 4);
  r.dep1 = __ldg(q + 5);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    r.off[i] = static_cast<long long>(__ldg(q + 6 + 6 * i)) << ((__ldg(q + 7 + 6 * i) >> 8) & 0xF);
    r.d0[i] = __ldg(q + 8 + 6 * i);
    r.d1[i] = __ldg(q + 9 + 6 * i);
  }
}

__device__ __forceinline__ int op_class(int op) {
  return op == OP_LINEAR ? CLS_LINEAR : op == OP_ATTENTION ? CLS_ATTN : CLS_ELEM;
}

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Acquire-wait every dependency flag of the record, spread over `nt` threads
// (thread t takes flattened entries t, t + nt, ...); npe > 1 waits on every PE's
// scoreboard (allreduce).  Returns true if this thread waited on anything.
__device__ __forceinline__ bool wait_deps(const LayerParams& p, const Rec& r, int rank, int npe,
                                          int t, int nt) {
  bool any = false;
  int base = 0;
  for (int row = r.dep0; row < r.dep1; ++row) {
    const int prod = __ldg(p.deps + row * 3), lo = __ldg(p.deps + row * 3 + 1),
              hi = __ldg(p.deps + row * 3 + 2);
    const int cnt = (hi - lo) * npe;
    int e = base + ((t - base) % nt + nt) % nt;
    for (; e < base + cnt; e += nt) {
      const int i = e - base;
      const int tile = lo + i / npe;
      const int pe = npe == 1 ? rank : i % npe;
      const uint64_t slot = static_cast<uint64_t>(prod) * p.max_tiles + tile;
      wait_geq_sys(p.sig[pe] + p.flag_base + slot, p.epoch, p.timeout_ns, p.err[rank],
                   0x8000000ull | slot);
      any = true;
    }
    base += cnt;
  }
  return any;
}

// release (task, tile) on PE `pe`'s scoreboard; a flag already at this epoch is a
// double release (scoreboard.py:50-56), reported on the releasing rank's error word
__device__ __forceinline__ void release_flag(const LayerParams& p, int rank, const Rec& r, int pe) {
  uint64_t* f = p.sig[pe] + p.flag_base + static_cast<uint64_t>(r.task_id) * p.max_tiles + r.tile;
  if (ld_acquire_sys(f) >= p.epoch)
    atomicCAS(p.err[rank], 0ull,
              0x9000000ull | (static_cast<uint64_t>(r.task_id) * p.max_tiles + r.tile));
  fence_sys();
  st_release_sys(f, p.epoch);
}

// bulk L2 prefetch of [ptr, ptr + bytes) in 64 KB pieces, spread over the calling threads
__device__ __forceinline__ void prefetch_l2(const void* ptr, long long bytes, int t, int nt) {
  const char* c = static_cast<const char*>(ptr);
  for (long long o = static_cast<long long>(t) << 16; o < bytes; o += static_cast<long long>(nt) << 16) {
    const long long n = min(bytes - o, 65536ll);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c + o), "r"(static_cast<uint32_t>(n & ~15ll))
                 : "memory");
  }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// trace rows are per queue (the CTA's queue index `q`, die-ranked or blockIdx)
__device__ __forceinline__ unsigned long long* trace_at(const LayerParams& p, int q, int idx) {
  return p.trace + (static_cast<long long>(q) * p.slots + idx) * 4;
}

__device__ __forceinline__ void tma_load_3d_l(void* smem_dst, const void* tmap, uint64_t* bar,
                                              int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Descriptor = (low word, constant high word): per-MMA address math is one add on
// the low word (the single MMA thread shares its SMSP with epilogue/softmax warps).
constexpr uint32_t kDescHi = (1024 >> 4) | (1u << (46 - 32)) | (2u << (61 - 32));
__device__ __forceinline__ uint64_t desc_from_lo(uint32_t lo) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(kDescHi));
  return d;
}
__device__ __forceinline__ uint32_t desc_lo_k(uint32_t addr) { return ((addr & 0x3FFFF) >> 4) | (1u << 16); }
__device__ __forceinline__ uint32_t desc_lo_mn(uint32_t addr, uint32_t lbo) {
  return ((addr & 0x3FFFF) >> 4) | (((lbo >> 4) & 0x3FFF) << 16);
}


// D[tmem] (+)= A[tmem] * B[smem]^T (A = P, bf16 pairs packed per 32-bit column)
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// 32 fp32 values -> 32 bf16 at dst (64 B, 16-byte aligned), masked by `ncols` valid
__device__ __forceinline__ void store_bf16x32(uint16_t* dst, const float (&f)[32], int ncols) {
  uint32_t pk[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(f[2 * i], f[2 * i + 1]);
  if (ncols >= 32) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) d4[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  } else {
    uint32_t* d2 = reinterpret_cast<uint32_t*>(dst);
#pragma unroll
    for (int i = 0; i < 16; ++i) {  // ncols is a multiple of 8 (checked on the host)
      if (2 * i < ncols) d2[i] = pk[i];
    }
  }
}

struct AttnGeom {
  int n_kv, kv0, hq, hkv, g, h, q_row0, np;
};

// task = (128-query tile i, heads [h, h + np)) with np = 1 or 2 heads of one KV group
__device__ __forceinline__ AttnGeom attn_geom(const int* cfg, const Rec& r) {
  AttnGeom a;
  a.hq = cfg[7];
  a.hkv = cfg[8];
  a.np = cfg[14] > 1 ? 2 : 1;
  const int seq = cfg[9];
  const int causal = cfg[12];
  const int per_row = a.hq / a.np;
  const int i = r.tile / per_row;
  a.h = (r.tile % per_row) * a.np;
  a.g = a.h / (a.hq / a.hkv);
  a.q_row0 = i * 128;
  const int tiles_per_seq = seq / 128;
  a.kv0 = (i / tiles_per_seq) * tiles_per_seq;
  a.n_kv = causal ? i - a.kv0 + 1 : tiles_per_seq;
  return a;
}

__global__ void __launch_bounds__(kLThreads, 1) layer_megakernel(const __grid_constant__ LayerParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kRegion);
  uint64_t* full_bar = bars;            // [4]
  uint64_t* empty_bar = bars + 4;       // [4]
  uint64_t* tfull = bars + 8;           // [2]
  uint64_t* tempty = bars + 10;         // [2]
  uint64_t* q_full = bars + 12;
  uint64_t* q_empty = bars + 13;
  uint64_t* kv_full = bars + 28;        // [5] ring slots
  uint64_t* kv_empty = bars + 34;       // [5]
  uint64_t* s_full = bars + 18;         // [2] per head stream
  uint64_t* o_ready = bars + 20;        // [2]
  uint64_t* p_full = bars + 22;         // [2]
  uint64_t* o_empty = bars + 24;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 26);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = p.fixed_rank >= 0 ? p.fixed_rank : static_cast<int>(blockIdx.x) / p.num_sms;
  int sm = static_cast<int>(blockIdx.x) % p.num_sms;
  int* qslot = reinterpret_cast<int*>(bars + 27);
  if (p.die_ctr && threadIdx.x == 0) {
    // one rank per launch: take the queue by die rank (die-0 CTAs count up from 0, die-1
    // CTAs down from num_sms - 1), so a wave of round-robin queues gives each die a
    // compact block of the grouped GEMM raster (tf_topo.cu; same scheme as tf_gemm.cu)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int d = p.sm_die[smid & 255] & 1;
    const unsigned long long old = atomicAdd(p.die_ctr, d ? (1ull << 32) : 1ull);
    const int lo = static_cast<int>(old & 0xFFFFFFFFull), hi = static_cast<int>(old >> 32);
    if (lo + hi + 1 == p.num_sms) atomicExch(p.die_ctr, 0ull);
    *qslot = d ? p.num_sms - 1 - hi : lo;
  }
  const CUtensorMap* maps = p.maps + (p.fixed_rank >= 0 ? 0 : rank) * p.num_maps;
  uint8_t* my_base = p.base[rank];

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
      mbar_init(&s_full[i], 1);
      mbar_init(&o_ready[i], 1);
      mbar_init(&p_full[i], 4);
    }
    for (int i = 0; i < kKVSlots; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(o_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (p.die_ctr) sm = *qslot;
  const int qrow = p.fixed_rank >= 0 ? sm : rank * p.num_sms + sm;  // this CTA's trace row
  const int n_tasks = p.counts[sm];
  int last_cls = -1;

  if (warp == 0) {
    // =========================================================== TMA producer
    int stage = 0;
    uint32_t phase = 0;
    int kv_it = 0, att_it = 0, ring_base = 0;
    __shared__ int ord[kThrottleTasks];  // this queue's linear tiles started so far, per task
    if (lane == 0)
      for (int i = 0; i < kThrottleTasks; ++i) ord[i] = 0;
    __syncwarp();
    for (int idx = 0; idx < n_tasks; ++idx) {
      Rec r;
      load_rec(p, idx, sm, r);
      const int* cfg = p.cfg + r.task_id * kCfgInts;
      const int op = __ldg(cfg);
      const int cls = op_class(op);
      if (cls == CLS_ELEM) continue;
      if (last_cls >= 0 && cls != last_cls) named_bar(1, kTensorThreads);
      last_cls = cls;
      const unsigned long long t_fetch = p.trace ? globaltimer_ns() : 0;
      const bool waited = __any_sync(0xffffffffu, wait_deps(p, r, rank, 1, lane, 32));
      __syncwarp();
      if (p.trace && lane == 0) {
        unsigned long long* tr = trace_at(p, qrow, idx);
        tr[0] = t_fetch;
        tr[1] = globaltimer_ns();
      }
      if (cls == CLS_LINEAR) {
        const int m = r.d0[0], k = r.d1[0], n = r.d0[1];
        (void)m;
        const int ntn = (n + 255) / 256;
        const int r0 = (r.tile / ntn) * 256, c0 = (r.tile % ntn) * 256;
        const CUtensorMap* ma = maps + __ldg(cfg + 5);
        const CUtensorMap* mb = maps + __ldg(cfg + 6);
        if (lane == 0) {
          if (p.lin_started && r.task_id < kThrottleTasks) {
            const int kk = ord[r.task_id]++;
            unsigned* ctr = p.lin_started + rank * kThrottleTasks + r.task_id;
            const long long need = static_cast<long long>(kk) * p.num_sms - p.num_sms / 2;
            if (need > 0) {
              const unsigned long long t0 = globaltimer_ns();
              while (true) {
                unsigned v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (static_cast<long long>(v) >= need) break;
                __nanosleep(64);
                if (globaltimer_ns() - t0 > p.timeout_ns) {
                  atomicCAS(reinterpret_cast<unsigned long long*>(p.err[rank]), 0ull, 0x7100000ull | r.task_id);
                  break;
                }
              }
            }
            atomicAdd(ctr, 1u);
          }
          if (waited) fence_proxy_async_global();
          for (int kb = 0; kb < k / 64; ++kb) {
            mbar_wait(&empty_bar[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kStage;
            mbar_arrive_expect_tx(&full_bar[stage], kStage);
            tma_load_2d(sa, ma, &full_bar[stage], kb * 64, r0);
            tma_load_2d(sa + kHalfBox, ma, &full_bar[stage], kb * 64, r0 + 128);
            tma_load_2d(sa + kAStage, mb, &full_bar[stage], kb * 64, c0);
            if (++stage == kRing) { stage = 0; phase ^= 1; }
          }
        }
        __syncwarp();
      } else {
        const AttnGeom a = attn_geom(cfg, r);
        const CUtensorMap* mq = maps + __ldg(cfg + 5);
        if (lane == 0) {
          if (waited) fence_proxy_async_global();
          mbar_wait(q_empty, (att_it & 1) ^ 1);
          mbar_arrive_expect_tx(q_full, a.np * 2 * kHalfBox);
          for (int t = 0; t < a.np; ++t) {
            tma_load_3d_l(smem + kQOff + t * 2 * kHalfBox, mq, q_full, 0, a.h + t, a.q_row0);
            tma_load_3d_l(smem + kQOff + t * 2 * kHalfBox + kHalfBox, mq, q_full, 64, a.h + t, a.q_row0);
          }
          for (int c = 0; c < 2 * a.n_kv; ++c) {  // K_j = 2j, V_j = 2j + 1
            const int j = c >> 1, kv = c & 1;
            const int gc = ring_base + c, sl = gc % kKVSlots;
            mbar_wait(&kv_empty[sl], ((gc / kKVSlots) & 1) ^ 1);
            uint8_t* dst = smem + kKVOff + sl * kKVSlot;
            const int row = (a.kv0 + j) * 128;
            const int head = a.hq + kv * a.hkv + a.g;
            mbar_arrive_expect_tx(&kv_full[sl], kKVSlot);
            tma_load_3d_l(dst, mq, &kv_full[sl], 0, head, row);
            tma_load_3d_l(dst + kHalfBox, mq, &kv_full[sl], 64, head, row);
          }
        }
        __syncwarp();
        kv_it += a.n_kv;
        ring_base += 2 * a.n_kv;
        ++att_it;
      }
    }
  } else if (warp == 1) {
    // =========================================================== MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int lin_it = 0, kv_it = 0, att_it = 0, ring_base = 0;
    constexpr uint32_t idesc_lin = umma_idesc_bf16(128, 256);
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128);
    constexpr uint32_t idesc_pv = umma_idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
    const uint32_t t_o = tmem + 256;
    for (int idx = 0; idx < n_tasks; ++idx) {
      Rec r;
      load_rec(p, idx, sm, r);
      const int* cfg = p.cfg + r.task_id * kCfgInts;
      const int op = __ldg(cfg);
      const int cls = op_class(op);
      if (cls == CLS_ELEM) continue;
      if (last_cls >= 0 && cls != last_cls) named_bar(1, kTensorThreads);
      last_cls = cls;
      if (cls == CLS_LINEAR) {
        // two M=128 halves per 256x256 tile share each B stage; half h accumulates in
        // TMEM columns [256h, 256h + 256) with its own full/empty pair.  At tile edges
        // half 1 trails by kLag k-blocks so the epilogue drains half 0 while half 1
        // finishes, and the next tile's half 0 starts while half 1 drains.
        const int nkb = r.d1[0] / 64;
        const uint32_t tph = lin_it & 1;
        const bool lagged = nkb >= 2 * kLag + 1;
        auto issue = [&](int st, int h, int kb) {
          const uint32_t a_lo = desc_lo_k(smem_u32(smem + st * kStage) + h * kHalfBox);
          const uint32_t b_lo = desc_lo_k(smem_u32(smem + st * kStage) + kAStage);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tmem + h * 256, desc_from_lo(a_lo + kk * 2), desc_from_lo(b_lo + kk * 2), idesc_lin,
                      (kb | kk) != 0);
        };
        mbar_wait(&tempty[0], tph ^ 1);
        if (!lagged) mbar_wait(&tempty[1], tph ^ 1);
        tc_fence_after();
        const int s0 = stage;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const bool head = lagged && kb < kLag;
          const bool tail = lagged && kb >= nkb - kLag;
          if (lane == 0) {
            issue(stage, 0, kb);
            if (!head && !tail) {
              issue(stage, 1, kb);
              umma_commit(&empty_bar[stage]);
            }
          }
          __syncwarp();
          if (lagged && kb == kLag - 1) {
            mbar_wait(&tempty[1], tph ^ 1);
            tc_fence_after();
            if (lane == 0)
              for (int j = 0; j < kLag; ++j) {
                const int st = (s0 + j) % kRing;
                issue(st, 1, j);
                umma_commit(&empty_bar[st]);
              }
            __syncwarp();
          }
          if (++stage == kRing) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) {
          umma_commit(&tfull[0]);
          if (lagged)
            for (int j = nkb - kLag; j < nkb; ++j) {
              const int st = (s0 + j) % kRing;
              issue(st, 1, j);
              umma_commit(&empty_bar[st]);
            }
          umma_commit(&tfull[1]);
        }
        __syncwarp();
        ++lin_it;
      } else {
        // per head stream t: S_t(0); then for each key tile j: PV_t(j) (A = P_t from TMEM)
        // and S_t(j+1) into the same columns -- in that order on the in-order tensor pipe,
        // so S_t(j+1) overwrites P_t(j) only after PV_t(j) read it and "S_t(j+1) complete"
        // implies "PV_t(j) complete".  With two heads the softmax of one head overlaps the
        // other head's PV + QK^T.
        const AttnGeom a = attn_geom(cfg, r);
        const int n = a.n_kv, np = a.np;
        mbar_wait(q_full, att_it & 1);
        mbar_wait(o_empty, (att_it & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          auto issue_s = [&](int t, int sl) {
            const uint32_t qa = desc_lo_k(smem_u32(smem + kQOff + t * 2 * kHalfBox));
            const uint32_t kb = desc_lo_k(smem_u32(smem + kKVOff + sl * kKVSlot));
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t off = (kk >> 2) * (kHalfBox >> 4) + (kk & 3) * 2;
              umma_bf16(tmem + t * 128, desc_from_lo(qa + off), desc_from_lo(kb + off), idesc_s, kk != 0);
            }
            umma_commit(&s_full[t]);
          };
          {
            const int gc = ring_base, sl = gc % kKVSlots;
            mbar_wait(&kv_full[sl], (gc / kKVSlots) & 1);
            tc_fence_after();
            for (int t = 0; t < np; ++t) issue_s(t, sl);
            umma_commit(&kv_empty[sl]);
          }
          for (int j = 0; j < n; ++j) {
            const int gv = ring_base + 2 * j + 1, vs = gv % kKVSlots;
            const int gk = ring_base + 2 * j + 2, ks = gk % kKVSlots;
            mbar_wait(&kv_full[vs], (gv / kKVSlots) & 1);
            if (j + 1 < n) mbar_wait(&kv_full[ks], (gk / kKVSlots) & 1);
            for (int t = 0; t < np; ++t) {
              mbar_wait(&p_full[t], (kv_it + j) & 1);
              tc_fence_after();
              const uint32_t vb = desc_lo_mn(smem_u32(smem + kKVOff + vs * kKVSlot), kHalfBox);
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                umma_bf16_ts(t_o + t * 128, tmem + t * 128 + kk * 8, desc_from_lo(vb + kk * (2048 >> 4)),
                             idesc_pv, (j | kk) != 0);
              if (j + 1 < n) issue_s(t, ks);
              else umma_commit(&o_ready[t]);
            }
            umma_commit(&kv_empty[vs]);
            if (j + 1 < n) umma_commit(&kv_empty[ks]);
          }
          umma_commit(q_empty);
        }
        __syncwarp();
        kv_it += n;
        ring_base += 2 * n;
        ++att_it;
      }
    }
  } else {
    // =========================================================== epilogue / softmax / elementwise
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;                 // TMEM lane = tile row
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    // warps 2-5 drain the tensor tasks; warps 6-7 run the elementwise tasks, so a
    // norm / allreduce never holds the accumulator drain (and with it the MMA) back
    const bool elem_grp = warp >= 6;
    const int gthreads = elem_grp ? 64 : 128;
    const int gbar = elem_grp ? 3 : 2;
    const int et = threadIdx.x - (elem_grp ? 192 : 64);  // thread index in the group
    const int nw = gthreads / 32;
    const int ew = warp - (elem_grp ? 6 : 2);            // warp index in the group
    int lin_it = 0, kv_it = 0, att_it = 0;
    for (int idx = 0; idx < n_tasks; ++idx) {
      Rec r;
      load_rec(p, idx, sm, r);
      const int* cfg = p.cfg + r.task_id * kCfgInts;
      const int op = __ldg(cfg);
      const int cls = op_class(op);
      if (cls != CLS_ELEM) {
        if (elem_grp) continue;
        if (last_cls >= 0 && cls != last_cls) named_bar(1, kTensorThreads);
        last_cls = cls;
      } else if (!elem_grp) {
        continue;
      }
      if (op == OP_LINEAR) {
        const int m = r.d0[0], n = r.d0[1];
        const int epi = __ldg(cfg + 4);
        const int out_slot = __ldg(cfg + 14);
        const int ntn = (n + 255) / 256;
        const int c0 = (r.tile % ntn) * 256;
        const int ldy = out_slot == 3 ? r.d1[3] : r.d1[2];
        uint16_t* y = reinterpret_cast<uint16_t*>(my_base + (out_slot == 3 ? r.off[3] : r.off[2]));
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
        mbar_wait(&tfull[hf], lin_it & 1);
        tc_fence_after();
        const uint32_t t_acc = tmem + lane_off + hf * 256;
        const int grow = (r.tile / ntn) * 256 + hf * 128 + row;
        const bool row_ok = grow < m;
        if (epi == EPI_SILU_MUL) {
          // tile columns [0,128) = gate rows, [128,256) = matching up rows -> 128 outputs
          uint16_t* dst = y + static_cast<long long>(grow) * ldy + (c0 >> 1);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t gv[32], uv[32];
            tmem_ld_32x32b_x32(t_acc + c * 32, gv);
            tmem_ld_32x32b_x32(t_acc + 128 + c * 32, uv);
            tmem_ld_wait();
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float g = __uint_as_float(gv[i]);
              o[i] = g / (1.f + __expf(-g)) * __uint_as_float(uv[i]);
            }
            if (row_ok) store_bf16x32(dst + c * 32, o, min(32, ldy - (c0 >> 1) - c * 32));
          }
        } else if (epi == EPI_ROPE) {
          const int seq = __ldg(cfg + 9);
          const int rope_cols = __ldg(cfg + 13);
          const float* rope = reinterpret_cast<const float*>(my_base + r.off[2]);
          const float* cs = rope + static_cast<long long>((row_ok ? grow : 0) % seq) * 128;
          uint16_t* dst = y + static_cast<long long>(grow) * ldy + c0;
#pragma unroll 1
          for (int hh = 0; hh < 2; ++hh) {
            const bool rot = c0 + hh * 128 < rope_cols;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
              uint32_t x1[32], x2[32];
              tmem_ld_32x32b_x32(t_acc + hh * 128 + c * 32, x1);
              tmem_ld_32x32b_x32(t_acc + hh * 128 + 64 + c * 32, x2);
              tmem_ld_wait();
              float o1[32], o2[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                const float a1 = __uint_as_float(x1[i]), a2 = __uint_as_float(x2[i]);
                const float co = rot ? __ldg(cs + c * 32 + i) : 1.f;
                const float si = rot ? __ldg(cs + 64 + c * 32 + i) : 0.f;
                o1[i] = rot ? a1 * co - a2 * si : a1;
                o2[i] = rot ? a2 * co + a1 * si : a2;
              }
              if (row_ok) {
                const int cb = c0 + hh * 128 + c * 32;
                store_bf16x32(dst + hh * 128 + c * 32, o1, min(32, ldy - cb));
                store_bf16x32(dst + hh * 128 + 64 + c * 32, o2, min(32, ldy - cb - 64));
              }
            }
          }
        } else {
          uint16_t* dst = y + static_cast<long long>(grow) * ldy + c0;
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_acc + c * 32, v);
            tmem_ld_wait();
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(v[i]);
            if (row_ok && c0 + c * 32 < ldy) store_bf16x32(dst + c * 32, o, min(32, ldy - c0 - c * 32));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[hf]);
        }
        ++lin_it;
      } else if (op == OP_ATTENTION) {
        const AttnGeom a = attn_geom(cfg, r);
        const int n = a.n_kv, np = a.np;
        const int causal = __ldg(cfg + 12);
        const float scale_log2 = __int_as_float(__ldg(cfg + 10)) * 1.4426950408889634f;
        float mrow[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
        for (int j = 0; j < n; ++j) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (t >= np) break;
            const uint32_t t_s = tmem + lane_off + t * 128;
            const uint32_t t_ot = tmem + lane_off + 256 + t * 128;
            mbar_wait(&s_full[t], (kv_it + j) & 1);
            tc_fence_after();
            uint32_t sv[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(t_s + c * 32, sv[c]);
            tmem_ld_wait();
            if (causal && j == n - 1) {  // diagonal tile only (warp-uniform branch)
#pragma unroll
              for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (c * 32 + i > row) sv[c][i] = __float_as_uint(-INFINITY);
            }
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(sv[c][i]));
            const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
            // lazy rescale: the running max may lag the true max by up to 2^8
            float alpha = 1.f;
            if (mt > mrow[t] + kLazyRescale) {
              alpha = ex2(mrow[t] - mt);
              mrow[t] = mt;
            }
            // O_t is stable (S_t(j) complete => PV_t(j-1) complete); rescale before P_t(j)
            if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
              for (int c = 0; c < 4; ++c) {
                uint32_t ov[32];
                tmem_ld_32x32b_x32(t_ot + c * 32, ov);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
                tmem_st_x32(t_ot + c * 32, ov);
              }
            }
            float sacc[4] = {0.f, 0.f, 0.f, 0.f};
            // P packed in place: pair (2i, 2i+1) of chunk c -> sv[c / 2][(c % 2) * 16 + i]
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float p0 = ex2(fmaf(__uint_as_float(sv[c][2 * i]), scale_log2, -mrow[t]));
                const float p1 = ex2(fmaf(__uint_as_float(sv[c][2 * i + 1]), scale_log2, -mrow[t]));
                sacc[i & 3] += p0 + p1;
                sv[c >> 1][(c & 1) * 16 + i] = pack_bf16x2(p0, p1);
              }
            l[t] = l[t] * alpha + ((sacc[0] + sacc[1]) + (sacc[2] + sacc[3]));
            tmem_st_x32(t_s, sv[0]);
            tmem_st_x32(t_s + 32, sv[1]);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[t]);
          }
        }
        const int ldo = r.d1[1];
        const bool row_ok = a.q_row0 + row < r.d0[1];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (t >= np) break;
          mbar_wait(&o_ready[t], att_it & 1);
          tc_fence_after();
          const float inv = 1.f / l[t];
          uint16_t* dst = reinterpret_cast<uint16_t*>(my_base + r.off[1]) +
                          static_cast<long long>(a.q_row0 + row) * ldo + (a.h + t) * 128;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(tmem + lane_off + 256 + t * 128 + c * 32, ov);
            tmem_ld_wait();
            float o[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(ov[i]) * inv;
            if (row_ok) store_bf16x32(dst + c * 32, o, 32);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_empty);
        kv_it += n;
        ++att_it;
      } else {
        // ------------------------------------------------ elementwise tasks (warps 6-7)
        // two-shot allreduce: row block b is reduced once, by rank b % world, which
        // P2P-stores the result into every PE and releases the tile on every PE's
        // scoreboard; the other ranks skip the task (no release of their own)
        const bool two_shot = op == OP_ALLREDUCE_RES && p.world > 1 && __ldg(cfg + 13) != 0;
        if (two_shot && r.tile % p.world != rank) continue;
        const int npe = op == OP_ALLREDUCE_RES ? p.world : 1;
        const int nout = two_shot ? p.world : 1;  // destinations of the outputs
        const unsigned long long t_fetch = p.trace ? globaltimer_ns() : 0;
        wait_deps(p, r, rank, npe, et, gthreads);
        named_bar(gbar, gthreads);
        if (p.trace && et == 0) {
          unsigned long long* tr = trace_at(p, qrow, idx);
          tr[0] = t_fetch;
          tr[1] = globaltimer_ns();
        }
        const int br = __ldg(cfg + 3);
        if (op == OP_RMSNORM) {
          // one warp per row; 8 x 16-byte loads in flight per lane, second pass hits L1/L2
          const int rows = r.d0[0], cols = r.d1[0];
          const float eps = __int_as_float(__ldg(cfg + 11));
          const uint16_t* x = reinterpret_cast<const uint16_t*>(my_base + r.off[0]);
          const uint16_t* g = reinterpret_cast<const uint16_t*>(my_base + r.off[1]);
          uint16_t* y = reinterpret_cast<uint16_t*>(my_base + r.off[2]);
          const int r0 = r.tile * br, r1 = min(r0 + br, rows);
          prefetch_l2(x + static_cast<long long>(r0) * cols, static_cast<long long>(r1 - r0) * cols * 2, et, gthreads);
          constexpr int U = 8;
          for (int rr = r0 + ew; rr < r1; rr += nw) {
            const uint16_t* xr = x + static_cast<long long>(rr) * cols;
            float ss = 0.f;
            for (int c0 = lane * 8; c0 < cols; c0 += 256 * U) {
              uint4 v[U];
#pragma unroll
              for (int u = 0; u < U; ++u)
                v[u] = c0 + u * 256 < cols ? *reinterpret_cast<const uint4*>(xr + c0 + u * 256)
                                           : make_uint4(0, 0, 0, 0);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  const float a0 = bf16lo(w[i]), a1 = bf16hi(w[i]);
                  ss += a0 * a0 + a1 * a1;
                }
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const float rstd = rsqrtf(ss / static_cast<float>(cols) + eps);
            uint16_t* yr = y + static_cast<long long>(rr) * cols;
            for (int c0 = lane * 8; c0 < cols; c0 += 256 * U) {
              uint4 v[U], gv[U];
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (c0 + u * 256 < cols) {
                  v[u] = *reinterpret_cast<const uint4*>(xr + c0 + u * 256);
                  gv[u] = __ldg(reinterpret_cast<const uint4*>(g + c0 + u * 256));
                }
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (c0 + u * 256 < cols) {
                  const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                  const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
                  uint32_t o[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i)
                    o[i] = pack_bf16x2(bf16lo(w[i]) * rstd * bf16lo(gw[i]), bf16hi(w[i]) * rstd * bf16hi(gw[i]));
                  *reinterpret_cast<uint4*>(yr + c0 + u * 256) = make_uint4(o[0], o[1], o[2], o[3]);
                }
            }
          }
        } else if (op == OP_ALLREDUCE_RES && __ldg(cfg + 15) == 0) {
          // y = (x_0 + x_1 + ... + x_{w-1}) + res, fp32 in ascending PE order, bf16 out;
          // 8 chunks of 8 elements per thread per round (loads of all PEs in flight)
          const int rows = r.d0[0], cols = r.d1[0];
          const int r0 = r.tile * br, r1 = min(r0 + br, rows);
          const long long lo = static_cast<long long>(r0) * cols / 8, hi = static_cast<long long>(r1) * cols / 8;
          const uint4* res = reinterpret_cast<const uint4*>(my_base + r.off[1]);
          uint4* y = reinterpret_cast<uint4*>(my_base + r.off[2]);
          for (int pe = 0; pe < p.world; ++pe)
            prefetch_l2(reinterpret_cast<const uint4*>(p.base[pe] + r.off[0]) + lo, (hi - lo) * 16, et, gthreads);
          prefetch_l2(res + lo, (hi - lo) * 16, et, gthreads);
          constexpr int U = 8;
          for (long long i0 = lo + et; i0 < hi; i0 += gthreads * U) {
            float acc[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
            for (int pe = 0; pe < p.world; ++pe) {
              const uint4* src = reinterpret_cast<const uint4*>(p.base[pe] + r.off[0]);
              uint4 v[U];
#pragma unroll
              for (int u = 0; u < U; ++u) v[u] = i0 + u * gthreads < hi ? src[i0 + u * gthreads] : make_uint4(0, 0, 0, 0);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  acc[u][2 * e] += bf16lo(w[e]);
                  acc[u][2 * e + 1] += bf16hi(w[e]);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const long long i = i0 + u * gthreads;
              if (i < hi) {
                const uint4 rv = res[i];
                const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  o[e] = pack_bf16x2(acc[u][2 * e] + bf16lo(w[e]), acc[u][2 * e + 1] + bf16hi(w[e]));
                const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
                if (nout == 1) {
                  y[i] = ov;
                } else {
                  for (int q = 0; q < nout; ++q)
                    reinterpret_cast<uint4*>(p.base[(rank + q) % nout] + r.off[2])[i] = ov;
                }
              }
            }
          }
        } else if (op == OP_ALLREDUCE_RES) {
          // fused with the following RMSNorm: one warp per row, y = sum_pe x_pe + res
          // (fp32, ascending PE, bf16), then yn = y * rsqrt(mean(y^2) + eps) * g
          const int rows = r.d0[0], cols = r.d1[0];
          const int r0 = r.tile * br, r1 = min(r0 + br, rows);
          const float eps = __int_as_float(__ldg(cfg + 11));
          const uint16_t* g = reinterpret_cast<const uint16_t*>(
              my_base + (static_cast<long long>(__ldg(cfg + 15) - 1) << 4));
          const long long lo = static_cast<long long>(r0) * cols, n_el = static_cast<long long>(r1 - r0) * cols;
          for (int pe = 0; pe < p.world; ++pe)
            prefetch_l2(reinterpret_cast<const uint16_t*>(p.base[pe] + r.off[0]) + lo, n_el * 2, et, gthreads);
          prefetch_l2(reinterpret_cast<const uint16_t*>(my_base + r.off[1]) + lo, n_el * 2, et, gthreads);
          constexpr int U = 4;
          for (int rr = r0 + ew; rr < r1; rr += nw) {
            const long long rb = static_cast<long long>(rr) * cols;
            const uint16_t* res = reinterpret_cast<const uint16_t*>(my_base + r.off[1]) + rb;
            uint16_t* y = reinterpret_cast<uint16_t*>(my_base + r.off[2]) + rb;
            uint16_t* yn = reinterpret_cast<uint16_t*>(my_base + r.off[3]) + rb;
            float ss = 0.f;
            for (int c0 = lane * 8; c0 < cols; c0 += 256 * U) {
              float acc[U][8];
#pragma unroll
              for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[u][e] = 0.f;
              for (int pe = 0; pe < p.world; ++pe) {
                const uint16_t* src = reinterpret_cast<const uint16_t*>(p.base[pe] + r.off[0]) + rb;
                uint4 v[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                  v[u] = c0 + u * 256 < cols ? *reinterpret_cast<const uint4*>(src + c0 + u * 256)
                                             : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                  const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    acc[u][2 * e] += bf16lo(w[e]);
                    acc[u][2 * e + 1] += bf16hi(w[e]);
                  }
                }
              }
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int c = c0 + u * 256;
                if (c < cols) {
                  const uint4 rv = *reinterpret_cast<const uint4*>(res + c);
                  const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
                  uint32_t o[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    o[e] = pack_bf16x2(acc[u][2 * e] + bf16lo(w[e]), acc[u][2 * e + 1] + bf16hi(w[e]));
                    const float a0 = bf16lo(o[e]), a1 = bf16hi(o[e]);
                    ss += a0 * a0 + a1 * a1;
                  }
                  const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
                  *reinterpret_cast<uint4*>(y + c) = ov;
                  for (int q = 1; q < nout; ++q)
                    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.base[(rank + q) % nout] + r.off[2]) +
                                              rb + c) = ov;
                }
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
            const float rstd = rsqrtf(ss / static_cast<float>(cols) + eps);
            for (int c0 = lane * 8; c0 < cols; c0 += 256 * U) {
              uint4 v[U], gv[U];
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (c0 + u * 256 < cols) {
                  v[u] = *reinterpret_cast<const uint4*>(y + c0 + u * 256);  // this lane's own stores
                  gv[u] = __ldg(reinterpret_cast<const uint4*>(g + c0 + u * 256));
                }
#pragma unroll
              for (int u = 0; u < U; ++u)
                if (c0 + u * 256 < cols) {
                  const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
                  const uint32_t gw[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
                  uint32_t o[4];
#pragma unroll
                  for (int i = 0; i < 4; ++i)
                    o[i] = pack_bf16x2(bf16lo(w[i]) * rstd * bf16lo(gw[i]), bf16hi(w[i]) * rstd * bf16hi(gw[i]));
                  const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
                  *reinterpret_cast<uint4*>(yn + c0 + u * 256) = ov;
                  for (int q = 1; q < nout; ++q)
                    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.base[(rank + q) % nout] + r.off[3]) +
                                              rb + c0 + u * 256) = ov;
                }
            }
          }
        }
      }
      // every task ends with its scoreboard release by its group
      named_bar(gbar, gthreads);
      if (et == 0) {
        if (op == OP_ALLREDUCE_RES && p.world > 1 && __ldg(cfg + 13) != 0)
          for (int q = 0; q < p.world; ++q) release_flag(p, rank, r, (rank + q) % p.world);
        else
          release_flag(p, rank, r, rank);
        if (p.trace) {
          unsigned long long* tr = trace_at(p, qrow, idx);
          tr[2] = globaltimer_ns();
          tr[3] = (static_cast<unsigned long long>(r.task_id) << 32) | static_cast<unsigned>(r.tile);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}

// spec (8 x int64): heap offset, ndims (2|3), dims[3] (innermost first), box[3]; bf16, 128B swizzle
int encode_spec(CUtensorMap* m, uint8_t* base, const int64_t* s) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const int nd = static_cast<int>(s[1]);
  if (nd != 2 && nd != 3) return fail(TF_ERR_INVALID, "tensor map spec needs 2 or 3 dims");
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  for (int i = 0; i < nd; ++i) {
    dims[i] = static_cast<cuuint64_t>(s[2 + i]);
    box[i] = static_cast<cuuint32_t>(s[5 + i]);
  }
  strides[0] = dims[0] * 2;
  if (nd == 3) strides[1] = dims[0] * dims[1] * 2;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, nd, base + s[0], dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TF_ERR_INVALID, "layer tensor map encode failed (code " + std::to_string(r) + ")");
  return TF_OK;
}

struct MapCache {
  std::string key;
  void* dev = nullptr;
};
std::mutex g_map_mu;
std::map<std::pair<const tf_team*, int>, MapCache> g_maps;

}  // namespace

// drop the tensor-map tables cached for a team (called by tf_team_destroy)
void layer_release_team(const tf_team* t) {
  std::lock_guard<std::mutex> lk(g_map_mu);
  for (auto it = g_maps.begin(); it != g_maps.end();) {
    if (it->first.first == t) {
      if (it->second.dev) cudaFree(it->second.dev);
      it = g_maps.erase(it);
    } else {
      ++it;
    }
  }
}
}  // namespace tf

using tf::fail;

extern "C" int tf_layer_megakernel_run(tf_team* t, int rank, const tf_layer_args* a, void* stream) {
  if (!t || !a) return fail(TF_ERR_INVALID, "NULL argument");
  if (a->num_sms < 1) return fail(TF_ERR_INVALID, "num_sms must be >= 1");
  if (a->num_maps < 0 || (a->num_maps > 0 && !a->map_specs))
    return fail(TF_ERR_INVALID, "bad tensor map specs");
  int first = 0, nranks = t->world, fixed = -1;
  if (t->ipc) {
    if (rank != t->my_rank) return fail(TF_ERR_INVALID, "IPC team: rank must be this process's rank");
    first = rank;
    nranks = 1;
    fixed = rank;
  } else {
    if (rank >= 0) {
      if (t->world != 1 || rank != 0)
        return fail(TF_ERR_CONFIG, "local team: pass rank -1 (all ranks co-scheduled in one launch)");
    }
    for (int pe = 1; pe < t->world; ++pe)
      if (t->pes[pe].device != t->pes[0].device)
        return fail(TF_ERR_CONFIG, "the co-scheduled megakernel needs every PE on one device");
  }
  tf::DeviceGuard guard(t->pes[first].device);
  const int grid = nranks * a->num_sms;
  if (grid > tf::num_sms_of_current_device())
    return fail(TF_ERR_CONFIG, "ranks * num_sms CTAs must be co-resident (<= SM count)");
  // tensor maps per launched rank, cached per (team, rank) by spec content
  std::string key(reinterpret_cast<const char*>(a->map_specs),
                  static_cast<size_t>(a->num_maps) * 8 * sizeof(int64_t));
  for (int rr = 0; rr < nranks; ++rr)  // a recycled team address must not reuse stale maps
    key.append(reinterpret_cast<const char*>(&t->pes[first + rr].base), sizeof(void*));
  void* dmaps = nullptr;
  {
    std::lock_guard<std::mutex> lk(tf::g_map_mu);
    auto& mc = tf::g_maps[{t, rank}];
    if (mc.dev == nullptr || mc.key != key) {
      std::vector<CUtensorMap> host(static_cast<size_t>(nranks) * std::max(a->num_maps, 1));
      for (int rr = 0; rr < nranks; ++rr)
        for (int i = 0; i < a->num_maps; ++i) {
          int rc = tf::encode_spec(&host[static_cast<size_t>(rr) * a->num_maps + i],
                                   t->pes[first + rr].base, a->map_specs + 8 * i);
          if (rc) return rc;
        }
      if (mc.dev) cudaFree(mc.dev);
      mc.dev = nullptr;
      TF_CUDA_TRY(cudaMalloc(&mc.dev, host.size() * sizeof(CUtensorMap)));
      TF_CUDA_TRY(cudaMemcpy(mc.dev, host.data(), host.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
      mc.key = key;
    }
    dmaps = mc.dev;
  }
  tf::LayerParams p{};
  p.queues = a->queues;
  p.counts = a->counts;
  p.deps = a->deps;
  p.cfg = a->layer_cfg;
  p.maps = static_cast<const CUtensorMap*>(dmaps);
  p.num_maps = a->num_maps;
  p.num_sms = a->num_sms;
  p.max_tiles = a->max_tiles;
  p.fixed_rank = fixed;
  p.world = t->world;
  p.flag_base = a->flag_base;
  p.epoch = a->epoch ? a->epoch : 1;
  p.timeout_ns = a->timeout_ns ? a->timeout_ns : t->timeout_ns;
  for (int pe = 0; pe < t->world; ++pe) {
    p.base[pe] = t->pes[pe].base;
    p.sig[pe] = t->pes[pe].sig;
    p.err[pe] = t->err_word(pe);
  }
  p.trace = reinterpret_cast<unsigned long long*>(a->trace);
  p.slots = a->trace_slots;
  {
    static const bool thr_on = [] {
      const char* e = getenv("TF_LAYER_THROTTLE");
      return !e || atoi(e) != 0;
    }();
    if (thr_on) {
      int cur = 0;
      cudaGetDevice(&cur);
      static std::mutex thr_mu;
      static std::map<int, unsigned*> thr_bufs;
      unsigned* buf = nullptr;
      {
        std::lock_guard<std::mutex> lk(thr_mu);
        auto it = thr_bufs.find(cur);
        if (it == thr_bufs.end()) {
          TF_CUDA_TRY(cudaMalloc(&buf, static_cast<size_t>(tf::kMaxWorld) * tf::kThrottleTasks * 4));
          thr_bufs[cur] = buf;
        } else {
          buf = it->second;
        }
      }
      TF_CUDA_TRY(cudaMemsetAsync(buf, 0, static_cast<size_t>(nranks) * tf::kThrottleTasks * 4,
                                  static_cast<cudaStream_t>(stream)));
      p.lin_started = buf;
    }
  }
  if (grid == a->num_sms) {  // one rank's queues per launch: rank them by die (TF_LAYER_DIE=0 off)
    static const bool die_on = [] {
      const char* e = getenv("TF_LAYER_DIE");
      return !e || atoi(e) != 0;
    }();
    int cur = 0;
    cudaGetDevice(&cur);
    unsigned long long* slot = nullptr;
    const uint8_t* tab = die_on ? tf::sm_die_table(cur, &slot) : nullptr;
    if (tab) {
      p.sm_die = tab;
      p.die_ctr = slot;
    }
  }
  static uint64_t attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    TF_CUDA_TRY(cudaFuncSetAttribute(tf::layer_megakernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tf::kLayerSmem));
    attr_done |= 1ull << dev;
  }
  tf::layer_megakernel<<<grid, tf::kLThreads, tf::kLayerSmem, static_cast<cudaStream_t>(stream)>>>(p);
  TF_CUDA_TRY(cudaGetLastError());
  return TF_OK;
}
