// Persistent, warp-specialised tcgen05 GEMM for sm_100a — the core tile of the
// fused collectives.
//
//   C[m, n] = sum_k A[m, k] * B[n, k]      (A, B bf16, K-major; fp32 in TMEM)
//
// This is the tile body of the reference's workers (ovs/kernels/ag_gemm.py:93-94,
// gemm_rs.py:123, 151) re-done for Blackwell:
//   warp 0      TMA producer: per tile, optionally acquire-waits the AllGather
//               arrival flags of the row chunks the tile covers
//               (ag_gemm.py:87-90), then streams 128x64 A and BNx64 B boxes
//               (128-byte swizzle) into a STAGES-deep smem ring.
//   warp 1      owns TMEM (2 x BN fp32 columns = double-buffered accumulator) and
//               issues tcgen05.mma (M=128, N=BN, K=16) from one lane.
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns, convert, store.  In
//               scatter mode each row slice goes straight to its owner's slot
//               buffer (gemm_rs.py:152-161) and a release-add bumps the owner's
//               per-row-tile arrival counter.
// Tile order is the reference's persistent stride (ag_gemm.py:81): CTA s runs
// steps s, s+grid, ...; each step -> swizzle_2d(group_m) -> tile_map[pid_m].
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "tf_internal.h"
#include "tf_ptx.cuh"

namespace tf {

namespace {

// K-major SW128 descriptor = (low word, constant high word): one add per MMA operand
constexpr uint32_t kDescHiK = (1024 >> 4) | (1u << (46 - 32)) | (2u << (61 - 32));
__device__ __forceinline__ uint64_t desc_from_lo(uint32_t lo) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(kDescHiK));
  return d;
}
__device__ __forceinline__ uint32_t desc_lo_k(uint32_t addr) { return ((addr & 0x3FFFF) >> 4) | (1u << 16); }


constexpr int BK = 64;                 // 64 bf16 = 128 B = one swizzle atom row
constexpr bool kDefaultMulticast = false;  // 4-CTA multicast clusters (TF_GEMM_MC overrides)
constexpr int kDefaultDieMode = 1;         // die-ranked cluster ids (TF_GEMM_DIE overrides)
#ifndef TF_GEMM_EARLY_RELEASE
#define TF_GEMM_EARLY_RELEASE 1
#endif
constexpr bool kEarlyRelease = TF_GEMM_EARLY_RELEASE;  // epilogue frees TMEM before its stores
#ifndef TF_GEMM_RELAXED_ARRIVE
#define TF_GEMM_RELAXED_ARRIVE 1
#endif
constexpr bool kRelaxedArrive = TF_GEMM_RELAXED_ARRIVE;  // "accumulator free" without MEMBAR.GPU
#ifndef TF_GEMM_LAG
#define TF_GEMM_LAG 2                  // k-blocks the second M-half trails at tile edges
#endif
constexpr int UMMA_K = 16;
constexpr int kThreads = 192;          // 6 warps
constexpr int kEpiWarp0 = 2;

struct KParams {
  int m, n, k;
  int num_pid_m, num_pid_n, group_m;
  int num_kb;
  const int32_t* tile_map;
  void* c;
  long long ldc;
  int vec_ok;                         // 16-byte aligned rows and n % 8 == 0
  const uint64_t* chunk_flags;
  unsigned long long epoch;
  long long rows_per_chunk;
  int rank, world;
  long long rows_per_rank;
  void* peer_slots[kMaxWorld];
  uint64_t* peer_counts[kMaxWorld];
  long long slot_ld;
  unsigned long long* err;
  unsigned long long timeout_ns;
  int dbg_skip_store;                 // experiments only (TF_DEBUG_SKIP_STORE)
  int tma_store;                      // epilogue 0: stage through smem + TMA bulk store
  // split-K tail: tiles [tail_base, num_tiles) are cut into split_s K-ranges each;
  // unit u writes fp32 partials to tile slot u of the workspace, fixed up afterwards
  int tail_base;
  int split_s;
  int total_work;
  // AllGather on the B (N-side) operand instead of A, and an N-tile permutation
  int wait_on_b;
  const int32_t* tile_map_n;
  // optional device event trace (tf_trace_enable): [count, pad, pad, pad][cap][4]
  unsigned long long* trace;
  int trace_cap;
  int trace_rank;
  int hint_a, hint_b;                 // L2 policy of the A / B TMA loads (l2_policy kinds)
  int ksnake;                         // odd waves walk K backwards (L2 reuse across waves)
  int chunks_per_rank;                // AG flags per source rank (trace payload in rank slots)
  // Grouped (MoE) mode, ag_moe.py:120-142: work item -> (slot, pid_n), slot record
  // {expert, first gathered row, rows, seg_start | seg_end << 16}; B is the stacked
  // [E * moe_n, K] expert weights.  Tiles acquire-wait the arrival counters of the
  // source ranks [seg_start, seg_end] their rows come from (ag_moe.py:131-132).
  const int4* moe_tab;
  int moe_n;
  const uint64_t* src_flags;          // [world] arrival counters (nullptr: no waits)
  unsigned long long src_target;      // value a source's counter reaches when it has landed
  // Pull engine (grouped AG): the first comm_ctas CTAs of the grid copy every peer's
  // expert-major rows into this rank's workspace, source (rank+i)%w at step i
  // (ag_moe.py:99-117), and release-add own_flags[src] when their share has landed.
  int comm_ctas;
  const uint8_t* peer_ws[kMaxWorld];
  uint8_t* own_ws;
  const int32_t* irb;                 // [world][E+1] row offsets of each expert in a source chunk
  const int32_t* dstb;                // [world][E]   gathered row of (source, expert) piece
  int n_experts;
  long long row_bytes;
  uint64_t* own_flags;
  // die-ranked cluster ids (TF_GEMM_DIE): sm_die[%smid] in {0,1}; die_ctr = this
  // launch's self-resetting counter (die-0 arrivals low word, die-1 high word).
  // die_mode 1: clusters on die 0 take the first positions of every wave; 2: also
  // reorder each full wave so its tiles in the lower half of the group's rows come
  // first (die 0 then works on those rows, die 1 on the upper half: A is not shared)
  const uint8_t* sm_die;
  unsigned long long* die_ctr;
  int die_mode;
};

// CG = CTAs per tile (1, or 2 = CTA pair with tcgen05 cta_group::2).
// MH = 128-row A blocks per CTA (1 or 2).  The tile is 128*CG*MH rows x BN columns;
// with MH = 2 each k-step issues two MMAs (one per 128*CG-row half) that share the
// B stage, so A+B operand traffic per FLOP drops by 25% (pair tile 512x256).
template <int CG, int MH, int BN>
struct Smem {
  static constexpr int kTileM = 128 * CG * MH;       // rows per tile
  static constexpr int kABlock = 128 * BK * 2;       // one 128-row A block (16 KB)
  static constexpr int kABytes = MH * kABlock;       // per CTA per stage
  static constexpr int kBRows = BN / CG;             // per CTA: BN/CG rows of B
  static constexpr int kBBytes = kBRows * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // epilogue staging: 4 warps x 2 buffers x (32 rows x 128 B), 128-byte swizzled
  static constexpr int kEpiBuf = 32 * 128;
  static constexpr int kEpiBytes = 4 * 2 * kEpiBuf;
  static constexpr int kBarBytes = 256;
  static constexpr int kMaxSmem = 232448;  // 227 KB opt-in per CTA on sm_100
  static constexpr int kFit = (kMaxSmem - 1024 - kBarBytes - kEpiBytes) / kStageBytes;
  static constexpr int kStages = kFit > 8 ? 8 : kFit;
  static constexpr int kTotal = 1024 /*align slack*/ + kStages * kStageBytes + kEpiBytes + kBarBytes;
  static constexpr int kAccCols = MH * BN;           // fp32 columns of one accumulator
  static constexpr int kAccStages = (2 * kAccCols <= 512) ? 2 : 1;
  static constexpr int kTmemCols = kAccStages * kAccCols <= 256 ? 256 : 512;
};

__device__ __forceinline__ void tile_coords(const KParams& p, int step, int& pid_m, int& pid_n) {
  // grouped order, ovs/swizzle.py:76-88
  const int per_group = p.group_m * p.num_pid_n;
  const int g = step / per_group;
  const int first_m = g * p.group_m;
  const int rows = min(p.num_pid_m - first_m, p.group_m);
  const int r = step - g * per_group;
  pid_m = first_m + r % rows;
  pid_n = r / rows;
  if (p.tile_map) pid_m = __ldg(p.tile_map + pid_m);
  if (p.tile_map_n) pid_n = __ldg(p.tile_map_n + pid_n);
}

// Geometry of one output tile: first row, row limit (exclusive), first B row.
struct TileGeo {
  int pid_m, pid_n;
  int row0, row_lim, b_row0;
  int seg;  // grouped: seg_start | seg_end << 16
};
template <bool GROUPED, int TILE_M, int BN, int NPAIR = 1>
__device__ __forceinline__ TileGeo tile_geo(const KParams& p, int step, int pair = 0) {
  TileGeo g;
  if constexpr (GROUPED) {
    // the reference's step -> (slot, pid_n) split, ag_moe.py:123-124
    const int slot = step / p.num_pid_n;
    g.pid_m = slot;
    g.pid_n = step - slot * p.num_pid_n;
    const int4 t = __ldg(p.moe_tab + slot);
    g.row0 = t.y;
    g.row_lim = t.y + t.z;
    g.b_row0 = t.x * p.moe_n + g.pid_n * BN;
    g.seg = t.w;
  } else {
    // NPAIR = 2: a work item is a pair of adjacent N tiles (one per CTA pair of the cluster)
    tile_coords(p, step, g.pid_m, g.pid_n);
    g.pid_n = g.pid_n * NPAIR + pair;
    g.row0 = g.pid_m * TILE_M;
    g.row_lim = p.m;
    g.b_row0 = g.pid_n * BN;
    g.seg = 0;
  }
  return g;
}

// Row offset, inside the tile, of this CTA's A block h: MMA h covers tile rows
// [h*128*CG, (h+1)*128*CG), CTA c of the pair supplies the c-th 128 of them.
template <int CG>
__device__ __forceinline__ int block_row(int h, uint32_t cta_rank) {
  return (h * CG + static_cast<int>(cta_rank)) * 128;
}

// die_mode 2: position o of a full wave of W steps -> step.  The wave's steps in
// order, those in the lower half of their group's rows first (stable), so die 0
// (positions [0, n0)) gets the lower rows and die 1 the upper rows of the wave.
__device__ __forceinline__ int wave_step(const KParams& p, int work, int W) {
  const int base = work - work % W;
  if (base + W > p.tail_base) return work;  // partial last wave: plain order
  const int per_group = p.group_m * p.num_pid_n;
  const int g = base / per_group;
  if ((base + W - 1) / per_group != g) return work;  // wave straddles two groups: plain order
  const int rows = min(p.num_pid_m - g * p.group_m, p.group_m);
  const int hr = (rows + 1) / 2;  // rows [0, hr) of the group are the "lower" half
  if (hr == rows) return work;
  // group-local steps are column-major: s = col * rows + row
  auto nlow_below = [&](int x) { return (x / rows) * hr + min(x % rows, hr); };
  const int a = base - g * per_group;
  const int la = nlow_below(a), nlow = nlow_below(a + W) - la;
  const int o = work - base;
  int s;
  if (o < nlow) {
    const int t = la + o;
    s = (t / hr) * rows + t % hr;
  } else {
    const int hu = rows - hr;
    const int t = (a - la) + (o - nlow);  // upper-half index
    s = (t / hu) * rows + hr + t % hu;
  }
  return g * per_group + s;
}

// Work item -> (tile step, k-block range, partial slot or -1).
__device__ __forceinline__ void decode_work(const KParams& p, int work, int& step, int& kb0,
                                            int& kb1, int& slot, int W = 0) {
  if (work < p.tail_base) {
    step = (p.die_mode == 2 && W > 0) ? wave_step(p, work, W) : work;
    kb0 = 0;
    kb1 = p.num_kb;
    slot = -1;
  } else {
    const int u = work - p.tail_base;
    const int j = u % p.split_s;
    step = p.tail_base + u / p.split_s;
    kb0 = j * p.num_kb / p.split_s;
    kb1 = (j + 1) * p.num_kb / p.split_s;
    slot = u;
  }
}

// Device trace record (4 x u64): kind|rank|cta|tile, t_start, t_end, payload.
// Kinds: 1 wait_chunks (payload = first_chunk << 32 | num_slots), 2 gemm_tile
// (payload = pid_m << 32 | pid_n), 3 epilogue (same payload).  %globaltimer ns.
__device__ __forceinline__ void trace_rec(const KParams& p, unsigned kind, int tile,
                                          unsigned long long t0, unsigned long long t1,
                                          unsigned long long payload) {
  if (!p.trace) return;
  const unsigned long long i = atomicAdd(p.trace, 1ull);
  if (i >= static_cast<unsigned long long>(p.trace_cap)) return;
  unsigned long long* e = p.trace + 4 + i * 4;
  e[0] = (static_cast<unsigned long long>(kind) << 56) |
         (static_cast<unsigned long long>(p.trace_rank & 0xFF) << 48) |
         (static_cast<unsigned long long>(blockIdx.x & 0xFFFF) << 32) | static_cast<unsigned>(tile);
  e[1] = t0;
  e[2] = t1;
  e[3] = payload;
}

// ---------------------------------------------------------------- MoE pull engine
// The reference's _pull_engine (ag_moe.py:99-117) as leading CTAs of the grouped
// GEMM launch: for step i = 1..w-1, source s = (rank+i)%w, this CTA copies its
// share (an even split of s's rows) of s's expert-major pieces from s's workspace
// into the same offsets of this rank's workspace.  Every workspace holds its own
// chunk at the gathered positions already (PRE), so a (source, expert) piece is one
// contiguous byte range at identical offsets on every PE.  One thread drives a
// ring of kPullSlots bulk copies (global -> shared -> global on the TMA engine);
// after the last piece of a source it waits for its stores to land and
// release-adds the source's arrival counter (target = comm_ctas).
constexpr int kPullPiece = 32768;
constexpr int kPullSlots = 6;

__device__ __forceinline__ void bulk_wait_read_le(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 5;" ::: "memory"); break;
  }
}

struct PieceIt {
  int e;
  long long off;     // bytes already produced from the current run
  long long lo, hi;  // this CTA's rows of the source chunk
};

__device__ __forceinline__ bool next_piece(const KParams& p, int s, PieceIt& it, const uint8_t*& src,
                                           uint8_t*& dst, uint32_t& bytes) {
  const int32_t* irb = p.irb + static_cast<long long>(s) * (p.n_experts + 1);
  while (it.e < p.n_experts) {
    const long long b0 = __ldg(irb + it.e), b1 = __ldg(irb + it.e + 1);
    const long long r0 = max(it.lo, b0), r1 = min(it.hi, b1);
    const long long run = (r1 - r0) * p.row_bytes;
    if (r1 > r0 && it.off < run) {
      const long long drow = __ldg(p.dstb + static_cast<long long>(s) * p.n_experts + it.e) + (r0 - b0);
      const long long off = drow * p.row_bytes + it.off;
      src = p.peer_ws[s] + off;
      dst = p.own_ws + off;
      bytes = static_cast<uint32_t>(min(static_cast<long long>(kPullPiece), run - it.off));
      it.off += bytes;
      return true;
    }
    if (b0 >= it.hi) break;
    ++it.e;
    it.off = 0;
  }
  it.e = p.n_experts;
  return false;
}

__device__ void moe_pull_engine(const KParams& p, uint8_t* smem) {
  if (threadIdx.x != 0) return;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kPullSlots * kPullPiece);
  for (int i = 0; i < kPullSlots; ++i) mbar_init(&bar[i], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int c = blockIdx.x, C = p.comm_ctas;
  uint8_t* dst_of[kPullSlots];
  uint32_t bytes_of[kPullSlots];
  unsigned long long nl = 0, ns = 0;  // pieces loaded / stored so far (all sources)
  for (int i = 1; i < p.world; ++i) {
    const int s = (p.rank + i) % p.world;
    const int32_t* irb = p.irb + static_cast<long long>(s) * (p.n_experts + 1);
    const long long rows = __ldg(irb + p.n_experts);
    PieceIt it;
    it.lo = rows * c / C;
    it.hi = rows * (c + 1) / C;
    it.off = 0;
    // first expert whose run ends after lo
    int lo_e = 0, hi_e = p.n_experts;
    while (lo_e < hi_e) {
      const int mid = (lo_e + hi_e) >> 1;
      if (__ldg(irb + mid + 1) <= it.lo) lo_e = mid + 1;
      else hi_e = mid;
    }
    it.e = lo_e;
    bool more = it.hi > it.lo;
    for (;;) {
      while (more && nl - ns < static_cast<unsigned long long>(kPullSlots)) {
        const uint8_t* src;
        uint8_t* dst;
        uint32_t bytes;
        if (!next_piece(p, s, it, src, dst, bytes)) {
          more = false;
          break;
        }
        const int slot = static_cast<int>(nl % kPullSlots);
        // the store that last used this slot (piece nl - kPullSlots) must have read it
        if (nl >= static_cast<unsigned long long>(kPullSlots))
          bulk_wait_read_le(static_cast<int>(ns - 1 - (nl - kPullSlots)));
        mbar_arrive_expect_tx(&bar[slot], bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + slot * kPullPiece)),
            "l"(src), "r"(bytes), "r"(smem_u32(&bar[slot]))
            : "memory");
        dst_of[slot] = dst;
        bytes_of[slot] = bytes;
        ++nl;
      }
      if (ns == nl) break;
      const int slot = static_cast<int>(ns % kPullSlots);
      mbar_wait(&bar[slot], static_cast<uint32_t>((ns / kPullSlots) & 1));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_of[slot]),
                   "r"(smem_u32(smem + slot * kPullPiece)), "r"(bytes_of[slot])
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++ns;
    }
    // this CTA's share of source s has landed: publish (notify(arrival, src), ag_moe.py:117)
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    fence_proxy_async_global();
    fence_sys();
    red_add_release_sys(p.own_flags + s, 1);
  }
}

template <int CG, int MH, int BN, bool OUT_F32, int EPI, bool AG_WAIT, bool GROUPED = false, int NPAIR = 1>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_a,
                      const __grid_constant__ CUtensorMap tmap_b,
                      const __grid_constant__ CUtensorMap tmap_c,
                      const __grid_constant__ CUtensorMap tmap_p,
                      const __grid_constant__ KParams p) {
  using S = Smem<CG, MH, BN>;
  constexpr int ACC = S::kAccStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + S::kStages * S::kABytes;
  uint8_t* smem_epi = smem + S::kStages * S::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_epi + S::kEpiBytes);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + S::kStages;
  uint64_t* tfull_bar = bars + 2 * S::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  if constexpr (GROUPED) {
    // leading CTAs (whole clusters) run the pull engine and leave
    if (static_cast<int>(blockIdx.x) < p.comm_ctas) {
      moe_pull_engine(p, smem);
      return;
    }
  }
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // NPAIR = 2: a 4-CTA cluster = two CTA pairs computing adjacent N tiles of the same
  // rows; each CTA TMA-loads half of its pair's A rows and multicasts them to the
  // matching CTA of the other pair, so A crosses L2 -> SM once per cluster.
  const uint32_t cta_rank = CG == 2 ? cluster_ctarank() : 0;
  const uint32_t prank = cta_rank & 1;              // rank inside the CTA pair
  const int pair = static_cast<int>(cta_rank >> 1); // which pair of the cluster
  const bool leader = prank == 0;
  constexpr int kCluster = CG * NPAIR;
  const int num_clusters = (static_cast<int>(gridDim.x) - p.comm_ctas) / kCluster;
  int* vcid_slot = reinterpret_cast<int*>(tmem_slot + 2);  // spare word after the TMEM slot
  if (p.die_mode && threadIdx.x == 0 && cta_rank == 0) {
    // die-ranked cluster id: die-0 clusters count up from 0, die-1 clusters down from
    // num_clusters - 1 (a bijection whatever the arrival order); the last arrival
    // resets the counter for the next launch that uses this slot
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int d = p.sm_die[smid & 255] & 1;
    const unsigned long long old = atomicAdd(p.die_ctr, d ? (1ull << 32) : 1ull);
    const int lo = static_cast<int>(old & 0xFFFFFFFFull), hi = static_cast<int>(old >> 32);
    if (lo + hi + 1 == num_clusters) atomicExch(p.die_ctr, 0ull);
    const int v = d ? num_clusters - 1 - hi : lo;
    *vcid_slot = v;  // the cluster's other CTAs read it after the cluster barrier below
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NPAIR);  // freed once every pair's MMAs read the stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4 * CG);  // every epilogue warp of the pair
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
    if (p.tma_store) tma_prefetch_desc(&tmap_c);
    if (p.split_s > 1) tma_prefetch_desc(&tmap_p);
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair(tmem_slot, S::kTmemCols);
    else tmem_alloc(tmem_slot, S::kTmemCols);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  int cluster_id = (static_cast<int>(blockIdx.x) - p.comm_ctas) / kCluster;
  if (p.die_mode) {
    if (cta_rank == 0) {
      cluster_id = *vcid_slot;
    } else {
      uint32_t v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(mapa_shared(smem_u32(vcid_slot), 0)) : "memory");
      cluster_id = static_cast<int>(v);
    }
  }

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint64_t ready_mask = 0;  // AllGather chunks already observed as arrived
      const uint64_t pol_a = l2_policy(p.hint_a), pol_b = l2_policy(p.hint_b);
      for (int work = cluster_id; work < p.total_work; work += num_clusters) {
        int step, kb0, kb1, slot;
        decode_work(p, work, step, kb0, kb1, slot, num_clusters);
        const TileGeo geo = tile_geo<GROUPED, S::kTileM, BN, NPAIR>(p, step, pair);
        const int pid_m = geo.pid_m, pid_n = geo.pid_n;
        const int tile_m0 = geo.row0;
        const int n0 = geo.b_row0 + S::kBRows * prank;    // this CTA's B rows
        if constexpr (GROUPED) {
          // wait(arrival, segment_start, segment_end) acquire -- ag_moe.py:131-132
          if (p.src_flags) {
            const int s0 = geo.seg & 0xFFFF, s1 = geo.seg >> 16;
            const unsigned long long tw0 = p.trace ? globaltimer_ns() : 0;
            bool waited = false;
            for (int sr = s0; sr <= s1; ++sr) {
              if (ready_mask & (1ull << sr)) continue;
              wait_geq_sys(p.src_flags + sr, p.src_target, p.timeout_ns, p.err,
                           0x1000000ull | static_cast<unsigned long long>(sr));
              ready_mask |= 1ull << sr;
              waited = true;
            }
            if (waited) {
              trace_rec(p, 1, pid_m * p.num_pid_n * NPAIR + pid_n, tw0, globaltimer_ns(),
                        (static_cast<unsigned long long>(s0) << 32) | static_cast<unsigned>(s1 - s0 + 1));
              fence_proxy_async_global();
            }
          }
        }
        if constexpr (AG_WAIT) {
          // wait(arrival, rank_beg, n) acquire -- ag_gemm.py:87-90 (this CTA's rows)
          bool waited = false;
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            // rows of the gathered operand this CTA loads: A blocks, or its B rows
            const int m0 = p.wait_on_b ? n0 : tile_m0 + block_row<CG>(h, prank);
            const int lim = p.wait_on_b ? p.n : p.m;
            const int span = p.wait_on_b ? S::kBRows : 128;
            if (m0 >= lim || (p.wait_on_b && h > 0) || (NPAIR == 2 && h != pair)) continue;
            const int r1 = min(m0 + span, lim) - 1;
            const int c_beg = static_cast<int>(m0 / p.rows_per_chunk);
            const int c_end = static_cast<int>(r1 / p.rows_per_chunk);
            const unsigned long long tw0 = p.trace ? globaltimer_ns() : 0;
            bool this_wait = false;
            for (int c = c_beg; c <= c_end; ++c) {
              if (ready_mask & (1ull << c)) continue;
              wait_geq_sys(p.chunk_flags + c, p.epoch, p.timeout_ns, p.err,
                           0x1000000ull | static_cast<unsigned long long>(c));
              ready_mask |= 1ull << c;
              waited = true;
              this_wait = true;
            }
            // wait(arrival, rank_beg, num_slots) as in the reference trace (rank slots)
            if (this_wait) {
              const int cpr = p.chunks_per_rank > 0 ? p.chunks_per_rank : 1;
              trace_rec(p, 1, pid_m * p.num_pid_n * NPAIR + pid_n, tw0, globaltimer_ns(),
                        (static_cast<unsigned long long>(c_beg / cpr) << 32) |
                            static_cast<unsigned>(c_end / cpr - c_beg / cpr + 1));
            }
          }
          // generic-proxy acquire -> async-proxy (TMA) reads of the same bytes
          if (waited) fence_proxy_async_global();
        }
        // K direction: odd waves run backwards so a wave starts on the k-slices the
        // previous wave touched last (still in L2); the MMA side is order-agnostic
        const bool krev = p.ksnake && (((work - cluster_id) / num_clusters) & 1);
        for (int kq = kb0; kq < kb1; ++kq) {
          const int kb = krev ? kb1 - 1 - (kq - kb0) : kq;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem_a + stage * S::kABytes;
          uint8_t* sb = smem_b + stage * S::kBBytes;
          if constexpr (NPAIR == 2) {
            // both CTAs of the pair receive both A blocks (one from each pair) + own B
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
            const uint16_t amask = static_cast<uint16_t>((1u << prank) | (1u << (2 + prank)));
            tma_load_2d_pair_mc(sa + pair * S::kABlock, &tmap_a, &full_bar[stage], kb * BK,
                                tile_m0 + block_row<CG>(pair, prank), amask);
            tma_load_2d_pair(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          } else if constexpr (CG == 2) {
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
#pragma unroll
            for (int h = 0; h < MH; ++h) {
              if (p.hint_a)
                tma_load_2d_pair_hint(sa + h * S::kABlock, &tmap_a, &full_bar[stage], kb * BK,
                                      tile_m0 + block_row<CG>(h, prank), pol_a);
              else
                tma_load_2d_pair(sa + h * S::kABlock, &tmap_a, &full_bar[stage], kb * BK,
                                 tile_m0 + block_row<CG>(h, prank));
            }
            if (p.hint_b) tma_load_2d_pair_hint(sb, &tmap_b, &full_bar[stage], kb * BK, n0, pol_b);
            else tma_load_2d_pair(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], S::kStageBytes);
#pragma unroll
            for (int h = 0; h < MH; ++h)
              tma_load_2d(sa + h * S::kABlock, &tmap_a, &full_bar[stage], kb * BK,
                          tile_m0 + block_row<CG>(h, prank));
            tma_load_2d(sb, &tmap_b, &full_bar[stage], kb * BK, n0);
          }
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && MH == 2) {
      // Two M-halves per tile share one TMEM allocation (no double buffer).  Each
      // half has its own full/empty barrier pair, and at tile boundaries the
      // second half's MMAs lag by L k-blocks: the epilogue drains half 0 while
      // half 1 finishes, and the next tile's half 0 starts while half 1 drains.
      constexpr uint32_t idesc = umma_idesc_bf16(128 * CG, BN);
      constexpr int L = TF_GEMM_LAG;
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      auto issue = [&](int st, int h, int kb) {
        const uint32_t a_lo = desc_lo_k(smem_u32(smem_a + st * S::kABytes) + h * S::kABlock);
        const uint32_t b_lo = desc_lo_k(smem_u32(smem_b + st * S::kBBytes));
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          const uint64_t ad = desc_from_lo(a_lo + kk * (UMMA_K * 2 >> 4));
          const uint64_t bd = desc_from_lo(b_lo + kk * (UMMA_K * 2 >> 4));
          if constexpr (CG == 2) umma_bf16_pair(tmem_base + h * BN, ad, bd, idesc, (kb | kk) != 0);
          else umma_bf16(tmem_base + h * BN, ad, bd, idesc, (kb | kk) != 0);
        }
      };
      // smem stages are released to every CTA whose producer writes them (both pairs
      // with NPAIR = 2); accumulator-ready goes to this pair's two CTAs only
      constexpr uint16_t kEmptyMask = NPAIR == 2 ? 0xF : 0x3;
      const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));
      auto release = [&](uint64_t* bar) {
        if constexpr (CG == 2) umma_commit_pair_mc(bar, kEmptyMask);
        else umma_commit(bar);
      };
      auto release_acc = [&](uint64_t* bar) {
        if constexpr (CG == 2) umma_commit_pair_mc(bar, pair_mask);
        else umma_commit(bar);
      };
      for (int work = cluster_id; work < p.total_work; work += num_clusters, ++local) {
        int step, kb0, kb1, slot;
        decode_work(p, work, step, kb0, kb1, slot, num_clusters);
        const uint32_t tph = local & 1;
        const int nkb = kb1 - kb0;
        const bool lagged = nkb >= 2 * L + 1;
        mbar_wait(&tempty_bar[0], tph ^ 1);
        if (!lagged) mbar_wait(&tempty_bar[1], tph ^ 1);
        tc_fence_after();
        const int s0 = stage;
        const unsigned long long tm0 = p.trace ? globaltimer_ns() : 0;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const bool head = lagged && kb < L;
          const bool tail = lagged && kb >= nkb - L;
          if (lane == 0) {
            issue(stage, 0, kb);
            if (!head && !tail) {
              issue(stage, 1, kb);
              release(&empty_bar[stage]);
            }
          }
          __syncwarp();
          if (lagged && kb == L - 1) {
            // catch half 1 up on the held head stages once its accumulator is free
            mbar_wait(&tempty_bar[1], tph ^ 1);
            tc_fence_after();
            if (lane == 0)
              for (int j = 0; j < L; ++j) {
                const int st = (s0 + j) % S::kStages;
                issue(st, 1, j);
                release(&empty_bar[st]);
              }
            __syncwarp();
          }
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) {
          release_acc(&tfull_bar[0]);  // half 0 complete: its epilogue can start
          if (lagged)
            for (int j = nkb - L; j < nkb; ++j) {
              const int st = (s0 + j) % S::kStages;
              issue(st, 1, j);
              release(&empty_bar[st]);
            }
          release_acc(&tfull_bar[1]);
          if (p.trace) {
            const TileGeo tg = tile_geo<GROUPED, S::kTileM, BN, NPAIR>(p, step, pair);
            const int pm = tg.pid_m, pn = tg.pid_n;
            trace_rec(p, 2, pm * p.num_pid_n * NPAIR + pn, tm0, globaltimer_ns(),
                      (static_cast<unsigned long long>(pm) << 32) | static_cast<unsigned>(pn));
          }
        }
        __syncwarp();
      }
    } else if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(128 * CG, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int work = cluster_id; work < p.total_work; work += num_clusters, ++local) {
        int step, kb0, kb1, slot;
        decode_work(p, work, step, kb0, kb1, slot, num_clusters);
        const int acc = local % ACC;
        const uint32_t acc_phase = (local / ACC) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * S::kAccCols;
        const unsigned long long tm0 = p.trace ? globaltimer_ns() : 0;
        for (int kb = 0; kb < kb1 - kb0; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_lo = desc_lo_k(smem_u32(smem_a + stage * S::kABytes));
            const uint32_t b_lo = desc_lo_k(smem_u32(smem_b + stage * S::kBBytes));
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; ++kk) {
              const uint64_t bd = desc_from_lo(b_lo + kk * (UMMA_K * 2 >> 4));
#pragma unroll
              for (int h = 0; h < MH; ++h) {
                const uint64_t ad = desc_from_lo(a_lo + (h * S::kABlock >> 4) + kk * (UMMA_K * 2 >> 4));
                if constexpr (CG == 2)
                  umma_bf16_pair(d_tmem + h * BN, ad, bd, idesc, (kb | kk) != 0);
                else
                  umma_bf16(d_tmem + h * BN, ad, bd, idesc, (kb | kk) != 0);
              }
            }
            // smem slot free (in both CTAs) once these MMAs retire
            if constexpr (CG == 2) umma_commit_pair_mc(&empty_bar[stage], NPAIR == 2 ? 0xF : 0x3);
            else umma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == S::kStages) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) {  // accumulator ready for the epilogues
          if constexpr (CG == 2) umma_commit_pair_mc(&tfull_bar[acc], static_cast<uint16_t>(0x3u << (2 * pair)));
          else umma_commit(&tfull_bar[acc]);
          if (p.trace) {
            const TileGeo tg = tile_geo<GROUPED, S::kTileM, BN, NPAIR>(p, step, pair);
            const int pm = tg.pid_m, pn = tg.pid_n;
            trace_rec(p, 2, pm * p.num_pid_n * NPAIR + pn, tm0, globaltimer_ns(),
                      (static_cast<unsigned long long>(pm) << 32) | static_cast<unsigned>(pn));
          }
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;          // TMEM lanes [32*quarter, 32*quarter+32)
    const int row_in_blk = quarter * 32 + lane;
    const uint32_t tempty_leader =
        CG == 2 ? mapa_shared(smem_u32(&tempty_bar[0]), 2 * pair) : smem_u32(&tempty_bar[0]);
    // TMA-store staging: this warp's two 32x128 B buffers (128-byte swizzled)
    uint8_t* epi_buf = smem_epi + (warp - kEpiWarp0) * 2 * S::kEpiBuf;
    int epi_slot = 0;
    unsigned long long epi_t0 = 0;
    constexpr int kColsPerStore = OUT_F32 ? 32 : 64;  // 128 B of one row
    int local = 0;
    for (int work = cluster_id; work < p.total_work; work += num_clusters, ++local) {
      int step, kb0, kb1, slot;
      decode_work(p, work, step, kb0, kb1, slot, num_clusters);
      const TileGeo geo = tile_geo<GROUPED, S::kTileM, BN, NPAIR>(p, step, pair);
      const int pid_m = geo.pid_m, pid_n = geo.pid_n;
      const int acc = local % ACC;
      const uint32_t acc_phase = (local / ACC) & 1;
      if (p.trace && warp == kEpiWarp0 && lane == 0) {
        // one event per work item: from the epilogue picking it up to its drain (below)
        epi_t0 = globaltimer_ns();
      }
      // MH == 2: one barrier pair per half (tfull[h] / tempty[h]); else per accumulator
      auto wait_full = [&](int h) {
        if constexpr (MH == 2) mbar_wait(&tfull_bar[h], local & 1);
        else mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
      };
      auto arrive_empty = [&](int h) {
        tc_fence_before();
        __syncwarp();
        if (p.trace && warp == kEpiWarp0 && lane == 0 && (MH == 1 || h == MH - 1))
          trace_rec(p, 3, pid_m * p.num_pid_n * NPAIR + pid_n, epi_t0, globaltimer_ns(),
                    (static_cast<unsigned long long>(pid_m) << 32) | static_cast<unsigned>(pid_n));
        const int b = MH == 2 ? h : acc;
        if (lane == 0) {
          if constexpr (CG == 2) {
            if constexpr (kRelaxedArrive) mbar_arrive_cluster_relaxed(tempty_leader + b * 8);
            else mbar_arrive_cluster(tempty_leader + b * 8);
          }
          else mbar_arrive(&tempty_bar[b]);
        }
      };
      if (EPI == 0 && slot >= 0) {
        // split-K tail unit: fp32 partial tile -> workspace slot (fixed up by tail_fixup_kernel)
#pragma unroll 1
        for (int h = 0; h < MH; ++h) {
          if (MH == 2 || h == 0) wait_full(h);
          const int prow0 = (slot * NPAIR + pair) * S::kTileM + block_row<CG>(h, prank) + quarter * 32;
          const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                 acc * S::kAccCols + h * BN;
#pragma unroll 1
          for (int cc = 0; cc < BN; cc += 32) {
            uint8_t* buf = epi_buf + epi_slot * S::kEpiBuf;
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + cc, v);
            if (lane == 0) tma_store_wait_read<1>();
            __syncwarp();
            tmem_ld_wait();
            uint8_t* my_row = buf + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(my_row + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmap_p, buf, cc, prow0);
              tma_store_commit();
            }
            epi_slot ^= 1;
          }
          if (MH == 2 || h == MH - 1) arrive_empty(h);
        }
        continue;
      }
      if constexpr (EPI == 0 && !OUT_F32 && !GROUPED && BN == 256) {
        if (p.tma_store && kEarlyRelease) {
          // Early release: the half's 256 fp32 columns come out of TMEM as packed bf16 in
          // registers (128 regs per thread), TMEM is handed back to the MMA warp at once,
          // and only then are the registers staged through swizzled smem and TMA-stored
          // -- the store traffic overlaps the next tile's MMAs instead of stalling them
#pragma unroll 1
          for (int h = 0; h < MH; ++h) {
            if (MH == 2 || h == 0) wait_full(h);
            const int wrow0 = geo.row0 + block_row<CG>(h, prank) + quarter * 32;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                   acc * S::kAccCols + h * BN;
            uint32_t pk[BN / 2];
#pragma unroll
            for (int cc = 0; cc < BN; cc += 64) {
              uint32_t v[64];
              tmem_ld_32x32b_x32(t_row + cc, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
              tmem_ld_32x32b_x32(t_row + cc + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j)
                pk[cc / 2 + j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
            }
            if (MH == 2 || h == MH - 1) arrive_empty(h);  // TMEM free: the next tile may start
#pragma unroll
            for (int cc = 0; cc < BN; cc += 64) {
              uint8_t* buf = epi_buf + epi_slot * S::kEpiBuf;
              // the store issued from this buffer two rounds ago must have read it
              if (lane == 0) tma_store_wait_read<1>();
              __syncwarp();
              uint8_t* my_row = buf + lane * 128;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my_row + ((j ^ (lane & 7)) << 4)) =
                    make_uint4(pk[cc / 2 + 4 * j], pk[cc / 2 + 4 * j + 1], pk[cc / 2 + 4 * j + 2],
                               pk[cc / 2 + 4 * j + 3]);
              fence_proxy_async_shared();
              __syncwarp();
              if (lane == 0 && wrow0 < p.m && pid_n * BN + cc < p.n && !p.dbg_skip_store)
                tma_store_2d(&tmap_c, buf, pid_n * BN + cc, wrow0);
              if (lane == 0) tma_store_commit();
              epi_slot ^= 1;
            }
          }
          continue;
        }
      }
      if (EPI == 0 && p.tma_store) {
        // 32-row x 128-byte boxes: TMEM -> regs -> swizzled smem -> cp.async.bulk.tensor
#pragma unroll 1
        for (int h = 0; h < MH; ++h) {
          if (MH == 2 || h == 0) wait_full(h);
          const int wrow0 = geo.row0 + block_row<CG>(h, prank) + quarter * 32;
          const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                 acc * S::kAccCols + h * BN;
          // grouped tiles end at their expert's last row: a band that crosses it is
          // stored row by row (a TMA box would overwrite the next expert's rows)
          const bool band_masked = GROUPED && wrow0 + 32 > geo.row_lim;
#pragma unroll 1
          for (int cc = 0; cc < BN; cc += kColsPerStore) {
            uint8_t* buf = epi_buf + epi_slot * S::kEpiBuf;
            uint32_t v[kColsPerStore];
            tmem_ld_32x32b_x32(t_row + cc, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
            if constexpr (!OUT_F32)
              tmem_ld_32x32b_x32(t_row + cc + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
            if (band_masked) {
              tmem_ld_wait();
              const int grow = wrow0 + lane;
              const int col0 = pid_n * BN + cc;
              if (grow < geo.row_lim && col0 < p.n) {
                uint8_t* dst = static_cast<uint8_t*>(p.c) +
                               (static_cast<long long>(grow) * p.ldc + col0) * (OUT_F32 ? 4 : 2);
                const int ncols = min(kColsPerStore, p.n - col0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  if (j * (16 / (OUT_F32 ? 4 : 2)) >= ncols) break;
                  uint4 q;
                  if constexpr (OUT_F32) {
                    q = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                  } else {
                    q = make_uint4(
                        pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                        pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                        pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                        pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
                  }
                  reinterpret_cast<uint4*>(dst)[j] = q;
                }
              }
              continue;
            }
            // the store issued from this buffer two rounds ago must have read it
            if (lane == 0) tma_store_wait_read<1>();
            __syncwarp();
            tmem_ld_wait();
            uint8_t* my_row = buf + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint4 q;
              if constexpr (OUT_F32) {
                q = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              } else {
                q = make_uint4(
                    pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
              }
              *reinterpret_cast<uint4*>(my_row + ((j ^ (lane & 7)) << 4)) = q;
            }
            fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0 && wrow0 < p.m && pid_n * BN + cc < p.n && !p.dbg_skip_store) {
              tma_store_2d(&tmap_c, buf, pid_n * BN + cc, wrow0);
            }
            if (lane == 0) tma_store_commit();
            epi_slot ^= 1;
          }
          // this half drained (stores read smem asynchronously, TMEM is free)
          if (MH == 2 || h == MH - 1) arrive_empty(h);
        }
        continue;
      }
#pragma unroll 1
      for (int h = 0; h < MH; ++h) {
        if (MH == 2 || h == 0) wait_full(h);
        const int row0 = pid_m * S::kTileM + block_row<CG>(h, prank);
        const int row = row0 + row_in_blk;
        const bool row_ok = row < p.m;
        uint8_t* dst_row = nullptr;
        if (row_ok) {
          if constexpr (EPI == 0) {
            dst_row = static_cast<uint8_t*>(p.c) +
                      (static_cast<long long>(row) * p.ldc) * (OUT_F32 ? 4 : 2);
          } else {
            // slot layout at the owner: [world][rows_per_rank][slot_ld], slot = source rank
            const int owner = static_cast<int>(row / p.rows_per_rank);
            const long long orow = row - owner * p.rows_per_rank;
            dst_row = static_cast<uint8_t*>(p.peer_slots[owner]) +
                      ((p.rank * p.rows_per_rank + orow) * p.slot_ld) * (OUT_F32 ? 4 : 2);
          }
        }
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                               acc * S::kAccCols + h * BN;
        if constexpr (EPI == 1 && !OUT_F32) {
          // Scatter to the owners through a per-warp smem transpose: each 64-column chunk
          // of the warp's 32 rows is staged (128-byte swizzled), then written out so that
          // one store instruction covers 4 rows x 128 contiguous bytes -- full-line
          // requests over NVLink instead of 16-byte pieces of 32 different rows.
          const int wrow0 = row0 + quarter * 32;
          if (p.vec_ok && !p.dbg_skip_store && (BN % 64) == 0) {
            uint8_t* buf = epi_buf;
#pragma unroll 1
            for (int cc = 0; cc < BN; cc += 64) {
              uint32_t v[64];
              tmem_ld_32x32b_x32(t_row + cc, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
              tmem_ld_32x32b_x32(t_row + cc + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
              tmem_ld_wait();
              __syncwarp();  // the previous chunk's reads of buf are done
              uint8_t* my_row = buf + lane * 128;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<uint4*>(my_row + ((j ^ (lane & 7)) << 4)) = make_uint4(
                    pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
              __syncwarp();
              const int col0 = pid_n * BN + cc;
              const int chunk = lane & 7;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int rr = i * 4 + (lane >> 3);
                const int grow = wrow0 + rr;
                const int cbase = col0 + chunk * 8;
                if (grow >= p.m || cbase >= p.n) continue;
                const uint4 q = *reinterpret_cast<const uint4*>(buf + rr * 128 + ((chunk ^ (rr & 7)) << 4));
                const int owner = static_cast<int>(grow / p.rows_per_rank);
                const long long orow = grow - owner * p.rows_per_rank;
                uint16_t* dst = static_cast<uint16_t*>(p.peer_slots[owner]) +
                                (p.rank * p.rows_per_rank + orow) * p.slot_ld + cbase;
                if (cbase + 8 <= p.n) {
                  *reinterpret_cast<uint4*>(dst) = q;
                } else {
                  const uint16_t* e = reinterpret_cast<const uint16_t*>(&q);
                  for (int t = 0; t < p.n - cbase; ++t) dst[t] = e[t];
                }
              }
            }
            __syncwarp();
            if constexpr (MH == 2) arrive_empty(h);  // this half drained
            continue;
          }
        }
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 32) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + cc, v);
          tmem_ld_wait();
          const int col0 = pid_n * BN + cc;
          if (!row_ok || col0 >= p.n || p.dbg_skip_store) continue;
          if (p.vec_ok && col0 + 32 <= p.n) {
            if constexpr (OUT_F32) {
              uint4* d = reinterpret_cast<uint4*>(dst_row + static_cast<long long>(col0) * 4);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                d[j] = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            } else {
              uint4* d = reinterpret_cast<uint4*>(dst_row + static_cast<long long>(col0) * 2);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                d[j] = make_uint4(
                    pack_bf16x2(__uint_as_float(v[8 * j + 0]), __uint_as_float(v[8 * j + 1])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 2]), __uint_as_float(v[8 * j + 3])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 4]), __uint_as_float(v[8 * j + 5])),
                    pack_bf16x2(__uint_as_float(v[8 * j + 6]), __uint_as_float(v[8 * j + 7])));
              }
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (col0 + j < p.n) {
                if constexpr (OUT_F32) {
                  reinterpret_cast<float*>(dst_row)[col0 + j] = __uint_as_float(v[j]);
                } else {
                  reinterpret_cast<uint16_t*>(dst_row)[col0 + j] =
                      static_cast<uint16_t>(pack_bf16x2(__uint_as_float(v[j]), 0.f) & 0xFFFF);
                }
              }
            }
          }
        }
        if constexpr (MH == 2) arrive_empty(h);  // this half drained
      }
      // accumulator drained: hand TMEM back to the leader's MMA warp
      if constexpr (MH == 1) arrive_empty(0);
      if constexpr (EPI == 1) {
        // publish: every thread's stores are made visible system-wide, the four
        // epilogue warps meet, then one thread release-adds the owners' counters
        // (one counter per 128-row block of the output).
        fence_sys();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == kEpiWarp0 * 32) {
#pragma unroll 1
          for (int h = 0; h < MH; ++h) {
            const int row0 = pid_m * S::kTileM + block_row<CG>(h, prank);
            if (row0 >= p.m) continue;
            const int r1 = min(row0 + 128, p.m) - 1;
            const int o0 = static_cast<int>(row0 / p.rows_per_rank);
            const int o1 = static_cast<int>(r1 / p.rows_per_rank);
            for (int o = o0; o <= o1; ++o) {
              if (p.trace) {
                // traced: the fetch-add's old value records which bump this was (the
                // reference's atomic_add signal event, gemm_rs.py:155-161)
                const unsigned long long t0 = globaltimer_ns();  // <= the add's visibility
                const unsigned long long old = atom_add_release_sys(p.peer_counts[o] + row0 / 128, 1);
                trace_push(p.trace, p.trace_cap, 4, p.trace_rank, row0 / 128, t0, globaltimer_ns(),
                           (static_cast<unsigned long long>(o) << 32) | static_cast<unsigned>(old + 1));
              } else {
                red_add_release_sys(p.peer_counts[o] + row0 / 128, 1);
              }
            }
          }
        }
      }
    }
  }

  if (warp >= kEpiWarp0 && lane == 0) tma_store_wait<0>();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair(tmem_base, S::kTmemCols);
    else tmem_dealloc(tmem_base, S::kTmemCols);
  }
}

// Split-K tail fix-up: tile i of the tail = sum over parts j (in order) of
// workspace slots i*split_s + j, converted and stored to C.  One CTA per
// (tail tile, 32-row band); 256 threads cover 256 columns... of BN.
template <int TILE_M, int BN, bool OUT_F32, int NPAIR = 1>
__global__ void __launch_bounds__(256) tail_fixup_kernel(const float* __restrict__ ws,
                                                         const __grid_constant__ KParams p) {
  // one CTA per (tail tile, 32-row band), one thread per column of the tile; with
  // NPAIR = 2 a tail work item holds two N tiles (pair q writes slot unit*2 + q)
  const int bands = TILE_M / 32;
  const int i = blockIdx.x / bands;
  const int band = blockIdx.x % bands;
  const int item = i / NPAIR, q = i % NPAIR;
  int pid_m, pid_n;
  tile_coords(p, p.tail_base + item, pid_m, pid_n);
  pid_n = pid_n * NPAIR + q;
  const int c = pid_n * BN + threadIdx.x;
  for (int r = 0; r < 32; ++r) {
    const int lrow = band * 32 + r;
    const int row = pid_m * TILE_M + lrow;
    if (row >= p.m) break;
    float acc = 0.f;
    for (int j = 0; j < p.split_s; ++j)  // fixed order: deterministic
      acc += ws[(static_cast<long long>((item * p.split_s + j) * NPAIR + q) * TILE_M + lrow) * BN +
                threadIdx.x];
    if (c < p.n) {
      if constexpr (OUT_F32)
        static_cast<float*>(p.c)[static_cast<long long>(row) * p.ldc + c] = acc;
      else
        static_cast<uint16_t*>(p.c)[static_cast<long long>(row) * p.ldc + c] =
            static_cast<uint16_t>(pack_bf16x2(acc, 0.f) & 0xFFFF);
    }
  }
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

CUtensorMapL2promotion l2_promotion() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TF_L2_PROMO");  // experiments: 0 none, 1 64B, 2 128B, 3 256B
    v = e ? atoi(e) : 3;
  }
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

int make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld,
                 int box_rows, int esz = 2, int box_cols = BK) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return fail(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esz)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt =
      esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TF_ERR_INVALID, "cuTensorMapEncodeTiled failed (code " + std::to_string(r) +
                                    "): rows=" + std::to_string(rows) +
                                    " cols=" + std::to_string(cols) + " ld=" + std::to_string(ld));
  return TF_OK;
}

template <int CG, int MH, int BN, bool OUT_F32, int EPI, bool AG_WAIT, bool GROUPED = false, int NPAIR = 1>
int launch_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
             const CUtensorMap& tp, const KParams& kp, int grid, cudaStream_t stream,
             const float* tail_ws) {
  auto kern = gemm_sm100_kernel<CG, MH, BN, OUT_F32, EPI, AG_WAIT, GROUPED, NPAIR>;
  using S = Smem<CG, MH, BN>;
  static uint64_t attr_done = 0;  // per template instance, bit per device
  static int max_clusters[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done & (1ull << dev))) {
    TF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal));
    if (NPAIR > 1) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr_done |= 1ull << dev;
  }
  if (NPAIR > 1 && dev < 64) {
    // a persistent grid must not exceed the co-resident 4-CTA clusters (GPC packing)
    if (!max_clusters[dev]) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3(grid);
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = S::kTotal;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = CG * NPAIR;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int mc = 0;
      if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc < 1) mc = 1 << 20;
      cudaGetLastError();
      max_clusters[dev] = mc;
      if (getenv("TF_GEMM_DEBUG")) fprintf(stderr, "[tf] max active %d-CTA clusters: %d\n", CG * NPAIR, mc);
    }
    const int cap = max_clusters[dev] * CG * NPAIR + kp.comm_ctas;
    if (grid > cap) grid = cap;
  }
  KParams kd = kp;
  {
    // die-ranked cluster ids (tf_topo.cu); TF_GEMM_DIE = 0 off, 1 ranked, 2 ranked + row split
    // (the row split is for the grouped raster of plain GEMMs only)
    static const int die_env = [] {
      const char* e = getenv("TF_GEMM_DIE");
      return e ? atoi(e) : kDefaultDieMode;
    }();
    if (die_env > 0) {
      unsigned long long* slot = nullptr;
      const uint8_t* tab = sm_die_table(dev, &slot);
      if (tab) {
        kd.sm_die = tab;
        kd.die_ctr = slot;
        kd.die_mode = GROUPED ? 1 : die_env;
      }
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = S::kTotal;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * NPAIR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tp, kd));
  if (kp.split_s > 1) {
    const int tail_tiles = (kp.total_work - kp.tail_base) / kp.split_s * NPAIR;
    tail_fixup_kernel<S::kTileM, BN, OUT_F32, NPAIR>
        <<<tail_tiles * (S::kTileM / 32), BN, 0, stream>>>(tail_ws, kp);
    TF_CUDA_TRY(cudaGetLastError());
  }
  return TF_OK;
}

template <int CG, int MH, int BN, int NPAIR = 1>
int dispatch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                const CUtensorMap& tp, const KParams& kp, int grid, const GemmLaunch& g,
                cudaStream_t s, const float* ws) {
  const bool ag = g.chunk_flags != nullptr;
  if (g.epilogue == 0) {
    if (g.out_f32)
      return ag ? launch_t<CG, MH, BN, true, 0, true, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws)
                : launch_t<CG, MH, BN, true, 0, false, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws);
    return ag ? launch_t<CG, MH, BN, false, 0, true, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws)
              : launch_t<CG, MH, BN, false, 0, false, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws);
  }
  if (g.out_f32) return launch_t<CG, MH, BN, true, 1, false, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws);
  return launch_t<CG, MH, BN, false, 1, false, false, NPAIR>(ta, tb, tc, tp, kp, grid, s, ws);
}

// Per-(device, stream) fp32 workspace for split-K tail partials (grown on demand).
float* tail_workspace(cudaStream_t s, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> bufs;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  auto& e = bufs[{dev, s}];
  if (e.second < bytes) {
    if (e.first) {
      cudaStreamSynchronize(s);
      cudaFree(e.first);
    }
    e.first = nullptr;
    e.second = 0;
    if (cudaMalloc(&e.first, bytes) != cudaSuccess) return nullptr;
    e.second = bytes;
  }
  return static_cast<float*>(e.first);
}

struct TraceBuf {
  unsigned long long* buf = nullptr;
  int64_t cap = 0;
};
std::mutex g_trace_mu;
std::map<int, TraceBuf> g_trace;

}  // namespace

int trace_buffer(int device, unsigned long long** buf) {
  std::lock_guard<std::mutex> lock(g_trace_mu);
  auto it = g_trace.find(device);
  if (it == g_trace.end() || !it->second.buf) {
    *buf = nullptr;
    return 0;
  }
  *buf = it->second.buf;
  return static_cast<int>(it->second.cap);
}

int num_sms_of_current_device() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n;
}

// Grouped (MoE) launch: tile table on the device, B = stacked expert weights,
// optional pull-engine CTAs in front (ag_moe.py:20-142).
int launch_grouped(const GemmLaunch& g, KParams kp, cudaStream_t stream) {
  if (g.block_m != 128 && g.block_m != 256)
    return fail(TF_ERR_CONFIG, "grouped GEMM: block_m must be 128 (one CTA) or 256 (CTA pair)");
  if (!kp.vec_ok) return fail(TF_ERR_INVALID, "grouped GEMM: n must be a multiple of 8 and C rows 16-byte aligned");
  const int cg = g.block_m == 128 ? 1 : 2;
  kp.num_pid_m = g.moe_slots;
  kp.moe_tab = static_cast<const int4*>(g.moe_tab);
  kp.moe_n = static_cast<int>(g.n);
  kp.src_flags = g.src_flags;
  kp.src_target = g.src_target;
  kp.comm_ctas = g.comm_ctas;
  if (g.comm_ctas % cg) return fail(TF_ERR_CONFIG, "pull-engine CTAs must fill whole clusters");
  for (int r = 0; r < kMaxWorld; ++r) kp.peer_ws[r] = g.peer_ws[r];
  kp.own_ws = g.own_ws;
  kp.irb = g.irb;
  kp.dstb = g.dstb;
  kp.n_experts = g.n_experts;
  kp.row_bytes = g.row_bytes;
  kp.own_flags = g.own_flags;
  CUtensorMap ta, tb, tc, tp;
  std::memset(&tp, 0, sizeof(tp));
  int rc = make_tmap_2d(&ta, g.a, g.m, g.k, g.lda, 128);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, g.b, static_cast<int64_t>(g.n_experts) * g.n, g.k, g.ldb, g.block_n / cg);
  if (rc) return rc;
  const int esz_c = g.out_f32 ? 4 : 2;
  rc = make_tmap_2d(&tc, g.c, g.m, g.n, g.ldc, 32, esz_c, 128 / esz_c);
  if (rc) return rc;
  kp.tma_store = 1;
  const int tiles = kp.num_pid_m * kp.num_pid_n;
  kp.tail_base = tiles;
  kp.split_s = 1;
  kp.total_work = tiles;
  int ctas = g.num_sms > 0 ? g.num_sms : num_sms_of_current_device();
  ctas -= g.comm_ctas;
  int clusters = ctas / cg;
  if (clusters < 1) clusters = 1;
  if (tiles > 0 && clusters > tiles) clusters = tiles;
  const int grid = g.comm_ctas + clusters * cg;
  if (tiles == 0 && g.comm_ctas == 0) return TF_OK;
  if (cg == 2) {
    if (g.block_n == 256)
      return g.out_f32 ? launch_t<2, 1, 256, true, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr)
                       : launch_t<2, 1, 256, false, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr);
    return g.out_f32 ? launch_t<2, 1, 128, true, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr)
                     : launch_t<2, 1, 128, false, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr);
  }
  if (g.block_n == 256)
    return g.out_f32 ? launch_t<1, 1, 256, true, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr)
                     : launch_t<1, 1, 256, false, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr);
  return g.out_f32 ? launch_t<1, 1, 128, true, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr)
                   : launch_t<1, 1, 128, false, 0, false, true>(ta, tb, tc, tp, kp, grid, stream, nullptr);
}

int launch_gemm(const GemmLaunch& g, cudaStream_t stream) {
  if (g.m < 0 || g.n < 0 || g.k < 0) return fail(TF_ERR_INVALID, "negative GEMM dimension");
  if (g.m == 0 || g.n == 0) return TF_OK;
  if (g.block_n != 128 && g.block_n != 256)
    return fail(TF_ERR_CONFIG, "block_n must be 128 or 256 on the tcgen05 path");
  if (g.block_m != 128 && g.block_m != 256 && g.block_m != 512)
    return fail(TF_ERR_CONFIG, "block_m must be 128 (one CTA), 256 (CTA pair) or 512 (CTA pair, two M=256 MMAs)");
  const int tile_m = g.block_m;
  if ((g.lda * 2) % 16 || (g.ldb * 2) % 16)
    return fail(TF_ERR_INVALID, "A/B row strides must be multiples of 16 bytes (K % 8 == 0)");
  if ((reinterpret_cast<uintptr_t>(g.a) | reinterpret_cast<uintptr_t>(g.b)) & 15)
    return fail(TF_ERR_INVALID, "A/B base pointers must be 16-byte aligned");
  if (g.m > INT32_MAX || g.n > INT32_MAX || g.k > INT32_MAX)
    return fail(TF_ERR_INVALID, "GEMM dimension exceeds int32");
  if (g.epilogue == 1 && (g.world < 1 || g.world > kMaxWorld || g.rows_per_rank <= 0))
    return fail(TF_ERR_INVALID, "scatter epilogue needs 1 <= world <= TF_MAX_WORLD");
  if (g.chunk_flags && ((g.wait_on_b ? g.n : g.m) + g.rows_per_chunk - 1) / g.rows_per_chunk > 64)
    return fail(TF_ERR_CONFIG, "AllGather wait supports at most 64 chunks");
  if (g.group_m < 1) return fail(TF_ERR_CONFIG, "group_m must be >= 1");

  KParams kp{};
  kp.m = static_cast<int>(g.m);
  kp.n = static_cast<int>(g.n);
  kp.k = static_cast<int>(g.k);
  kp.num_pid_m = static_cast<int>((g.m + tile_m - 1) / tile_m);
  kp.num_pid_n = static_cast<int>((g.n + g.block_n - 1) / g.block_n);
  kp.group_m = g.group_m;
  kp.num_kb = static_cast<int>((g.k + BK - 1) / BK);
  kp.tile_map = g.tile_map;
  kp.c = g.c;
  kp.ldc = g.epilogue == 1 ? g.slot_ld : g.ldc;
  const int esz = g.out_f32 ? 4 : 2;
  const uintptr_t cbase = g.epilogue == 1 ? 0 : reinterpret_cast<uintptr_t>(g.c);
  bool vec = ((kp.ldc * esz) % 16 == 0) && (g.n % 8 == 0) && (cbase % 16 == 0);
  if (g.epilogue == 1)
    for (int r = 0; r < g.world; ++r) vec = vec && (reinterpret_cast<uintptr_t>(g.peer_slots[r]) % 16 == 0);
  kp.vec_ok = vec ? 1 : 0;
  kp.chunk_flags = g.chunk_flags;
  kp.epoch = g.epoch;
  kp.rows_per_chunk = g.rows_per_chunk > 0 ? g.rows_per_chunk : (g.m > 0 ? g.m : 1);
  kp.rank = g.rank;
  kp.world = g.world;
  kp.rows_per_rank = g.rows_per_rank > 0 ? g.rows_per_rank : g.m;
  for (int r = 0; r < kMaxWorld; ++r) {
    kp.peer_slots[r] = g.peer_slots[r];
    kp.peer_counts[r] = g.peer_counts[r];
  }
  kp.slot_ld = g.slot_ld;
  kp.err = g.err;
  kp.timeout_ns = g.timeout_ns;
  kp.dbg_skip_store = getenv("TF_DEBUG_SKIP_STORE") ? 1 : 0;
  kp.wait_on_b = g.wait_on_b ? 1 : 0;
  kp.tile_map_n = g.tile_map_n;
  kp.trace = nullptr;
  kp.trace_cap = 0;
  kp.trace_rank = g.trace_rank;
  {
    static int ha = -1, hb = -1;  // L2 policies of the operand loads (TF_L2_HINT_A/B experiments)
    if (ha < 0) {
      const char* ea = getenv("TF_L2_HINT_A");
      const char* eb = getenv("TF_L2_HINT_B");
      ha = ea ? atoi(ea) : 0;
      hb = eb ? atoi(eb) : 0;
    }
    kp.hint_a = ha;
    kp.hint_b = hb;
    const char* ks = getenv("TF_GEMM_KSNAKE");
    kp.ksnake = ks ? atoi(ks) : 0;
    kp.chunks_per_rank = g.chunks_per_rank;
  }
  {
    std::lock_guard<std::mutex> lock(g_trace_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    auto it = g_trace.find(dev);
    if (it != g_trace.end() && it->second.buf) {
      kp.trace = it->second.buf;
      kp.trace_cap = static_cast<int>(it->second.cap);
    }
  }
  if (g.k == 0) return fail(TF_ERR_INVALID, "K must be >= 1");
  if (g.moe_tab) return launch_grouped(g, kp, stream);

  const int cg = tile_m == 128 ? 1 : 2;
  const int mh = tile_m == 512 ? 2 : 1;
  if (mh == 2 && g.block_n != 256)
    return fail(TF_ERR_CONFIG, "block_m 512 requires block_n 256");
  CUtensorMap ta, tb;
  int rc = make_tmap_2d(&ta, g.a, g.m, g.k, g.lda, 128);
  if (rc) return rc;
  rc = make_tmap_2d(&tb, g.b, g.n, g.k, g.ldb, g.block_n / cg);
  if (rc) return rc;
  // C through TMA stores when rows are 16-byte aligned (else per-thread stores)
  CUtensorMap tc;
  std::memset(&tc, 0, sizeof(tc));
  kp.tma_store = 0;
  if (g.epilogue == 0 && kp.vec_ok && !getenv("TF_DEBUG_NO_TMA_STORE")) {
    const int esz_c = g.out_f32 ? 4 : 2;
    rc = make_tmap_2d(&tc, g.c, g.m, g.n, g.ldc, 32, esz_c, 128 / esz_c);
    if (rc) return rc;
    kp.tma_store = 1;
  }

  // 4-CTA clusters (two CTA pairs sharing A through TMA multicast) for the 512x256
  // pair tile when N splits into tile pairs; TF_GEMM_MC=0 keeps 2-CTA clusters
  int npair = 1;
  {
    const char* mc = getenv("TF_GEMM_MC");
    const bool want = mc ? atoi(mc) != 0 : kDefaultMulticast;
    if (want && mh == 2 && kp.num_pid_n % 2 == 0 && !g.wait_on_b && !g.tile_map_n) npair = 2;
  }
  kp.num_pid_n /= npair;  // work items are N-tile pairs
  const int tiles = kp.num_pid_m * kp.num_pid_n;
  int ctas = g.num_sms > 0 ? g.num_sms : num_sms_of_current_device();
  int clusters = ctas / (cg * npair);
  if (clusters < 1) clusters = 1;
  if (clusters > tiles) clusters = tiles;
  const int grid = clusters * cg * npair;
  // Split-K tail: when the last wave is at most half full, cut its tiles into
  // K-ranges so every cluster gets work (wave quantization on 148 SMs).
  kp.tail_base = tiles;
  kp.split_s = 1;
  kp.total_work = tiles;
  CUtensorMap tp;
  std::memset(&tp, 0, sizeof(tp));
  float* tail_ws = nullptr;
  {
    const int rem = tiles % clusters;
    int split = rem > 0 ? clusters / rem : 1;
    if (split > 8) split = 8;
    while (split > 1 && kp.num_kb / split < 4) --split;
    if (g.epilogue == 0 && tiles > clusters && rem > 0 && split >= 2 && !g.no_tail_split &&
        !g.wait_on_b &&
        !getenv("TF_DEBUG_NO_SPLITK")) {
      const int tile_m_rows = tile_m;
      const size_t bytes = static_cast<size_t>(rem) * split * npair * tile_m_rows * g.block_n * 4;
      tail_ws = tail_workspace(stream, bytes);
      if (tail_ws) {
        rc = make_tmap_2d(&tp, tail_ws, static_cast<int64_t>(rem) * split * npair * tile_m_rows,
                          g.block_n, g.block_n, 32, 4, 32);
        if (rc) return rc;
        kp.tail_base = tiles - rem;
        kp.split_s = split;
        kp.total_work = kp.tail_base + rem * split;
      }
    }
  }
  if (mh == 2 && npair == 2) return dispatch_bn<2, 2, 256, 2>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
  if (mh == 2) return dispatch_bn<2, 2, 256>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
  if (cg == 2) {
    if (g.block_n == 256) return dispatch_bn<2, 1, 256>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
    return dispatch_bn<2, 1, 128>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
  }
  if (g.block_n == 256) return dispatch_bn<1, 1, 256>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
  return dispatch_bn<1, 1, 128>(ta, tb, tc, tp, kp, grid, g, stream, tail_ws);
}

}  // namespace tf

// ---------------------------------------------------------------- trace C ABI
using tf::fail;
extern "C" {

int tf_trace_enable(int device, int64_t capacity) {
  if (capacity < 1 || capacity > (1 << 26)) return fail(TF_ERR_INVALID, "trace capacity out of range");
  std::lock_guard<std::mutex> lock(tf::g_trace_mu);
  auto& t = tf::g_trace[device];
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (t.buf) cudaFree(t.buf);
  t.buf = nullptr;
  const size_t bytes = (4 + static_cast<size_t>(capacity) * 4) * sizeof(unsigned long long);
  cudaError_t e = cudaMalloc(&t.buf, bytes);
  if (e == cudaSuccess) e = cudaMemset(t.buf, 0, bytes);
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(TF_ERR_CUDA, std::string("trace buffer: ") + cudaGetErrorString(e));
  t.cap = capacity;
  return TF_OK;
}

int tf_trace_disable(int device) {
  std::lock_guard<std::mutex> lock(tf::g_trace_mu);
  auto it = tf::g_trace.find(device);
  if (it != tf::g_trace.end() && it->second.buf) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    cudaFree(it->second.buf);
    cudaSetDevice(prev);
  }
  tf::g_trace.erase(device);
  return TF_OK;
}

int tf_trace_read(int device, uint64_t* host, int64_t capacity, int64_t* count) {
  std::lock_guard<std::mutex> lock(tf::g_trace_mu);
  auto it = tf::g_trace.find(device);
  if (it == tf::g_trace.end() || !it->second.buf) return fail(TF_ERR_INVALID, "tracing is not enabled");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  unsigned long long n = 0;
  cudaError_t e = cudaMemcpy(&n, it->second.buf, sizeof(n), cudaMemcpyDeviceToHost);
  if (n > static_cast<unsigned long long>(it->second.cap)) n = it->second.cap;
  if (n > static_cast<unsigned long long>(capacity)) n = capacity;
  if (e == cudaSuccess && n)
    e = cudaMemcpy(host, it->second.buf + 4, n * 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(it->second.buf, 0, sizeof(unsigned long long));
  cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(TF_ERR_CUDA, std::string("trace read: ") + cudaGetErrorString(e));
  *count = static_cast<int64_t>(n);
  return TF_OK;
}

}  // extern "C"
