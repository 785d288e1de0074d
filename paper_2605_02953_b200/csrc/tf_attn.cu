// AllGather-KV fused with flash-attention forward (BASELINE config 3; SURVEY
// §8(f) #2, the fused continuation of row A13).
//
//   O[q, h, :] = softmax(Q[q, h, :] . K_all[:, g(h), :]^T * scale) . V_all[:, g(h), :]
//
// The K/V shards are gathered into the symmetric workspace with the AG pull
// protocol (ovs/kernels/ag_gemm.py:55-69): local copy + flag, copy-engine pulls
// of chunk (rank+i)%w, one flag per source chunk.  One CTA per (128-query tile,
// head); it walks the key tiles starting at its own chunk (gather order) and
// acquire-waits a chunk's flag before its first TMA load of that chunk.
//
// Per CTA (320 threads, two 128-query tiles A and B of one head):
//   warp 0      TMA: Q_A and Q_B once, then K_j and V_j (128 keys x 128 dims each)
//               through a 5-slot ring (K0 V0 K1 V1 ...).
//   warp 1      MMA (one lane), per tile t: S_t(0) = Q_t K_0^T, then for every key
//               tile j: O_t += P_t(j) V_j (A = P_t from TMEM, B = V from smem,
//               MN-major) followed by S_t(j+1) into the same TMEM columns -- the
//               in-order tensor pipe reads P_t(j) before S_t(j+1) overwrites it.
//   warps 2-5   softmax of tile A, warps 6-9 softmax of tile B, one query row per
//               thread: S row from TMEM, online max/sum in fp32 (ex2.approx with
//               the scale folded into an FFMA), lazy rescale -- the running max
//               may lag the true max by up to 2^8 before O is rescaled in TMEM --
//               P packed to bf16 over the first 64 columns of S_t, O / l as bf16.
// While one warpgroup is on the ALUs/SFU the tensor pipe works on the other
// tile's QK^T and PV.  TMEM: S/P_A [0,128), S/P_B [128,256), O_A [256,384),
// O_B [384,512).  An opt-in CTA-pair variant (TF_ATTN_PAIR=1) splits K and V
// across two CTAs with cta_group::2 MMAs.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

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

constexpr int kQT = 128;      // queries per tile (two tiles per CTA)
constexpr int kKT = 128;      // keys per tile
constexpr int kD = 128;       // head dim (fixed for this kernel)
constexpr int kHalf = 16384;  // one 128-row x 64-col bf16 box (128-byte rows)

struct AttnParams {
  int s_local, s_total, hq, hkv;
  int n_tiles;              // key tiles over s_total
  int start_tile;           // gather order: first key tile of this rank's own chunk
  int tiles_per_chunk;
  float scale_log2;         // softmax scale * log2(e)
  void* out;                // [s_local, hq, d] bf16
  const uint64_t* chunk_flags;
  unsigned long long epoch;
  unsigned long long* err;
  unsigned long long timeout_ns;
  // direct mode: K/V tiles of chunk c are read over NVLink straight from rank c's
  // workspace through chunk_maps[c] (K) / chunk_maps[nchunks + c] (V), once rank c's
  // own flag peer_flags[c] reaches the epoch -- no staging copy
  int direct, nchunks;
  const CUtensorMap* chunk_maps;
  const uint64_t* peer_flags[kMaxWorld];
  const void* q;            // [s_local, hq, d] bf16 (the pair kernel stages Q rows into TMEM)
};

// Two 128-query tiles (A, B) per CTA share every K/V tile; each has its own
// softmax warpgroup, S and O in TMEM, and P buffer in smem, so the tensor pipe
// runs one tile's QK^T / PV while the other tile's softmax is on the ALUs.
// TF_ATTN_SPLIT_ROWS=2 (opt-in): eight softmax warps per query tile, two per TMEM lane
// quarter, each taking 64 of a row's 128 keys (the row max combined through shared
// memory).  Measured slower than four warps per tile (3.89 vs 3.47 ms per rank).
#ifndef TF_ATTN_SPLIT_ROWS
#define TF_ATTN_SPLIT_ROWS 1  // 2 measured slower: 3.89 vs 3.47 ms per rank (same box)
#endif
constexpr int kRowSplit = TF_ATTN_SPLIT_ROWS;
#if defined(TF_ATTN_EARLY_S) && TF_ATTN_EARLY_S && TF_ATTN_SPLIT_ROWS == 2
#error "TF_ATTN_EARLY_S needs the four-warp softmax (TF_ATTN_SPLIT_ROWS=1)"
#endif
struct AttnSmem {
  static constexpr int kQ = 2 * kHalf;        // one Q tile, 32 KB
  static constexpr int kSlot = 2 * kHalf;     // one K or V tile (128 keys x 128 dims), 32 KB
  static constexpr int kSlots = 5;            // ring K0 V0 K1 V1 ...
  static constexpr int kBars = 256;
  // row-max halves, bf16 [j & 1][tile][half][row] (the same two values give every warp of a
  // row the same max); reused as fp32 [tile][half][row] row sums at the end
  static constexpr int kXchg = kRowSplit == 2 ? 2 * 2 * 2 * 128 * 2 : 0;
  // no alignment slack in the split variant (dynamic smem starts 1 KB-aligned: checked)
  static constexpr int kSlack = kRowSplit == 2 ? 0 : 1024;
  static constexpr int kTotal = kSlack + 2 * kQ + kSlots * kSlot + kBars + kXchg;
};
constexpr int kAttnThreads2 = 64 + 2 * 4 * kRowSplit * 32;  // TMA, MMA, 2 tiles x 4 x split softmax warps
constexpr float kLazyRescale = 8.0f;          // log2 units the running max may lag (FA4)

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const void* tmap, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// MN-major, 128-byte-swizzled operand (V as the B operand of P.V): 64 MN
// elements per 128-byte row, MN blocks `lbo` bytes apart, 8-row K groups 1024 B.
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFF) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
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

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


// position of K_j (kv = 0) / V_j (kv = 1) in the ring's load sequence K0 K1 V0 K2 V1 ...
__device__ __forceinline__ int ring_index(int j, int kv, int n) {
  if (!kv) return j == 0 ? 0 : 2 * j - 1;
  return j <= n - 2 ? 2 * j + 2 : 2 * n - 1;
}
__device__ __forceinline__ void ring_decode(int c, int n, int& j, int& kv) {
  if (c == 0) { j = 0; kv = 0; return; }
  if (c == 2 * n - 1) { j = n - 1; kv = 1; return; }
  if (c & 1) { j = (c + 1) / 2; kv = 0; } else { j = (c - 2) / 2; kv = 1; }
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (FA4's trick to offload the SFU): k = round(x) through the
// 1.5 * 2^23 magic add, 2^(x-k) by a degree-3 polynomial on [-0.5, 0.5] (rel. error
// < 1e-4, below bf16's 2^-8), and k added straight into the exponent bits.
#ifndef TF_ATTN_SPLIT_P
#define TF_ATTN_SPLIT_P 1  // release P's first 64 keys to the MMA before the rest
#endif
#ifndef TF_ATTN_MMA_POLL
#define TF_ATTN_MMA_POLL 0
#endif
#if TF_ATTN_MMA_POLL == 1
#define MMA_WAIT mbar_wait_poll
#elif TF_ATTN_MMA_POLL == 2
#define MMA_WAIT mbar_wait
#else
#define MMA_WAIT mbar_wait_spin
#endif
#ifndef TF_ATTN_SM_SLEEP
#define TF_ATTN_SM_SLEEP 0
#endif
#if TF_ATTN_SM_SLEEP
#define SM_WAIT mbar_wait
#else
#define SM_WAIT mbar_wait_spin
#endif
// TF_ATTN_EARLY_S=1: P_t(j) lives in the upper 64 columns of S_t, so QK^T for keys
// 0-63 of tile j+1 (N=64, into the lower 64 columns) is issued as soon as the softmax
// has read S_t(j) into registers ("S free"), overlapping the exponentials; only keys
// 64-127 of S_t(j+1) still wait behind PV_t(j) on the in-order tensor pipe
// Measured slower (session 3, one box): 3.88-3.90 vs 3.54-3.62 ms per rank -- the two
// N=64 halves read Q from shared memory twice, and QK^T is shared-memory bound here.
#ifndef TF_ATTN_EARLY_S
#define TF_ATTN_EARLY_S 0
#endif
#ifndef TF_ATTN_STAGGER
#define TF_ATTN_STAGGER 0  // per-CTA rotation inside a chunk: measured neutral (no L2 hot spot)
#endif
#ifndef TF_EXP2_EMU_MASK
#define TF_EXP2_EMU_MASK 7  // 1 pair in 8 on the FMA pipe (12.5%): 3.63 vs 3.70 ms; 25% is slower (3.84)
#endif
__device__ __forceinline__ float ex2_fma(float x) {
  const float y = fmaxf(x, -126.f);
  const float t = y + 12582912.f;
  const float f = y - (t - 12582912.f);
  const float pl = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
  return __int_as_float(__float_as_int(pl) + (__float_as_int(t) << 23));
}

// Blackwell paired-fp32 ops (FFMA2 / FADD2) and the 3-input max (FMNMX3): the
// softmax is issue-bound, these halve its FMA/ADD/MAX instruction count.
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// two 2^x on the FMA pipe with paired ops (same polynomial as ex2_fma)
__device__ __forceinline__ void ex2_fma2(float x0, float x1, float& r0, float& r1) {
  const uint64_t y = f2pack(fmaxf(x0, -126.f), fmaxf(x1, -126.f));
  const uint64_t t = fadd2(y, f2pack(12582912.f, 12582912.f));
  const uint64_t k = fadd2(t, f2pack(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(k, f2pack(-1.f, -1.f), y);
  uint64_t pl = ffma2(f2pack(0.0555041f, 0.0555041f), f, f2pack(0.2402265f, 0.2402265f));
  pl = ffma2(pl, f, f2pack(0.6931472f, 0.6931472f));
  pl = ffma2(pl, f, f2pack(1.0f, 1.0f));
  float p0, p1, t0, t1;
  f2unpack(pl, p0, p1);
  f2unpack(t, t0, t1);
  r0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  r1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// Warp-converged issue: every lane runs the MMA loop (so descriptor math stays on
// the uniform datapath) and elect.sync picks the one lane that issues.
__device__ __forceinline__ void umma_ss_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// cta_group::2 forms of the warp-converged issue helpers (the leader CTA's MMA warp)
__device__ __forceinline__ void umma_ss_pair_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                   uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_ts_pair_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                   uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_mc_elect(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T: the A operand (P, bf16 pairs packed per 32-bit
// column, rows = lanes) is read from tensor memory, so P never touches shared memory
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

#ifdef TF_ATTN_TRACE
// debug: SM clock stamps of CTA (0, 0) per key tile: [j][0..1] softmax t got S,
// [2..3] softmax t released P, [4..5] MMA issued PV_t, [6..7] MMA issued S_t(j+1),
// [8] MMA has V_j and K_j+1, [9] producer issues K_j, [10] producer issues V_j
__device__ long long g_attn_trace[512][20];
#define ATTN_STAMP(j, e) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && (j) < 512) g_attn_trace[j][e] = clock64(); } while (0)
// cross-SM (globaltimer ns) stamps of the first CTA pair: slots 10 + 5 * cta + e
#define ATTN_GSTAMP(j, e) \
  do { if (blockIdx.x < 2 && blockIdx.y == 0 && (j) < 512) g_attn_trace[j][10 + 5 * blockIdx.x + (e)] = globaltimer_ns(); } while (0)
#else
#define ATTN_STAMP(j, e) do { } while (0)
#define ATTN_GSTAMP(j, e) do { } while (0)
#endif

__global__ void __launch_bounds__(kAttnThreads2, 1)
    ag_attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ AttnParams p) {
  using S = AttnSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  if constexpr (S::kSlack == 0) {
    if (smem != smem_raw) __trap();  // the layout above has no room to realign
  }
  uint8_t* sq = smem;                               // Q_A, Q_B
  uint8_t* sring = sq + 2 * S::kQ;                  // 5 slots: K0 V0 K1 V1 ...
  uint64_t* bars = reinterpret_cast<uint64_t*>(sring + S::kSlots * S::kSlot);
  uint64_t* q_full = bars;
  uint64_t* r_full = bars + 1;     // [5]
  uint64_t* r_empty = bars + 6;    // [5]
  uint64_t* s_full = bars + 11;    // [2] per Q tile
  uint64_t* p_full = bars + 13;    // [2]
  uint64_t* o_ready = bars + 15;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  uint64_t* p_half = bars + 18;    // [2] first 64 keys of P_t written
  uint64_t* s_free = bars + 20;    // [2] S_t(j) read into the softmax registers (TF_ATTN_EARLY_S)
  constexpr uint32_t kPCol = TF_ATTN_EARLY_S ? 64 : 0;  // P_t's first column inside S_t

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 2 * kQT;
  const bool has_b = q0 + kQT < p.s_local;
  const int nq = has_b ? 2 : 1;
  const int h = blockIdx.y;
  const int g = h / (p.hq / p.hkv);
  const int n = p.n_tiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < S::kSlots; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_half[i], 4 * kRowSplit);  // split: half-1 warps also report "O rescaled"
      mbar_init(&o_ready[i], 1);
      mbar_init(&s_free[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // TMEM: S_A [0,128) S_B [128,256) (P_t packed bf16 in the first 64 columns of S_t),
  //       O_A [256,384) O_B [384,512)
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, nq * S::kQ);
      for (int t = 0; t < nq; ++t) {
        tma_load_3d(sq + t * S::kQ, &tq, q_full, 0, h, q0 + t * kQT);
        tma_load_3d(sq + t * S::kQ + kHalf, &tq, q_full, 64, h, q0 + t * kQT);
      }
      uint32_t ready = 0;
      // gather order: own chunk first, chunks in rank order; inside a chunk each CTA
      // starts at its own offset so the CTAs sharing a KV head do not all request the
      // same tile from L2 at once (same-line hot spots stretched loads to ~3.6k clk)
      const int tpc = p.tiles_per_chunk;
      const int rot = TF_ATTN_STAGGER ? static_cast<int>((blockIdx.x * 8 + blockIdx.y % 8) % tpc) : 0;
      for (int c = 0; c < 2 * n; ++c) {  // K_j = 2j, V_j = 2j + 1
        const int j = c >> 1, kv = c & 1;
        const int kt = ((p.start_tile / tpc + j / tpc) % (n / tpc)) * tpc + (rot + j) % tpc;
        const int chunk = kt / p.tiles_per_chunk;
        if (!kv && !(ready & (1u << chunk)) && (p.direct || p.chunk_flags)) {
          const uint64_t* f = p.direct ? p.peer_flags[chunk] : p.chunk_flags + chunk;
          wait_geq_sys(f, p.epoch, p.timeout_ns, p.err, 0x1000000ull | static_cast<unsigned>(chunk));
          fence_proxy_async_global();
          ready |= 1u << chunk;
        }
        const int sl = c % S::kSlots;
        mbar_wait(&r_empty[sl], ((c / S::kSlots) & 1) ^ 1);
        uint8_t* dst = sring + sl * S::kSlot;
        const CUtensorMap* m = p.direct ? p.chunk_maps + kv * p.nchunks + chunk : (kv ? &tv : &tk);
        const int row = p.direct ? (kt - chunk * p.tiles_per_chunk) * kKT : kt * kKT;
        mbar_arrive_expect_tx(&r_full[sl], S::kSlot);
        ATTN_STAMP(j, 9 + kv);
        tma_load_3d(dst, m, &r_full[sl], 0, g, row);
        tma_load_3d(dst + kHalf, m, &r_full[sl], 64, g, row);
      }
    }
  } else if (warp == 1) {
    // per Q tile t: S_t(0); then for each j: PV_t(j) (A = P_t from TMEM), S_t(j+1) into the
    // same columns -- issued in that order, the tensor pipe reads P_t(j) before S_t(j+1)
    // overwrites it, and S_t(j+1) completing implies PV_t(j) completed (O_t is stable for
    // the softmax's rescale)
    constexpr uint32_t idesc_s = umma_idesc_bf16(kQT, kKT);
    constexpr uint32_t idesc_pv = umma_idesc_bf16(kQT, kD) | (1u << 16);  // B (V) MN-major
    {  // all 32 lanes: uniform control flow, one elected lane issues
      MMA_WAIT(q_full, 0);
      tc_fence_after();
      // descriptors as (low word + compile-time delta, constant high word): the per-MMA
      // address math is one add, so the single MMA thread issues without long gaps
      // (it shares its SMSP with two softmax warps)
      constexpr uint32_t kDescHi = (1024 >> 4) | (1u << (46 - 32)) | (2u << (61 - 32));
      constexpr uint32_t kLoK = 1u << 16;                    // K-major SW128, LBO field 1
      constexpr uint32_t kLoV = ((kHalf >> 4) & 0x3FFF) << 16;  // MN-major V, LBO = kHalf
      auto mk = [](uint32_t lo) {
        uint64_t d;
        asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(kDescHi));
        return d;
      };
      const uint32_t q_lo0 = ((smem_u32(sq) & 0x3FFFF) >> 4) | kLoK;
      const uint32_t ring_lo = (smem_u32(sring) & 0x3FFFF) >> 4;
      auto issue_s = [&](int t, int sl) {
        const uint32_t qa = q_lo0 + t * (S::kQ >> 4);
        const uint32_t kb = (ring_lo + sl * (S::kSlot >> 4)) | kLoK;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kHalf >> 4) + (kk & 3) * 2;
          umma_ss_elect(tmem + t * 128, mk(qa + off), mk(kb + off), idesc_s, kk != 0);
        }
        umma_commit_elect(&s_full[t]);
      };
      // keys [64 hf, 64 hf + 64) of S_t into columns [64 hf, +64) (no commit)
      constexpr uint32_t idesc_s64 = umma_idesc_bf16(kQT, kKT / 2);
      auto issue_s_half = [&](int t, int sl, int hf) {
        const uint32_t qa = q_lo0 + t * (S::kQ >> 4);
        const uint32_t kb = (ring_lo + sl * (S::kSlot >> 4) + hf * ((64 * 128) >> 4)) | kLoK;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (kHalf >> 4) + (kk & 3) * 2;
          umma_ss_elect(tmem + t * 128 + hf * 64, mk(qa + off), mk(kb + off), idesc_s64, kk != 0);
        }
      };
      (void)issue_s_half;
      MMA_WAIT(&r_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < nq; ++t) issue_s(t, 0);
      umma_commit_elect(&r_empty[0]);
      for (int j = 0; j < n; ++j) {
        const int cv = 2 * j + 1, vs = cv % S::kSlots;
        const int ck = 2 * j + 2, ks = ck % S::kSlots;
        MMA_WAIT(&r_full[vs], (cv / S::kSlots) & 1);
        ATTN_STAMP(j, 11);
        if (j + 1 < n) MMA_WAIT(&r_full[ks], (ck / S::kSlots) & 1);
        ATTN_STAMP(j, 8);
        const uint32_t vb = (ring_lo + vs * (S::kSlot >> 4)) | kLoV;
        for (int t = 0; t < nq; ++t) {
          const uint32_t pa = tmem + t * 128 + kPCol, od = tmem + 256 + t * 128;
#if TF_ATTN_EARLY_S
          if (j + 1 < n) {  // S_t(j+1) keys 0-63 while the softmax works on S_t(j)
            MMA_WAIT(&s_free[t], j & 1);
            tc_fence_after();
            issue_s_half(t, ks, 0);
          }
#endif
          // keys 0-63 of P_t(j) as soon as the softmax has them, keys 64-127 after
          if (t == 0) ATTN_STAMP(j, 16);
          MMA_WAIT(&p_half[t], j & 1);
          if (t == 0) ATTN_STAMP(j, 17);
          tc_fence_after();
          ATTN_STAMP(j, 4 + t);
#pragma unroll
          for (int kk = 0; kk < kKT / 32; ++kk)
            umma_ts_elect(od, pa + kk * 8, mk(vb + kk * (2048 >> 4)), idesc_pv, (j | kk) != 0);
          MMA_WAIT(&p_full[t], j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = kKT / 32; kk < kKT / 16; ++kk)
            umma_ts_elect(od, pa + kk * 8, mk(vb + kk * (2048 >> 4)), idesc_pv, 1);
          ATTN_STAMP(j, 6 + t);
#if TF_ATTN_EARLY_S
          if (j + 1 < n) {
            issue_s_half(t, ks, 1);  // over P_t(j): the pipe has read it for PV_t(j)
            umma_commit_elect(&s_full[t]);
          } else {
            umma_commit_elect(&o_ready[t]);
          }
#else
          if (j + 1 < n) issue_s(t, ks);
          else umma_commit_elect(&o_ready[t]);
#endif
        }
        umma_commit_elect(&r_empty[vs]);
        if (j + 1 < n) umma_commit_elect(&r_empty[ks]);
      }
    }
    __syncwarp();
  } else if constexpr (kRowSplit == 2) {
    // two warps per TMEM lane quarter and tile: half h takes keys / O columns [64h, 64h+64)
    const int t = (warp - 2) >> 3;                 // Q tile of this warp
    const int half = ((warp - 2) >> 2) & 1;
    if (t < nq) {
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
      const uint32_t t_s = tmem + lane_off + t * 128;
      const uint32_t t_o = tmem + lane_off + 256 + t * 128 + half * 64;
      // [j & 1][tile][half][row] bf16 row maxima, rounded up (both warps of a row then
      // derive the same max from the same two values)
      __nv_bfloat16* xm = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<uint8_t*>(bars) + S::kBars);
      const uint32_t bar_id = 1 + t * 4 + quarter;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        SM_WAIT(&s_full[t], j & 1);
        tc_fence_after();
        uint32_t sv[2][32];
        tmem_ld_32x32b_x32(t_s + half * 64, sv[0]);
        tmem_ld_32x32b_x32(t_s + half * 64 + 32, sv[1]);
        tmem_ld_wait();
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            mx[c] = fmax3(mx[c], __uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1]));
        __nv_bfloat16* x = xm + ((j & 1) * 2 + t) * 256;
        x[half * 128 + row] = __float2bfloat16_ru(fmaxf(mx[0], mx[1]));
        // both warps of these rows hold their S in registers from here on (P may overwrite S)
        asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
        const float mt = fmaxf(__bfloat162float(x[row]), __bfloat162float(x[128 + row])) * p.scale_log2;
        float alpha = 1.f;
        if (mt > m + kLazyRescale) {
          alpha = ex2(m - mt);
          m = mt;
        }
        // O_t is stable (S_t(j) complete implies PV_t(j-1) complete): rescale this half
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[16];
            tmem_ld_32x32b_x16(t_o + c * 16, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_32x32b_x16(t_o + c * 16, ov);
          }
          tmem_st_wait();
        }
        if (half == 1) {  // "O rescaled" for the first PV half (keys 0-63 come from half 0)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_half[t]);
        }
        uint64_t sum2 = f2pack(0.f, 0.f);
        const uint64_t scale2 = f2pack(p.scale_log2, p.scale_log2), negm2 = f2pack(-m, -m);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float a0, a1;
            f2unpack(ffma2(f2pack(__uint_as_float(sv[c][2 * i]), __uint_as_float(sv[c][2 * i + 1])), scale2,
                           negm2),
                     a0, a1);
            float p0, p1;
            if (TF_EXP2_EMU_MASK >= 0 && (i & TF_EXP2_EMU_MASK) == 0) {
              ex2_fma2(a0, a1, p0, p1);
            } else {
              p0 = ex2(a0);
              p1 = ex2(a1);
            }
            sum2 = fadd2(sum2, f2pack(p0, p1));
            sv[0][c * 16 + i] = pack_bf16x2(p0, p1);
          }
        tmem_st_32x32b_x32(t_s + half * 32, sv[0]);  // P keys [64 half, +64) as bf16 pairs
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(half == 0 ? &p_half[t] : &p_full[t]);
        float s0, s1;
        f2unpack(sum2, s0, s1);
        l = l * alpha + (s0 + s1);
      }
      mbar_wait_spin(&o_ready[t], 0);
      tc_fence_after();
      // row sums through this tile's own exchange slots ([parity h][tile t] holds half h's
      // 128 floats): the other tile's warps may still be in their loop
      float* lsum = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + S::kBars);
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      lsum[(half * 2 + t) * 128 + row] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
      const float inv = 1.f / (lsum[t * 128 + row] + lsum[(2 + t) * 128 + row]);
      const int q = q0 + t * kQT + row;
      uint16_t* dst = static_cast<uint16_t*>(p.out) + (static_cast<long long>(q) * p.hq + h) * kD + half * 64;
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(t_o + c * 32, ov);
        tmem_ld_wait();
        if (q < p.s_local) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            d4[i] = make_uint4(pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
        }
      }
    }
  } else {
    const int t = (warp - 2) >> 2;                 // Q tile of this warpgroup
    if (t < nq) {
      const int quarter = warp & 3;
      const int row = quarter * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
      const uint32_t t_s = tmem + lane_off + t * 128;
      const uint32_t t_o = tmem + lane_off + 256 + t * 128;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        SM_WAIT(&s_full[t], j & 1);
        tc_fence_after();
        if (threadIdx.x % 128 == 64) ATTN_STAMP(j, t);
        uint32_t sv[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(t_s + c * 32, sv[c]);
        tmem_ld_wait();
#if TF_ATTN_EARLY_S
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_free[t]);  // the MMA may overwrite S_t's lower columns
#endif
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 2)
            mx[c] = fmax3(mx[c], __uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1]));
        const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
        // lazy rescale: keep a stale running max unless the new one exceeds it by > 8
        float alpha = 1.f;
        if (mt > m + kLazyRescale) {
          alpha = ex2(m - mt);
          m = mt;
        }
        // O_t is stable: S_t(j) completing implies PV_t(j-1) completed; rescale before any
        // part of P_t(j) is released to the MMA
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 8; ++c) {
            uint32_t ov[16];
            tmem_ld_32x32b_x16(t_o + c * 16, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_32x32b_x16(t_o + c * 16, ov);
          }
        }
        uint64_t sum2 = f2pack(0.f, 0.f);
        const uint64_t scale2 = f2pack(p.scale_log2, p.scale_log2), negm2 = f2pack(-m, -m);
        // P row packed in place of the first 64 S columns (the whole row is in registers),
        // in two halves of 64 keys: PV on the first half overlaps the second half's exps
#pragma unroll
        for (int hk = 0; hk < 2; ++hk) {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = 2 * hk + cc;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float a0, a1;
              f2unpack(ffma2(f2pack(__uint_as_float(sv[c][2 * i]), __uint_as_float(sv[c][2 * i + 1])),
                             scale2, negm2), a0, a1);
              const bool emu = TF_EXP2_EMU_MASK >= 0 && (i & TF_EXP2_EMU_MASK) == 0;
#ifdef TF_ATTN_EXP_CHEAP  // bottleneck experiment: no SFU work
              const float p0 = a0 * 0.001f, p1 = a1 * 0.001f;
              (void)emu;
#else
              float p0, p1;
              if (emu) {
                ex2_fma2(a0, a1, p0, p1);
              } else {
                p0 = ex2(a0);
                p1 = ex2(a1);
              }
#endif
              sum2 = fadd2(sum2, f2pack(p0, p1));
              sv[hk][cc * 16 + i] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st_32x32b_x32(t_s + kPCol + hk * 32, sv[hk]);
#if TF_ATTN_SPLIT_P
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(hk == 0 ? &p_half[t] : &p_full[t]);
          if (hk == 1 && threadIdx.x % 128 == 64) ATTN_STAMP(j, 2 + t);
          if (hk == 1 && threadIdx.x % 128 == 0) ATTN_STAMP(j, 14 + t);
          if (hk == 1 && threadIdx.x % 128 == 32) ATTN_STAMP(j, 12 + t);
#else
          if (hk == 1) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&p_half[t]);
              mbar_arrive(&p_full[t]);
            }
          }
#endif
        }
        float s0, s1;
        f2unpack(sum2, s0, s1);
        l = l * alpha + (s0 + s1);
      }
      mbar_wait_spin(&o_ready[t], 0);
      tc_fence_after();
      const float inv = 1.f / l;
      const int q = q0 + t * kQT + row;
      uint16_t* dst = static_cast<uint16_t*>(p.out) + (static_cast<long long>(q) * p.hq + h) * kD;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t ov[32];
        tmem_ld_32x32b_x32(t_o + c * 32, ov);
        tmem_ld_wait();
        if (q < p.s_local) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            d4[i] = make_uint4(pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
                               pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
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


// ---------------------------------------------------------------- CTA-pair variant
// A cluster of two CTAs runs four 128-query tiles (two per CTA) against the same
// key/value tiles with cta_group::2 MMAs issued by the leader: S_t = [Q_t(cta0);
// Q_t(cta1)] K^T is one M=256 MMA whose B operand (the 128 keys) is split 64/64
// between the two CTAs' shared memory, and O_t += P_t V is one M=256 TS-MMA (P_t
// from each CTA's TMEM) whose B operand (V, N = 128 dims) is split 64/64.  Each CTA
// therefore stages only half of every K and V tile, which halves the shared-memory
// operand traffic of Q K^T -- the limiter of the single-CTA kernel.
struct AttnPairSmem {
  static constexpr int kQ = 2 * kHalf;        // one Q tile, 32 KB
  static constexpr int kSlot = 16384;         // half a K tile (64 keys x 128 dims) or half a V tile (128 keys x 64 dims)
  static constexpr int kSlots = 10;
  static constexpr int kBars = 256;
  static constexpr int kTotal = 1024 + 2 * kQ + kSlots * kSlot + kBars;
};

__device__ __forceinline__ void tma_load_3d_pair(void* smem_dst, const void* tmap, uint64_t* bar,
                                                 int32_t c0, int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__global__ void __maxnreg__(168)
    ag_attn_fwd_pair_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                            const __grid_constant__ CUtensorMap tv, const __grid_constant__ AttnParams p) {
  using S = AttnPairSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sq = smem;                               // Q_A, Q_B of this CTA
  uint8_t* sring = sq + 2 * S::kQ;                  // K0 V0 K1 V1 ... halves
  uint64_t* bars = reinterpret_cast<uint64_t*>(sring + S::kSlots * S::kSlot);
  uint64_t* q_full = bars;         // leader: both CTAs' Q bytes
  uint64_t* r_full = bars + 1;     // [10] leader: both halves of a K or V tile
  uint64_t* r_empty = bars + 11;   // [10] each CTA (multicast commits)
  uint64_t* s_full = bars + 21;    // [2] each CTA (multicast commits)
  uint64_t* p_full = bars + 23;    // [2] leader: 4 softmax warps x 2 CTAs
  uint64_t* o_ready = bars + 25;   // [2] each CTA (multicast commits)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 27);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int q0 = (blockIdx.x >> 1) * 4 * kQT + static_cast<int>(cta) * 2 * kQT;  // this CTA's two tiles
  const int h = blockIdx.y;
  const int g = h / (p.hq / p.hkv);
  const int n = p.n_tiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < S::kSlots; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
      mbar_init(&o_ready[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  // TMEM (each CTA, its 128 query rows): S/P_A [0,128) S/P_B [128,256) O_A [256,384) O_B [384,512)
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      if (leader) mbar_arrive_expect_tx(q_full, 2 * 2 * S::kQ);
      for (int t = 0; t < 2; ++t) {
        tma_load_3d_pair(sq + t * S::kQ, &tq, q_full, 0, h, q0 + t * kQT);
        tma_load_3d_pair(sq + t * S::kQ + kHalf, &tq, q_full, 64, h, q0 + t * kQT);
      }
      uint32_t ready = 0;
      for (int c = 0; c < 2 * n; ++c) {  // K_j = 2j, V_j = 2j + 1
        const int j = c >> 1, kv = c & 1;
        const int kt = (p.start_tile + j) % n;     // gather order: own chunk first
        const int chunk = kt / p.tiles_per_chunk;
        if (!kv && p.chunk_flags && !(ready & (1u << chunk))) {
          wait_geq_sys(p.chunk_flags + chunk, p.epoch, p.timeout_ns, p.err,
                       0x1000000ull | static_cast<unsigned>(chunk));
          fence_proxy_async_global();
          ready |= 1u << chunk;
        }
        const int sl = c % S::kSlots;
        mbar_wait(&r_empty[sl], ((c / S::kSlots) & 1) ^ 1);
        uint8_t* dst = sring + sl * S::kSlot;
        if (leader) mbar_arrive_expect_tx(&r_full[sl], 2 * S::kSlot);
        if (!kv) {  // this CTA's 64 keys of K_j, all 128 dims (two 64-dim boxes)
          const int row = kt * 128 + static_cast<int>(cta) * 64;
          tma_load_3d_pair(dst, &tk, &r_full[sl], 0, g, row);
          tma_load_3d_pair(dst + 8192, &tk, &r_full[sl], 64, g, row);
        } else {    // all 128 keys of V_j, this CTA's 64 dims
          tma_load_3d_pair(dst, &tv, &r_full[sl], static_cast<int>(cta) * 64, g, kt * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(2 * kQT, 128);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(2 * kQT, kD) | (1u << 16);  // B (V) MN-major
      auto issue_s = [&](int t, int sl) {
        const uint32_t qa = smem_u32(sq + t * S::kQ);
        const uint32_t kb = smem_u32(sring + sl * S::kSlot);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          umma_bf16_pair(tmem + t * 128, umma_desc_k_sw128(qa + (kk >> 2) * kHalf + (kk & 3) * 32),
                         umma_desc_k_sw128(kb + (kk >> 2) * 8192 + (kk & 3) * 32), idesc_s, kk != 0);
        umma_commit_pair_mc(&s_full[t], 0x3);
      };
      mbar_wait_spin(q_full, 0);
      mbar_wait_spin(&r_full[0], 0);
      tc_fence_after();
      for (int t = 0; t < 2; ++t) issue_s(t, 0);
      umma_commit_pair_mc(&r_empty[0], 0x3);
      for (int j = 0; j < n; ++j) {
        const int cv = 2 * j + 1, vs = cv % S::kSlots;
        const int ck = 2 * j + 2, ks = ck % S::kSlots;
        mbar_wait_spin(&r_full[vs], (cv / S::kSlots) & 1);
        if (j + 1 < n) mbar_wait_spin(&r_full[ks], (ck / S::kSlots) & 1);
        for (int t = 0; t < 2; ++t) {
          mbar_wait_spin(&p_full[t], j & 1);
          tc_fence_after();
          const uint32_t vb = smem_u32(sring + vs * S::kSlot);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts_pair(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                              umma_desc_mn_sw128(vb + kk * 2048, 16384), idesc_pv, (j | kk) != 0);
          if (j + 1 < n) issue_s(t, ks);
          else umma_commit_pair_mc(&o_ready[t], 0x3);
        }
        umma_commit_pair_mc(&r_empty[vs], 0x3);
        if (j + 1 < n) umma_commit_pair_mc(&r_empty[ks], 0x3);
      }
    }
    __syncwarp();
  } else {
    const int t = (warp - 2) >> 2;                 // Q tile of this warpgroup
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t t_s = tmem + lane_off + t * 128;
    const uint32_t t_o = tmem + lane_off + 256 + t * 128;
    const uint32_t p_full_leader = mapa_shared(smem_u32(&p_full[t]), 0);
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      mbar_wait_spin(&s_full[t], j & 1);
      tc_fence_after();
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(t_s + c * 32, sv[c]);
      tmem_ld_wait();
      float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) mx[i & 3] = fmaxf(mx[i & 3], __uint_as_float(sv[c][i]));
      const float mt = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * p.scale_log2;
      float alpha = 1.f;
      if (mt > m + kLazyRescale) {
        alpha = ex2(m - mt);
        m = mt;
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t ov[16];
          tmem_ld_32x32b_x16(t_o + c * 16, ov);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st_32x32b_x16(t_o + c * 16, ov);
        }
      }
      float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = ex2(fmaf(__uint_as_float(sv[c][2 * i]), p.scale_log2, -m));
          const float p1 = ex2(fmaf(__uint_as_float(sv[c][2 * i + 1]), p.scale_log2, -m));
          sacc[i & 3] += p0 + p1;
          sv[c >> 1][(c & 1) * 16 + i] = pack_bf16x2(p0, p1);
        }
      l = l * alpha + ((sacc[0] + sacc[1]) + (sacc[2] + sacc[3]));
      tmem_st_32x32b_x32(t_s, sv[0]);
      tmem_st_32x32b_x32(t_s + 32, sv[1]);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(p_full_leader);
    }
    mbar_wait_spin(&o_ready[t], 0);
    tc_fence_after();
    const float inv = 1.f / l;
    const int q = q0 + t * kQT + row;
    uint16_t* dst = static_cast<uint16_t*>(p.out) + (static_cast<long long>(q) * p.hq + h) * kD;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32b_x32(t_o + c * 32, ov);
      tmem_ld_wait();
      if (q < p.s_local) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

// ---------------------------------------------------------------- CTA-pair, S double-buffered
// A cluster of two CTAs runs ONE 128-query tile per CTA (256 rows per pair) with
// cta_group::2 MMAs issued by the leader: S(j) = Q K_j^T is one M=256 MMA whose B
// operand (128 keys) is split 64/64 across the two CTAs' shared memory, O += P(j) V_j
// one M=256 TS-MMA (P from each CTA's TMEM, V's 128 dims split 64/64).  With one
// query tile per CTA, TMEM holds THREE S buffers next to O (S0, S1, S2, O = 4 x 128
// columns), so the tensor pipe computes S(j+1), S(j+2) while the softmax works on S(j):
// the single-CTA kernel's chain softmax(j) -> PV(j) -> S(j+1) -> softmax(j+1) is
// broken, and each CTA stages half of every K and V tile (shared-memory traffic per
// key tile 96 KB vs 128 KB for the same work).  MMA order per key tile j:
//   PV(j) (needs P(j)), then S(j+3) into P(j)'s buffer -- the in-order tensor pipe
//   reads P(j) before S(j+3) overwrites it.  The third buffer absorbs the cross-CTA
//   hand-off latency (the leader's MMA needs both CTAs' P(j)).
// O rescale (lazy, rare): softmax(j) first waits for PV(j-1) (pv_bar parity; PV(j+1)
// cannot complete before softmax(j) ends, so the parity wait cannot alias).
#ifndef TF_ATTN_Q_TMEM
#define TF_ATTN_Q_TMEM 1  // Q staged in TMEM: QK^T as a TS-MMA, no Q reads from shared memory
#endif
constexpr bool kQInTmem = TF_ATTN_Q_TMEM;
struct AttnPair2Smem {
  static constexpr int kQ = kQInTmem ? 0 : 2 * kHalf;  // this CTA's Q tile, 32 KB (smem variant)
  static constexpr int kSlot = 16384;         // half a K tile (64 keys x 128 dims) or half a V tile (128 keys x 64 dims)
  static constexpr int kSlots = kQInTmem ? 13 : 11;
  static constexpr int kBars = 512;  // 33 barrier words + the TMEM slot
  static constexpr int kXchg = 2 * 2 * 128 * 4;  // row-max halves [j & 1][half][row]
  static constexpr int kTotal = 1024 + kQ + kSlots * kSlot + kBars + kXchg;
};
constexpr int kAttnPair2Threads = 320;        // TMA, MMA, 8 softmax warps (2 per TMEM lane quarter)
// TMEM: three S buffers + O, or (Q in TMEM) two S buffers + O + Q (64 columns of bf16 pairs)
constexpr int kSBuf = kQInTmem ? 2 : 3;
constexpr int kOCol = kSBuf * 128;
constexpr int kQCol = 384;

__global__ void __maxnreg__(255)
    ag_attn_fwd_pair2_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                             const __grid_constant__ CUtensorMap tv, const __grid_constant__ AttnParams p) {
  using S = AttnPair2Smem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sq = smem;
  uint8_t* sring = sq + S::kQ;                      // K0 V0 K1 V1 ... halves
  uint64_t* bars = reinterpret_cast<uint64_t*>(sring + S::kSlots * S::kSlot);
  uint64_t* q_full = bars;                          // leader: both CTAs' Q bytes
  uint64_t* r_full = bars + 1;                      // [kSlots] leader: both halves of a K or V tile
  uint64_t* r_empty = r_full + S::kSlots;           // [kSlots] each CTA (multicast commits)
  uint64_t* s_full = r_empty + S::kSlots;           // [kSBuf] each CTA: S(j) in buffer j % kSBuf
  uint64_t* p_full = s_full + kSBuf;                // [kSBuf] leader: 8 softmax warps x 2 CTAs
  uint64_t* pv_bar = p_full + kSBuf;                // [2] each CTA: PV(j) complete, by j & 1
  uint64_t* o_ready = pv_bar + 2;                   // each CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_ready + 1);
  static_assert((1 + 2 * S::kSlots + 2 * kSBuf + 4) * 8 <= S::kBars, "barrier area");

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int q0 = (blockIdx.x >> 1) * 2 * kQT + static_cast<int>(cta) * kQT;  // this CTA's tile
  const int h = blockIdx.y;
  const int g = h / (p.hq / p.hkv);
  const int n = p.n_tiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, kQInTmem ? 16 : 1);  // Q rows in TMEM: 8 softmax warps x 2 CTAs
    for (int i = 0; i < S::kSlots; ++i) {
      mbar_init(&r_full[i], 1);
      mbar_init(&r_empty[i], 1);
    }
    for (int i = 0; i < kSBuf; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 16);
    }
    for (int i = 0; i < 2; ++i) mbar_init(&pv_bar[i], 1);
    mbar_init(o_ready, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      if constexpr (!kQInTmem) {
        if (leader) mbar_arrive_expect_tx(q_full, 2 * S::kQ);
        tma_load_3d_pair(sq, &tq, q_full, 0, h, q0);
        tma_load_3d_pair(sq + kHalf, &tq, q_full, 64, h, q0);
      }
      uint32_t ready = 0;
      for (int c = 0; c < 2 * n; ++c) {  // K_j = 2j, V_j = 2j + 1
        const int j = c >> 1, kv = c & 1;
        const int kt = (p.start_tile + j) % n;     // gather order: own chunk first
        const int chunk = kt / p.tiles_per_chunk;
        if (!kv && p.chunk_flags && !(ready & (1u << chunk))) {
          wait_geq_sys(p.chunk_flags + chunk, p.epoch, p.timeout_ns, p.err,
                       0x1000000ull | static_cast<unsigned>(chunk));
          fence_proxy_async_global();
          ready |= 1u << chunk;
        }
        const int sl = c % S::kSlots;
        mbar_wait(&r_empty[sl], ((c / S::kSlots) & 1) ^ 1);
        ATTN_STAMP(j, 5 + kv);
        if (!kv) ATTN_GSTAMP(j, 3);
        uint8_t* dst = sring + sl * S::kSlot;
        if (leader) mbar_arrive_expect_tx(&r_full[sl], 2 * S::kSlot);
        if (!kv) {  // this CTA's 64 keys of K_j, all 128 dims (two 64-dim boxes)
          const int row = kt * 128 + static_cast<int>(cta) * 64;
          tma_load_3d_pair(dst, &tk, &r_full[sl], 0, g, row);
          tma_load_3d_pair(dst + 8192, &tk, &r_full[sl], 64, g, row);
        } else {    // all 128 keys of V_j, this CTA's 64 dims
          tma_load_3d_pair(dst, &tv, &r_full[sl], static_cast<int>(cta) * 64, g, kt * 128);
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // all 32 lanes run the loop (descriptor math stays on the uniform datapath: a low
      // word plus compile-time deltas over a constant high word), elect.sync issues
      constexpr uint32_t idesc_s = umma_idesc_bf16(2 * kQT, 128);
      constexpr uint32_t idesc_pv = umma_idesc_bf16(2 * kQT, kD) | (1u << 16);  // B (V) MN-major
      constexpr uint32_t kDescHi = (1024 >> 4) | (1u << (46 - 32)) | (2u << (61 - 32));
      constexpr uint32_t kLoK = 1u << 16;                       // K-major SW128, LBO field 1
      constexpr uint32_t kLoV = ((16384 >> 4) & 0x3FFF) << 16;  // MN-major V, LBO = 16 KB
      auto mk = [](uint32_t lo) {
        uint64_t d;
        asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "r"(lo), "r"(kDescHi));
        return d;
      };
      const uint32_t q_lo = ((smem_u32(sq) & 0x3FFFF) >> 4) | kLoK;
      const uint32_t ring_lo = (smem_u32(sring) & 0x3FFFF) >> 4;
      auto issue_s = [&](int j) {  // S(j) into buffer j % 3
        const int c = 2 * j, sl = c % S::kSlots;
        MMA_WAIT(&r_full[sl], (c / S::kSlots) & 1);
        tc_fence_after();
        const uint32_t k_lo = (ring_lo + sl * (S::kSlot >> 4)) | kLoK;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          if constexpr (kQInTmem)
            umma_ts_pair_elect(tmem + (j % kSBuf) * 128, tmem + kQCol + kk * 8,
                               mk(k_lo + (kk >> 2) * (8192 >> 4) + (kk & 3) * 2), idesc_s, kk != 0);
          else
            umma_ss_pair_elect(tmem + (j % kSBuf) * 128, mk(q_lo + (kk >> 2) * (kHalf >> 4) + (kk & 3) * 2),
                               mk(k_lo + (kk >> 2) * (8192 >> 4) + (kk & 3) * 2), idesc_s, kk != 0);
        }
        umma_commit_pair_mc_elect(&s_full[j % kSBuf], 0x3);
        umma_commit_pair_mc_elect(&r_empty[sl], 0x3);
      };
      MMA_WAIT(q_full, 0);
      for (int j = 0; j < kSBuf && j < n; ++j) issue_s(j);
      for (int j = 0; j < n; ++j) {
        const int b = j % kSBuf;
        const int cv = 2 * j + 1, vs = cv % S::kSlots;
        MMA_WAIT(&r_full[vs], (cv / S::kSlots) & 1);
        if (lane == 0) ATTN_STAMP(j, 8);
        MMA_WAIT(&p_full[b], (j / kSBuf) & 1);
        if (lane == 0) { ATTN_STAMP(j, 2); ATTN_GSTAMP(j, 2); }
        tc_fence_after();
        const uint32_t v_lo = (ring_lo + vs * (S::kSlot >> 4)) | kLoV;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts_pair_elect(tmem + kOCol, tmem + b * 128 + kk * 8, mk(v_lo + kk * (2048 >> 4)), idesc_pv,
                             (j | kk) != 0);
        umma_commit_pair_mc_elect(&pv_bar[j & 1], 0x3);
        umma_commit_pair_mc_elect(&r_empty[vs], 0x3);
        if (lane == 0) ATTN_STAMP(j, 3);
        if (j + kSBuf < n) issue_s(j + kSBuf);
        if (lane == 0) ATTN_STAMP(j, 4);
      }
      umma_commit_pair_mc_elect(o_ready, 0x3);
    }
    __syncwarp();
  } else {
    // two warps per TMEM lane quarter: `half` 0 takes keys / O columns [0,64), half 1
    // [64,128) of the same 32 rows; the row max is combined through shared memory
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t t_o = tmem + lane_off + kOCol + half * 64;
    const uint32_t p_full_leader0 = mapa_shared(smem_u32(&p_full[0]), 0);
    float* xmax = reinterpret_cast<float*>(sring + S::kSlots * S::kSlot + S::kBars);  // [2][2][128]
    if constexpr (kQInTmem) {
      // this warp's 32 query rows x 64 dims of Q -> TMEM columns [kQCol + 32 half, +32)
      const int q = q0 + row;
      uint32_t qv[32];
      if (q < p.s_local) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p.q) +
                                                          (static_cast<long long>(q) * p.hq + h) * kD + half * 64);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 v = __ldg(src + i);
          qv[4 * i] = v.x;
          qv[4 * i + 1] = v.y;
          qv[4 * i + 2] = v.z;
          qv[4 * i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) qv[i] = 0u;
      }
      tmem_st_32x32b_x32(tmem + lane_off + kQCol + half * 32, qv);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(q_full), 0));
    }
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      const int b = j % kSBuf;
      const uint32_t t_s = tmem + lane_off + b * 128;
      SM_WAIT(&s_full[b], (j / kSBuf) & 1);
      tc_fence_after();
      if (threadIdx.x == 64) { ATTN_STAMP(j, 0); ATTN_GSTAMP(j, 0); }
      uint32_t sv[2][32];
      tmem_ld_32x32b_x32(t_s + half * 64, sv[0]);
      tmem_ld_32x32b_x32(t_s + half * 64 + 32, sv[1]);
      tmem_ld_wait();
      float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 2)
          mx[c] = fmax3(mx[c], __uint_as_float(sv[c][i]), __uint_as_float(sv[c][i + 1]));
      float* xm = xmax + (j & 1) * 256;
      xm[half * 128 + row] = fmaxf(mx[0], mx[1]);
      // both halves of these rows hold their S in registers now (P may overwrite S)
      asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
      const float mt = fmaxf(xm[row], xm[128 + row]) * p.scale_log2;
      float alpha = 1.f;
      if (mt > m + kLazyRescale) {
        alpha = ex2(m - mt);
        m = mt;
      }
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // O must hold PV(j-1) before it is rescaled
        mbar_wait_spin(&pv_bar[(j - 1) & 1], ((j - 1) >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t ov[16];
          tmem_ld_32x32b_x16(t_o + c * 16, ov);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
          tmem_st_32x32b_x16(t_o + c * 16, ov);
        }
      }
      uint64_t sum2 = f2pack(0.f, 0.f);
      const uint64_t scale2 = f2pack(p.scale_log2, p.scale_log2), negm2 = f2pack(-m, -m);
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          float a0, a1;
          f2unpack(ffma2(f2pack(__uint_as_float(sv[c][2 * i]), __uint_as_float(sv[c][2 * i + 1])), scale2,
                         negm2),
                   a0, a1);
          float p0, p1;
          if (TF_EXP2_EMU_MASK >= 0 && (i & TF_EXP2_EMU_MASK) == 0) {
            ex2_fma2(a0, a1, p0, p1);
          } else {
            p0 = ex2(a0);
            p1 = ex2(a1);
          }
          sum2 = fadd2(sum2, f2pack(p0, p1));
          pk[c * 16 + i] = pack_bf16x2(p0, p1);
        }
      float s0, s1;
      f2unpack(sum2, s0, s1);
      l = l * alpha + (s0 + s1);  // this half's keys; the halves are added at the end
      tmem_st_32x32b_x32(t_s + half * 32, pk);  // P of keys [64 half, 64 half + 64) as bf16 pairs
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(p_full_leader0 + b * 8);
      if (threadIdx.x == 64) { ATTN_STAMP(j, 1); ATTN_GSTAMP(j, 1); }
      if (threadIdx.x == 192) ATTN_STAMP(j, 7);
    }
    mbar_wait_spin(o_ready, 0);
    tc_fence_after();
    float* lsum = xmax;  // reuse the exchange buffer: [half][row]
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    lsum[half * 128 + row] = l;
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    const float inv = 1.f / (lsum[row] + lsum[128 + row]);
    const int q = q0 + row;
    uint16_t* dst = static_cast<uint16_t*>(p.out) + (static_cast<long long>(q) * p.hq + h) * kD + half * 64;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32b_x32(t_o + c * 32, ov);
      tmem_ld_wait();
      if (q < p.s_local) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          d4[i] = make_uint4(pack_bf16x2(__uint_as_float(ov[8 * i]) * inv, __uint_as_float(ov[8 * i + 1]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 2]) * inv, __uint_as_float(ov[8 * i + 3]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 4]) * inv, __uint_as_float(ov[8 * i + 5]) * inv),
                             pack_bf16x2(__uint_as_float(ov[8 * i + 6]) * inv, __uint_as_float(ov[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tmap_3d(CUtensorMap* map, const void* base, int64_t rows, int64_t heads, int box_rows = 128) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    enc = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(heads),
                        static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(kD * 2), static_cast<cuuint64_t>(heads * kD * 2)};
  cuuint32_t box[3] = {64, 1, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TF_ERR_INVALID, "attention tensor map encode failed");
  return TF_OK;
}

// Device table of 2w tensor maps (K then V) over every rank's own chunk in its
// workspace at buf_off, cached per (team, rank, chunk addresses).
std::mutex g_chunk_mu;
std::map<std::string, void*> g_chunk_maps;

int chunk_maps_for(tf_team* t, int rank, size_t buf_off, size_t chunk_bytes, int64_t sl, int64_t hkv,
                   int w, void** out) {
  std::string key(reinterpret_cast<const char*>(&t), sizeof(t));
  key.append(reinterpret_cast<const char*>(&rank), sizeof(rank));
  const int64_t geom[3] = {sl, hkv, w};  // a recycled address must not reuse other dims
  key.append(reinterpret_cast<const char*>(geom), sizeof(geom));
  std::vector<const uint8_t*> bases;
  for (int c = 0; c < w; ++c) {
    bases.push_back(t->pes[c].base + buf_off + c * chunk_bytes);                     // K chunk c
    bases.push_back(t->pes[c].base + buf_off + chunk_bytes * w + c * chunk_bytes);   // V chunk c
  }
  key.append(reinterpret_cast<const char*>(bases.data()), bases.size() * sizeof(void*));
  std::lock_guard<std::mutex> lk(g_chunk_mu);
  auto it = g_chunk_maps.find(key);
  if (it != g_chunk_maps.end()) {
    *out = it->second;
    return TF_OK;
  }
  std::vector<CUtensorMap> host(2 * w);
  for (int c = 0; c < w; ++c) {
    int rc = make_tmap_3d(&host[c], bases[2 * c], sl, hkv);
    if (rc) return rc;
    rc = make_tmap_3d(&host[w + c], bases[2 * c + 1], sl, hkv);
    if (rc) return rc;
  }
  void* dev = nullptr;
  TF_CUDA_TRY(cudaMalloc(&dev, host.size() * sizeof(CUtensorMap)));
  TF_CUDA_TRY(cudaMemcpy(dev, host.data(), host.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
  g_chunk_maps[key] = dev;
  *out = dev;
  return TF_OK;
}

}  // namespace
}  // namespace tf

using tf::fail;

extern "C" int tf_ag_kv_attention(tf_team* t, int rank, const tf_attn_fwd_args* a, int phase,
                                  void* stream, void* comm_stream) {
  if (!t || !a || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "bad team/rank/args");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  if (a->d != tf::kD) return fail(TF_ERR_CONFIG, "the fused attention kernel is built for head dim 128");
  if (a->hq < 1 || a->hkv < 1 || a->hq % a->hkv) return fail(TF_ERR_INVALID, "need hq % hkv == 0");
  if (a->s_local < 1 || a->s_local % tf::kKT)
    return fail(TF_ERR_INVALID, "s_local must be a positive multiple of 128");
  const int w = t->world;
  const int64_t sl = a->s_local, st = sl * w;
  if (st / tf::kKT / (sl / tf::kKT) > 32) return fail(TF_ERR_CONFIG, "at most 32 chunks");
  const int64_t krow = a->hkv * a->d;
  const size_t chunk_bytes = static_cast<size_t>(sl) * krow * 2;
  auto s = static_cast<cudaStream_t>(stream);
  auto cs = comm_stream ? static_cast<cudaStream_t>(comm_stream) : s;
  int rc = TF_OK;
  const std::string key = "attn:" + std::to_string(st) + "x" + std::to_string(krow);
  // [parity][K chunks | V chunks], flags [parity][w]
  tf::Workspace* ws = t->workspace(key, 2 * 2 * chunk_bytes * w, 2 * w, &rc);
  if (!ws) return rc;
  if (phase & TF_PHASE_PRE) {
    const uint64_t e = ++ws->epoch[rank];
    const int par = static_cast<int>(e & 1);
    uint8_t* kbuf = t->pes[rank].base + ws->data_off + par * 2 * chunk_bytes * w;
    uint8_t* vbuf = kbuf + chunk_bytes * w;
    TF_CUDA_TRY(cudaMemcpyAsync(kbuf + rank * chunk_bytes, a->k, chunk_bytes, cudaMemcpyDefault, s));
    TF_CUDA_TRY(cudaMemcpyAsync(vbuf + rank * chunk_bytes, a->v, chunk_bytes, cudaMemcpyDefault, s));
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
    const size_t buf_off = ws->data_off + par * 2 * chunk_bytes * w;
    uint8_t* kbuf = t->pes[rank].base + buf_off;
    uint8_t* vbuf = kbuf + chunk_bytes * w;
    // CTA-pair variant (TF_ATTN_PAIR=1) when the local sequence splits into groups of
    // 4 query tiles; measured slower than the single-CTA kernel at config 3 (4.75 vs
    // 3.88 ms/rank: the pair's softmax warpgroups run in lockstep across two SMs), so
    // it is opt-in
    const char* pair_env = getenv("TF_ATTN_PAIR");
    const int pair_mode = pair_env ? atoi(pair_env) : 0;
    const bool pair2 = pair_mode == 2 && sl % (2 * tf::kQT) == 0;
    const bool pair = (pair_mode == 1 && sl % (4 * tf::kQT) == 0) || pair2;
    // single-CTA kernel: K/V read over NVLink straight from each owner's chunk (no
    // staging copy; TF_ATTN_DIRECT=0 restores the copy-engine pull into this rank's
    // workspace); the pair variant keeps the pull
    const char* direct_env = getenv("TF_ATTN_DIRECT");
    const bool direct = !pair && (!direct_env || atoi(direct_env));
    if (w > 1) {
      rc = tf::team_barrier_wait(t, rank, s);
      if (rc) return rc;
      if (cs != s && !direct) {
        cudaEvent_t ev;
        TF_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        TF_CUDA_TRY(cudaEventRecord(ev, s));
        TF_CUDA_TRY(cudaStreamWaitEvent(cs, ev, 0));
        cudaEventDestroy(ev);
      }
      for (int i = 1; i < w && !direct; ++i) {
        const int src = (rank + i) % w;  // pull order of ag_gemm.py:64-69
        const uint8_t* pk = t->pes[src].base + buf_off;
        TF_CUDA_TRY(cudaMemcpyAsync(kbuf + src * chunk_bytes, pk + src * chunk_bytes, chunk_bytes,
                                    cudaMemcpyDefault, cs));
        TF_CUDA_TRY(cudaMemcpyAsync(vbuf + src * chunk_bytes, pk + chunk_bytes * w + src * chunk_bytes,
                                    chunk_bytes, cudaMemcpyDefault, cs));
        rc = tf::stream_signal_set(t, rank, ws->sig_base + par * w + src, e, cs);
        if (rc) return rc;
      }
    }
    CUtensorMap tq, tk, tv;
    rc = tf::make_tmap_3d(&tq, a->q, sl, a->hq);
    if (rc) return rc;
    rc = tf::make_tmap_3d(&tk, kbuf, st, a->hkv, pair ? 64 : 128);
    if (rc) return rc;
    rc = tf::make_tmap_3d(&tv, vbuf, st, a->hkv);
    if (rc) return rc;
    tf::AttnParams p{};
    p.s_local = static_cast<int>(sl);
    p.s_total = static_cast<int>(st);
    p.hq = static_cast<int>(a->hq);
    p.hkv = static_cast<int>(a->hkv);
    p.n_tiles = static_cast<int>(st / tf::kKT);
    p.tiles_per_chunk = static_cast<int>(sl / tf::kKT);
    p.start_tile = rank * p.tiles_per_chunk;
    p.scale_log2 = a->scale * 1.4426950408889634f;
    p.out = a->out;
    p.q = a->q;
    p.chunk_flags = t->pes[rank].sig + ws->sig_base + par * w;
    p.direct = direct ? 1 : 0;
    p.nchunks = w;
    if (direct) {
      for (int c = 0; c < w; ++c) p.peer_flags[c] = t->pes[c].sig + ws->sig_base + par * w + c;
      void* maps = nullptr;
      rc = tf::chunk_maps_for(t, rank, buf_off, chunk_bytes, sl, a->hkv, w, &maps);
      if (rc) return rc;
      p.chunk_maps = static_cast<const CUtensorMap*>(maps);
    }
    p.epoch = e;
    p.err = t->err_word(rank);
    p.timeout_ns = t->timeout_ns;
    static uint64_t attr_done = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_done & (1ull << dev))) {
      TF_CUDA_TRY(cudaFuncSetAttribute(tf::ag_attn_fwd_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tf::AttnSmem::kTotal));
      TF_CUDA_TRY(cudaFuncSetAttribute(tf::ag_attn_fwd_pair_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tf::AttnPairSmem::kTotal));
      TF_CUDA_TRY(cudaFuncSetAttribute(tf::ag_attn_fwd_pair2_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       tf::AttnPair2Smem::kTotal));
      attr_done |= 1ull << dev;
    }
    if (pair) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(static_cast<unsigned>(2 * sl / ((pair2 ? 2 : 4) * tf::kQT)), static_cast<unsigned>(a->hq));
      cfg.blockDim = dim3(pair2 ? tf::kAttnPair2Threads : 320);
      cfg.dynamicSmemBytes = pair2 ? tf::AttnPair2Smem::kTotal : tf::AttnPairSmem::kTotal;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (pair2) TF_CUDA_TRY(cudaLaunchKernelEx(&cfg, tf::ag_attn_fwd_pair2_kernel, tq, tk, tv, p));
      else TF_CUDA_TRY(cudaLaunchKernelEx(&cfg, tf::ag_attn_fwd_pair_kernel, tq, tk, tv, p));
    }
    dim3 grid(static_cast<unsigned>((sl + 2 * tf::kQT - 1) / (2 * tf::kQT)), static_cast<unsigned>(a->hq));
    if (!pair) tf::ag_attn_fwd_kernel<<<grid, tf::kAttnThreads2, tf::AttnSmem::kTotal, s>>>(tq, tk, tv, p);
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, tf::ag_attn_fwd_kernel);
      return fail(TF_ERR_CUDA, std::string("attention launch: ") + cudaGetErrorString(le) +
                                   " (regs " + std::to_string(fa.numRegs) + ", max threads " +
                                   std::to_string(fa.maxThreadsPerBlock) + ", static smem " +
                                   std::to_string(fa.sharedSizeBytes) + ", max dyn smem " +
                                   std::to_string(fa.maxDynamicSharedSizeBytes) + ", dyn " +
                                   std::to_string(tf::AttnSmem::kTotal) + ")");
    }
    if (w > 1 && cs != s) {
      cudaEvent_t ev;
      TF_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      TF_CUDA_TRY(cudaEventRecord(ev, cs));
      TF_CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
      cudaEventDestroy(ev);
    }
  }
  return TF_OK;
}

#ifdef TF_ATTN_TRACE
extern "C" int tf_attn_trace_dump(long long* out) {
  return cudaMemcpyFromSymbol(out, tf::g_attn_trace, sizeof(tf::g_attn_trace)) == cudaSuccess ? 0 : 5;
}
#endif
