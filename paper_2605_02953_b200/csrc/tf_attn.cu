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
// Per CTA (192 threads):
//   warp 0      TMA: Q tile once, then K/V tiles (128 keys x 128 dims each) into a
//               2-stage ring.
//   warp 1      MMA (one lane): S_j = Q K_j^T (M=128, N=128, K=d) into a
//               double-buffered TMEM S; O += P_j V_j (A = P from smem, K-major;
//               B = V from smem, MN-major) into TMEM O.
//   warps 2-5   softmax, one query row per thread: S row from TMEM, online
//               max/sum in fp32 (exp2 with the scale folded in), O row rescaled
//               in TMEM when the max grows, P row written to smem as bf16
//               (128-byte swizzled K-major), final O / l stored as bf16.
// TMEM: S0 [0,128), S1 [128,256), O [256,384) fp32 columns.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

constexpr int kQT = 128;      // queries per CTA
constexpr int kKT = 128;      // keys per tile
constexpr int kD = 128;       // head dim (fixed for this kernel)
constexpr int kHalf = 16384;  // one 128-row x 64-col bf16 box (128-byte rows)
constexpr int kAttnThreads = 192;

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
};

struct AttnSmem {
  static constexpr int kQ = 2 * kHalf;        // 32 KB
  static constexpr int kKV = 4 * kHalf;       // K (2 halves) + V (2 halves) = 64 KB
  static constexpr int kStages = 2;
  static constexpr int kP = 2 * kHalf;        // 32 KB
  static constexpr int kBars = 256;
  static constexpr int kTotal = 1024 + kQ + kStages * kKV + kP + kBars;
};

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
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kAttnThreads, 1)
    ag_attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ AttnParams p) {
  using S = AttnSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sq = smem;
  uint8_t* skv = sq + S::kQ;                 // stage s: K at s*kKV, V at s*kKV + 2*kHalf
  uint8_t* sp = skv + S::kStages * S::kKV;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sp + S::kP);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;    // [2]
  uint64_t* kv_empty = bars + 3;   // [2]
  uint64_t* s_full = bars + 5;     // [2]
  uint64_t* s_empty = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* pv_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_tile = blockIdx.x;
  const int h = blockIdx.y;
  const int g = h / (p.hq / p.hkv);
  const int n = p.n_tiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, S::kQ);
      tma_load_3d(sq, &tq, q_full, 0, h, q_tile * kQT);
      tma_load_3d(sq + kHalf, &tq, q_full, 64, h, q_tile * kQT);
      uint32_t ready = 0;
      for (int j = 0; j < n; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        const int kt = (p.start_tile + j) % n;     // gather order: own chunk first
        const int chunk = kt / p.tiles_per_chunk;
        if (p.chunk_flags && !(ready & (1u << chunk))) {
          wait_geq_sys(p.chunk_flags + chunk, p.epoch, p.timeout_ns, p.err,
                       0x1000000ull | static_cast<unsigned>(chunk));
          fence_proxy_async_global();
          ready |= 1u << chunk;
        }
        uint8_t* kb = skv + st * S::kKV;
        mbar_arrive_expect_tx(&kv_full[st], S::kKV);
        tma_load_3d(kb, &tk, &kv_full[st], 0, g, kt * kKT);
        tma_load_3d(kb + kHalf, &tk, &kv_full[st], 64, g, kt * kKT);
        tma_load_3d(kb + 2 * kHalf, &tv, &kv_full[st], 0, g, kt * kKT);
        tma_load_3d(kb + 3 * kHalf, &tv, &kv_full[st], 64, g, kt * kKT);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kQT, kKT);                    // K-major A and B
    constexpr uint32_t idesc_pv = umma_idesc_bf16(kQT, kD) | (1u << 16);      // B (V) MN-major
    mbar_wait(q_full, 0);
    tc_fence_after();
    auto issue_pv = [&](int jj) {
      const int st = jj & 1;
      mbar_wait(p_full, jj & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t pa = smem_u32(sp);
        const uint32_t vb = smem_u32(skv + st * S::kKV + 2 * kHalf);
#pragma unroll
        for (int kk = 0; kk < kKT / 16; ++kk) {
          const uint64_t ad = umma_desc_k_sw128(pa + (kk >> 2) * kHalf + (kk & 3) * 32);
          const uint64_t bd = umma_desc_mn_sw128(vb + kk * 2048, kHalf);
          umma_bf16(t_o, ad, bd, idesc_pv, (jj | kk) != 0);
        }
        umma_commit(&kv_empty[st]);
        umma_commit(pv_done);
      }
      __syncwarp();
    };
    for (int j = 0; j < n; ++j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);
      mbar_wait(&s_empty[st], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t qa = smem_u32(sq);
        const uint32_t kb = smem_u32(skv + st * S::kKV);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
          umma_bf16(tmem + st * kKT, umma_desc_k_sw128(qa + off), umma_desc_k_sw128(kb + off),
                    idesc_s, kk != 0);
        }
        umma_commit(&s_full[st]);
      }
      __syncwarp();
      if (j > 0) issue_pv(j - 1);
    }
    issue_pv(n - 1);
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    float m = -INFINITY, l = 0.f;
    uint8_t* prow = sp + row * 128;
    for (int j = 0; j < n; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem + lane_off + st * kKT + c * 32, sv[c]);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);
      float mx = m;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(sv[c][i]) * p.scale_log2);
      const float alpha = exp2f(m - mx);  // 0 on the first tile (m = -inf)
      float sum = 0.f;
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = exp2f(__uint_as_float(sv[c][2 * i]) * p.scale_log2 - mx);
          const float p1 = exp2f(__uint_as_float(sv[c][2 * i + 1]) * p.scale_log2 - mx);
          sum += p0 + p1;
          pk[c][i] = pack_bf16x2(p0, p1);
        }
      l = l * alpha + sum;
      m = mx;
      if (j > 0) {
        // P buffer and O are free once P_{j-1} V_{j-1} has completed
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha < 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld_32x32b_x32(t_o + lane_off + c * 32, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * alpha);
            tmem_st_32x32b_x32(t_o + lane_off + c * 32, ov);
          }
          tmem_st_wait();
        }
      }
      // P row -> smem, 128-byte swizzled K-major (halves of 64 keys, 16 KB apart)
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = c * 4 + q;            // 16-byte chunk of the 256-byte row
          const int half = chunk >> 3, jj = chunk & 7;
          *reinterpret_cast<uint4*>(prow + half * kHalf + ((jj ^ (row & 7)) << 4)) =
              make_uint4(pk[c][4 * q], pk[c][4 * q + 1], pk[c][4 * q + 2], pk[c][4 * q + 3]);
        }
      fence_proxy_async_shared();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 [q, h, :]
    mbar_wait(pv_done, (n - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    const int q = q_tile * kQT + row;
    uint16_t* dst = static_cast<uint16_t*>(p.out) + (static_cast<long long>(q) * p.hq + h) * kD;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld_32x32b_x32(t_o + lane_off + c * 32, ov);
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
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_tmap_3d(CUtensorMap* map, const void* base, int64_t rows, int64_t heads) {
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
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(TF_ERR_INVALID, "attention tensor map encode failed");
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
    if (w > 1) {
      rc = tf::team_barrier_wait(t, rank, s);
      if (rc) return rc;
      if (cs != s) {
        cudaEvent_t ev;
        TF_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        TF_CUDA_TRY(cudaEventRecord(ev, s));
        TF_CUDA_TRY(cudaStreamWaitEvent(cs, ev, 0));
        cudaEventDestroy(ev);
      }
      for (int i = 1; i < w; ++i) {
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
    rc = tf::make_tmap_3d(&tk, kbuf, st, a->hkv);
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
    p.chunk_flags = t->pes[rank].sig + ws->sig_base + par * w;
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
      attr_done |= 1ull << dev;
    }
    dim3 grid(static_cast<unsigned>(sl / tf::kQT), static_cast<unsigned>(a->hq));
    tf::ag_attn_fwd_kernel<<<grid, tf::kAttnThreads, tf::AttnSmem::kTotal, s>>>(tq, tk, tv, p);
    TF_CUDA_TRY(cudaGetLastError());
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
