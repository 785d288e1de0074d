// AllGather + grouped GEMM for expert-routed tokens (tf_ag_moe_group_gemm) --
// the reference's MoE hot loop, ovs/kernels/ag_moe.py:20-142, re-done as one
// launch per call: pull-engine CTAs (the reference's `pull` process) and the
// persistent tcgen05 grouped GEMM (its `gemm{sm}` workers) share the grid.
//
// Layout per PE and call parity (double-buffered by call epoch, like tf_ag_gemm):
//   rows   [max_rows][k] bf16   the gathered operand in EXPERT-MAJOR order: the
//                               piece of (source s, expert e) lives at rows
//                               expert_base[e] + sum_{s'<s} routing[s', e] on every
//                               PE, so a grouped tile (block_m rows of one expert)
//                               is contiguous and TMA-loadable, and a pull of
//                               source s is E contiguous byte ranges at identical
//                               offsets in s's workspace and ours.
//   tables int4 sched[slots] {expert, first row, rows, seg_start | seg_end << 16}
//          int32 irb[world][E+1]  (in-rank expert bases, ag_moe.py:54-55)
//          int32 dstb[world][E]   (gathered row of each piece)
//   flags  u64 arrival[world]     per-source counters, zeroed in PRE, released by
//                                 each pull CTA after its share of the source
//                                 landed; a tile waits for count == comm CTAs.
// The reference gathers rank-major and re-gathers rows per tile (_gather_rows,
// ag_moe.py:145-160); placing pieces expert-major at pull time is the same data
// movement with the permutation folded into the copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "tf_internal.h"
#include "tf_ptx.cuh"
#include "tf_team.h"

namespace tf {
namespace {

// own chunk (rank-major, grouped by expert) -> own workspace at its expert-major rows
__global__ void __launch_bounds__(256) agmoe_local_copy_kernel(
    const uint8_t* __restrict__ tokens, long long ld_bytes, uint8_t* __restrict__ ws,
    const int32_t* __restrict__ irb, const int32_t* __restrict__ dstb, int n_experts, long long rows,
    long long row_bytes) {
  const int lane = threadIdx.x & 31;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const long long vecs = row_bytes / 16;
  for (long long j = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < rows;
       j += warps) {
    int lo = 0, hi = n_experts - 1;  // last expert with irb[e] <= j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(irb + mid) <= j) lo = mid;
      else hi = mid - 1;
    }
    const long long drow = __ldg(dstb + lo) + (j - __ldg(irb + lo));
    const uint4* src = reinterpret_cast<const uint4*>(tokens + j * ld_bytes);
    uint4* dst = reinterpret_cast<uint4*>(ws + drow * row_bytes);
    for (long long v = lane; v < vecs; v += 32) dst[v] = __ldg(src + v);
  }
}

struct Plan {
  int world = 1, E = 0, cg = 1, block_m = 128, block_n = 256, comm_ctas = 0;
  int64_t total = 0, max_rows = 0, row_bytes = 0, slots = 0, max_slots = 0;
  size_t rows_bytes = 0, tab_bytes = 0;
  std::vector<int64_t> rows_by_rank, expert_base, tokens_per_expert;
  std::vector<int32_t> irb, dstb;  // [world][E+1], [world][E]
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int make_plan(const tf_team* t, const tf_agmoe_args* a, Plan& P) {
  if (!a) return fail(TF_ERR_INVALID, "args is NULL");
  if (!a->routing) return fail(TF_ERR_INVALID, "routing is NULL");
  if (a->n_experts < 1 || a->n_experts > (1 << 16)) return fail(TF_ERR_INVALID, "n_experts out of range");
  if (a->k < 8 || a->k % 8) return fail(TF_ERR_INVALID, "k must be a positive multiple of 8 (16-byte rows)");
  if (a->n < 8 || a->n % 8) return fail(TF_ERR_INVALID, "n must be a positive multiple of 8");
  const int bm = a->block_m ? a->block_m : 128;
  const int bn = a->block_n ? a->block_n : 256;
  if (bm != 128 && bm != 256) return fail(TF_ERR_CONFIG, "block_m must be 128 or 256 for the grouped GEMM");
  if (bn != 128 && bn != 256) return fail(TF_ERR_CONFIG, "block_n must be 128 or 256");
  P.world = t->world;
  P.E = static_cast<int>(a->n_experts);
  P.block_m = bm;
  P.block_n = bn;
  P.cg = bm == 256 ? 2 : 1;
  const int w = P.world, E = P.E;
  P.rows_by_rank.assign(w, 0);
  P.tokens_per_expert.assign(E, 0);
  for (int s = 0; s < w; ++s)
    for (int e = 0; e < E; ++e) {
      const int64_t c = a->routing[static_cast<int64_t>(s) * E + e];
      if (c < 0) return fail(TF_ERR_INVALID, "routing counts must be >= 0");
      P.rows_by_rank[s] += c;
      P.tokens_per_expert[e] += c;
    }
  P.expert_base.assign(E + 1, 0);
  for (int e = 0; e < E; ++e) P.expert_base[e + 1] = P.expert_base[e] + P.tokens_per_expert[e];
  P.total = P.expert_base[E];
  if (P.total >= (int64_t{1} << 31)) return fail(TF_ERR_INVALID, "total rows exceed int32");
  P.max_rows = a->max_rows > 0 ? a->max_rows : P.total;
  if (P.total > P.max_rows)
    return fail(TF_ERR_INVALID, "total routed rows " + std::to_string(P.total) + " exceed max_rows " +
                                    std::to_string(P.max_rows));
  P.irb.assign(static_cast<size_t>(w) * (E + 1), 0);
  P.dstb.assign(static_cast<size_t>(w) * E, 0);
  std::vector<int64_t> rank_cum(E, 0);  // sum_{s' < s} routing[s', e]
  for (int s = 0; s < w; ++s) {
    int64_t acc = 0;
    for (int e = 0; e < E; ++e) {
      P.irb[static_cast<size_t>(s) * (E + 1) + e] = static_cast<int32_t>(acc);
      P.dstb[static_cast<size_t>(s) * E + e] = static_cast<int32_t>(P.expert_base[e] + rank_cum[e]);
      const int64_t c = a->routing[static_cast<int64_t>(s) * E + e];
      acc += c;
      rank_cum[e] += c;
    }
    P.irb[static_cast<size_t>(s) * (E + 1) + E] = static_cast<int32_t>(acc);
  }
  P.slots = 0;
  for (int e = 0; e < E; ++e) P.slots += (P.tokens_per_expert[e] + bm - 1) / bm;
  P.max_slots = (P.max_rows + bm - 1) / bm + E;
  P.row_bytes = a->k * 2;
  // one rank: the caller's rows are already expert-major, no gathered copy is kept
  P.rows_bytes = w == 1 ? 0 : align_up(static_cast<size_t>(std::max<int64_t>(P.max_rows, 1)) * P.row_bytes, 1024);
  P.tab_bytes = align_up(static_cast<size_t>(P.max_slots) * 16 + P.irb.size() * 4 + P.dstb.size() * 4, 1024);
  int cc = a->num_comm_sms > 0 ? a->num_comm_sms : 8;
  cc = (cc + P.cg - 1) / P.cg * P.cg;
  P.comm_ctas = w > 1 ? cc : 0;
  return TF_OK;
}

// host tile table in schedule order (swizzle_ag_moe) or plain tile order
int build_table(const tf_agmoe_args* a, const Plan& P, int rank, std::vector<int32_t>& tab) {
  const int w = P.world, E = P.E;
  int64_t nt = 0;
  int rc = tf_moe_schedule(a->routing, w, E, rank, w, P.block_m, &nt, nullptr, nullptr, nullptr, nullptr,
                           nullptr);
  if (rc) return rc;
  if (nt != P.slots) return fail(TF_ERR_PROTOCOL, "schedule tile count mismatch");
  std::vector<int64_t> eid(nt), tm(nt), s0(nt), s1(nt), st(nt);
  if (nt) {
    rc = tf_moe_schedule(a->routing, w, E, rank, w, P.block_m, &nt, eid.data(), tm.data(), s0.data(),
                         s1.data(), st.data());
    if (rc) return rc;
  }
  std::vector<int64_t> tile_base(E + 1, 0);
  for (int e = 0; e < E; ++e) tile_base[e + 1] = tile_base[e] + (P.tokens_per_expert[e] + P.block_m - 1) / P.block_m;
  std::vector<int64_t> order(nt);
  for (int64_t i = 0; i < nt; ++i) order[i] = i;
  if (!a->swizzle)  // _identity_order (ag_moe.py:85-94): stable sort by tiled_m
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return tm[x] < tm[y]; });
  tab.assign(static_cast<size_t>(nt) * 4, 0);
  for (int64_t i = 0; i < nt; ++i) {
    const int64_t j = order[i];
    const int e = static_cast<int>(eid[j]);
    const int64_t off = (tm[j] - tile_base[e]) * P.block_m;
    const int64_t rows = std::min<int64_t>(P.block_m, P.tokens_per_expert[e] - off);
    tab[4 * i + 0] = e;
    tab[4 * i + 1] = static_cast<int32_t>(P.expert_base[e] + off);
    tab[4 * i + 2] = static_cast<int32_t>(rows);
    tab[4 * i + 3] = static_cast<int32_t>(s0[j] | (s1[j] << 16));
  }
  return TF_OK;
}

}  // namespace
}  // namespace tf

using tf::fail;

extern "C" int tf_ag_moe_group_gemm(tf_team* t, int rank, const tf_agmoe_args* a, int phase, void* stream) {
  if (!t || rank < 0 || rank >= t->world) return fail(TF_ERR_INVALID, "rank out of range");
  if (!t->is_local(rank)) return fail(TF_ERR_INVALID, "rank is not owned by this process");
  tf::Plan P;
  int rc = tf::make_plan(t, a, P);
  if (rc) return rc;
  if (t->world > 16) return fail(TF_ERR_CONFIG, "ag_moe_group_gemm supports world <= 16");
  const int w = P.world;
  const std::string key = "agmoe:" + std::to_string(P.max_rows) + "x" + std::to_string(a->k) + ":" +
                          std::to_string(P.E) + ":" + std::to_string(P.block_m);
  const size_t per_par = P.rows_bytes + P.tab_bytes;
  tf::Workspace* ws = t->workspace(key, 2 * per_par, 2 * w, &rc);
  if (!ws) return rc;
  auto s = static_cast<cudaStream_t>(stream);
  const int64_t lda = a->lda ? a->lda : a->k;
  const int64_t rows_r = P.rows_by_rank[rank];
  if (rows_r > 0 && !a->tokens) return fail(TF_ERR_INVALID, "tokens is NULL");
  if ((lda * 2) % 16) return fail(TF_ERR_INVALID, "token row stride must be a multiple of 16 bytes");

  auto par_base = [&](int pe, int par) { return t->pes[pe].base + ws->data_off + par * per_par; };
  if (phase & TF_PHASE_PRE) {
    const uint64_t e = ++ws->epoch[rank];
    const int par = static_cast<int>(e & 1);
    uint8_t* own = par_base(rank, par);
    uint8_t* tab = own + P.rows_bytes;
    std::vector<int32_t> host;
    rc = tf::build_table(a, P, rank, host);
    if (rc) return rc;
    const size_t sched_bytes = host.size() * 4;
    host.resize(P.max_slots * 4, 0);
    host.insert(host.end(), P.irb.begin(), P.irb.end());
    host.insert(host.end(), P.dstb.begin(), P.dstb.end());
    (void)sched_bytes;
    TF_CUDA_TRY(cudaMemcpyAsync(tab, host.data(), host.size() * 4, cudaMemcpyHostToDevice, s));
    if (w > 1) {
      uint64_t* flags = t->pes[rank].sig + ws->sig_base + par * w;
      TF_CUDA_TRY(cudaMemsetAsync(flags, 0, w * sizeof(uint64_t), s));
      const int32_t* irb_d = reinterpret_cast<const int32_t*>(tab + P.max_slots * 16);
      const int32_t* dstb_d = irb_d + static_cast<size_t>(w) * (P.E + 1);
      if (rows_r > 0) {
        const int blocks = static_cast<int>(std::min<int64_t>((rows_r + 7) / 8, 148 * 4));
        tf::agmoe_local_copy_kernel<<<blocks, 256, 0, s>>>(
            static_cast<const uint8_t*>(a->tokens), lda * 2, own, irb_d + static_cast<size_t>(rank) * (P.E + 1),
            dstb_d + static_cast<size_t>(rank) * P.E, P.E, rows_r, P.row_bytes);
        TF_CUDA_TRY(cudaGetLastError());
      }
      rc = tf::stream_signal_set(t, rank, ws->sig_base + par * w + rank, P.comm_ctas, s);
      if (rc) return rc;
      rc = tf::team_barrier_arrive(t, rank, s);
      if (rc) return rc;
    }
  }
  if (phase & TF_PHASE_MAIN) {
    const int par = static_cast<int>(ws->epoch[rank] & 1);
    uint8_t* own = par_base(rank, par);
    uint8_t* tab = own + P.rows_bytes;
    if (w > 1) {
      rc = tf::team_barrier_wait(t, rank, s);
      if (rc) return rc;
    }
    if (P.total == 0) return TF_OK;
    tf::GemmLaunch g;
    g.b = a->weights;
    g.ldb = a->k;
    g.m = P.total;
    g.n = a->n;
    g.k = a->k;
    g.block_m = P.block_m;
    g.block_n = P.block_n;
    g.group_m = 1;
    g.num_sms = a->num_gemm_sms > 0 ? a->num_gemm_sms + P.comm_ctas : 0;
    g.out_f32 = a->out_dtype == TF_DTYPE_F32 ? 1 : 0;
    g.c = a->out;
    g.ldc = a->ldo ? a->ldo : a->n;
    g.moe_tab = tab;
    g.moe_slots = static_cast<int>(P.slots);
    g.n_experts = P.E;
    g.err = t->err_word(rank);
    g.timeout_ns = t->timeout_ns;
    g.trace_rank = rank;
    if (w == 1) {
      // one source: the caller's rows are already expert-major
      g.a = a->tokens;
      g.lda = lda;
    } else {
      g.a = own;
      g.lda = a->k;
      uint64_t* flags = t->pes[rank].sig + ws->sig_base + par * w;
      g.src_flags = flags;
      g.src_target = P.comm_ctas;
      g.comm_ctas = P.comm_ctas;
      for (int pe = 0; pe < w; ++pe) g.peer_ws[pe] = par_base(pe, par);
      g.own_ws = own;
      g.irb = reinterpret_cast<const int32_t*>(tab + P.max_slots * 16);
      g.dstb = g.irb + static_cast<size_t>(w) * (P.E + 1);
      g.row_bytes = P.row_bytes;
      g.own_flags = flags;
      g.rank = rank;
      g.world = w;
    }
    rc = tf::launch_gemm(g, s);
    if (rc) return rc;
  }
  return TF_OK;
}
