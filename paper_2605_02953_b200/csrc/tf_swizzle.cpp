// Host-side tile-order tables (bit-identical to the reference swizzles).
//
//   tf_swizzle_2d   <- ovs/swizzle.py:76-88   (grouped launch order)
//   tf_tile_map     <- ovs/swizzle.py:109-185 (gather / scatter maps, incl.
//                      multi-node straddle rules; single node collapses to the
//                      rotations of swizzle.py:94-103)
//   tf_moe_schedule <- ovs/swizzle.py:225-286 (expert-grouped, arrival-staged)
//
// The device kernels consume tf_tile_map's output as an int32 table indexed by
// pid_m (the GEMM kernel applies swizzle_2d itself, see tf_gemm.cu).
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "tf_internal.h"

namespace {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct NodeRange {
  int64_t node, first, last;
};

// Per-node inclusive row-tile ranges in visiting order; a tile straddling two
// nodes is kept by the last-visited node (gather) or the first-visited (scatter).
std::vector<NodeRange> node_ranges(int64_t m, int64_t bm, int nnodes, int64_t first_node,
                                   bool gather) {
  std::vector<NodeRange> out;
  const int64_t per_node = m / nnodes;
  for (int pos = 0; pos < nnodes; ++pos) {
    const int64_t node = (first_node + pos) % nnodes;
    const int64_t lo = node * per_node, hi = (node + 1) * per_node;
    int64_t first = lo / bm;
    int64_t last = (hi - 1) / bm;
    const bool head_shared = lo != 0 && (lo - 1) / bm == first;
    const bool tail_shared = hi != m && hi / bm == last;
    if (gather) {
      if (pos == 0 && head_shared) ++first;
      if (tail_shared && (pos == 0 || pos != nnodes - 1)) --last;
    } else {
      if (pos != 0 && head_shared) ++first;
      if (pos == nnodes - 1 && tail_shared) --last;
    }
    out.push_back({node, first, last});
  }
  return out;
}

}  // namespace

extern "C" int tf_swizzle_2d(int64_t pid, int64_t num_pid_m, int64_t num_pid_n, int group_m,
                             int64_t* pid_m, int64_t* pid_n) {
  if (group_m < 1) return tf::fail(TF_ERR_INVALID, "group_size_m must be >= 1");
  if (pid < 0 || pid >= num_pid_m * num_pid_n)
    return tf::fail(TF_ERR_INVALID, "pid " + std::to_string(pid) + " out of range");
  const int64_t per_group = static_cast<int64_t>(group_m) * num_pid_n;
  const int64_t g = pid / per_group, r = pid % per_group;
  const int64_t first = g * group_m;
  const int64_t rows = std::min<int64_t>(num_pid_m - first, group_m);
  *pid_m = first + r % rows;
  *pid_n = r / rows;
  return TF_OK;
}

extern "C" int tf_tile_map(int64_t m, int rank, int world, int nnodes, int block_m, int mode,
                           int32_t* out, int64_t out_len) {
  if (world < 1 || nnodes < 1) return tf::fail(TF_ERR_INVALID, "world_size and nnodes must be >= 1");
  if (world % nnodes) return tf::fail(TF_ERR_INVALID, "world_size not divisible by nnodes");
  if (m % world) return tf::fail(TF_ERR_INVALID, "M must divide evenly across ranks");
  if (rank < 0 || rank >= world) return tf::fail(TF_ERR_INVALID, "rank out of range");
  if (block_m < 1) return tf::fail(TF_ERR_INVALID, "block_m must be >= 1");
  if (mode != 0 && mode != 1) return tf::fail(TF_ERR_INVALID, "mode must be 0 (gather) or 1 (scatter)");
  const int64_t tiles = cdiv(m, block_m);
  if (out_len < tiles) return tf::fail(TF_ERR_INVALID, "output table too small");
  const bool gather = mode == 0;
  const int lws = world / nnodes;
  const int node = rank / lws, local = rank % lws;
  const int64_t rows_rank = m / world, rows_node = m / nnodes;
  const int64_t first_node = gather ? node : node + 1;
  int64_t pos = 0;
  for (const NodeRange& nr : node_ranges(m, block_m, nnodes, first_node, gather)) {
    const int64_t count = nr.last - nr.first + 1;
    if (count <= 0) continue;
    const int64_t start_tile =
        gather ? cdiv(rows_node * nr.node + rows_rank * local, block_m)
               : (rows_node * nr.node + rows_rank * (local + 1)) / block_m;
    const int64_t rot = std::max<int64_t>(0, start_tile - nr.first);
    for (int64_t i = 0; i < count; ++i) out[pos++] = static_cast<int32_t>(nr.first + (i + rot) % count);
  }
  if (pos != tiles) return tf::fail(TF_ERR_PROTOCOL, "node tile ranges do not partition the tile space");
  return TF_OK;
}

extern "C" int tf_moe_schedule(const int64_t* counts, int world, int n_experts, int rank,
                               int local_world, int block_m, int64_t* ntiles, int64_t* expert_id,
                               int64_t* tiled_m, int64_t* segment_start, int64_t* segment_end,
                               int64_t* stage) {
  if (world < 1 || local_world < 1 || world % local_world)
    return tf::fail(TF_ERR_INVALID, "tp_size must be a multiple of local_tp_size");
  if (rank < 0 || rank >= world) return tf::fail(TF_ERR_INVALID, "rank out of range");
  if (block_m < 1) return tf::fail(TF_ERR_INVALID, "block_size_m must be >= 1");
  if (n_experts < 0) return tf::fail(TF_ERR_INVALID, "n_experts must be >= 0");
  for (int64_t i = 0; i < static_cast<int64_t>(world) * n_experts; ++i)
    if (counts[i] < 0) return tf::fail(TF_ERR_INVALID, "token counts must be >= 0");
  // (expert, stage, global tile, seg0, seg1)
  std::vector<std::tuple<int64_t, int64_t, int64_t, int64_t, int64_t>> rows;
  int64_t gtile = 0;
  std::vector<int64_t> ends(world);
  for (int e = 0; e < n_experts; ++e) {
    int64_t acc = 0;
    for (int s = 0; s < world; ++s) {
      acc += counts[static_cast<int64_t>(s) * n_experts + e];
      ends[s] = acc;  // inclusive prefix over source ranks
    }
    const int64_t total = acc;
    for (int64_t t = 0; t < cdiv(total, block_m); ++t) {
      const int64_t r0 = t * block_m, r1 = std::min(r0 + block_m, total);
      // first source whose inclusive prefix exceeds the row (searchsorted 'right')
      const int64_t s0 = std::upper_bound(ends.begin(), ends.end(), r0) - ends.begin();
      const int64_t s1 = std::upper_bound(ends.begin(), ends.end(), r1 - 1) - ends.begin();
      int64_t st = 0;
      for (int64_t s = s0; s <= s1; ++s) st = std::max<int64_t>(st, ((s - rank) % world + world) % world);
      rows.emplace_back(e, st, gtile, s0, s1);
      ++gtile;
    }
  }
  std::stable_sort(rows.begin(), rows.end(), [](const auto& a, const auto& b) {
    return std::tie(std::get<0>(a), std::get<1>(a), std::get<2>(a)) <
           std::tie(std::get<0>(b), std::get<1>(b), std::get<2>(b));
  });
  *ntiles = static_cast<int64_t>(rows.size());
  if (!expert_id) return TF_OK;
  for (size_t i = 0; i < rows.size(); ++i) {
    expert_id[i] = std::get<0>(rows[i]);
    stage[i] = std::get<1>(rows[i]);
    tiled_m[i] = std::get<2>(rows[i]);
    segment_start[i] = std::get<3>(rows[i]);
    segment_end[i] = std::get<4>(rows[i]);
  }
  return TF_OK;
}
