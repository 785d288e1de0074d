"""Oracle restatement of the tile-order permutations (test infrastructure only).

Follows /root/reference/pkg/src/overlapsim/swizzle.py:
  grouped launch order           swizzle.py:76-88
  single-node rotations          swizzle.py:94-103
  per-node visiting ranges       swizzle.py:109-141
  inter-node gather/scatter map  swizzle.py:144-185
  MoE dynamic schedule           swizzle.py:207-286
  text render                    swizzle.py:294-322
Everything is restated with explicit integer arithmetic so the C++ tables in the
product library can be compared entry-for-entry.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GATHER = "ag_gemm"
SCATTER = "gemm_rs"


def ceil_div(a: int, b: int) -> int:
    return (a + b - 1) // b


def grouped_pid(step: int, tiles_m: int, tiles_n: int, group: int) -> tuple[int, int]:
    """Linear tile id -> (pid_m, pid_n), row-grouped (swizzle.py:76-88)."""
    if group < 1:
        raise ValueError("group_size_m must be >= 1")
    if step < 0 or step >= tiles_m * tiles_n:
        raise ValueError(f"pid {step} out of range")
    per_group = group * tiles_n
    g, r = divmod(step, per_group)
    m0 = g * group
    rows = min(group, tiles_m - m0)
    return m0 + r % rows, r // rows


def gather_rotation(pid_m: int, m: int, rank: int, world: int, block_m: int) -> int:
    """swizzle.py:94-97 -- step 0 lands on the rank's own (first fully-owned) row tile."""
    tiles = ceil_div(m, block_m)
    shift = ceil_div(rank * (m // world), block_m)
    return (pid_m + shift) % tiles


def scatter_rotation(pid_m: int, m: int, rank: int, world: int, block_m: int) -> int:
    """swizzle.py:100-103 -- step 0 lands on the successor's rows."""
    tiles = ceil_div(m, block_m)
    shift = ((rank + 1) * (m // world)) // block_m
    return (pid_m + shift) % tiles


def _node_ranges(m: int, block_m: int, nnodes: int, first_node: int, mode: str):
    """Inclusive tile range per visited node, straddlers kept once (swizzle.py:109-141)."""
    rows_per_node = m // nnodes
    out = []
    for pos in range(nnodes):
        node = (first_node + pos) % nnodes
        lo_row, hi_row = node * rows_per_node, (node + 1) * rows_per_node
        first = lo_row // block_m
        last = (hi_row - 1) // block_m
        head_shared = lo_row != 0 and (lo_row - 1) // block_m == first
        tail_shared = hi_row != m and hi_row // block_m == last
        if mode == GATHER:
            # straddlers go to the node visited LAST
            if pos == 0 and head_shared:
                first += 1
            if tail_shared and (pos == 0 or pos != nnodes - 1):
                last -= 1
        elif mode == SCATTER:
            # straddlers go to the node visited FIRST
            if pos != 0 and head_shared:
                first += 1
            if pos == nnodes - 1 and tail_shared:
                last -= 1
        else:
            raise ValueError(f"unknown swizzle mode {mode!r}")
        out.append((node, first, last))
    return out


def tile_map(m: int, rank: int, world: int, nnodes: int, block_m: int, mode: str) -> np.ndarray:
    """Entry j = row-tile computed at step j (swizzle.py:144-185)."""
    if world % nnodes:
        raise ValueError("world_size not divisible by nnodes")
    if m % world:
        raise ValueError("M must divide evenly across ranks")
    lws = world // nnodes
    node, local = divmod(rank, lws)
    rows_rank = m // world
    rows_node = m // nnodes
    first_node = node if mode == GATHER else node + 1
    seq: list[int] = []
    for nid, first, last in _node_ranges(m, block_m, nnodes, first_node, mode):
        count = last - first + 1
        if count <= 0:
            continue
        if mode == GATHER:
            start_tile = ceil_div(rows_node * nid + rows_rank * local, block_m)
        else:
            start_tile = (rows_node * nid + rows_rank * (local + 1)) // block_m
        rot = max(0, start_tile - first)
        seq.extend(first + (i + rot) % count for i in range(count))
    if len(seq) != ceil_div(m, block_m):
        raise AssertionError("node ranges must partition the tile space")
    return np.asarray(seq, dtype=np.int64)


def ag_gemm_tile_map(m, rank, world, nnodes, block_m):
    return tile_map(m, rank, world, nnodes, block_m, GATHER)


def gemm_rs_tile_map(m, rank, world, nnodes, block_m):
    return tile_map(m, rank, world, nnodes, block_m, SCATTER)


@dataclass(frozen=True)
class MoeSchedule:
    """Same fields as swizzle.py:207-222."""

    expert_id: np.ndarray
    tiled_m: np.ndarray
    segment_start: np.ndarray
    segment_end: np.ndarray
    stage: np.ndarray
    ntiles: int


def moe_schedule(counts, rank: int, n_experts: int, world: int, lws: int, block_m: int) -> MoeSchedule:
    """Expert-grouped, arrival-stage-ordered tile schedule (swizzle.py:225-286).

    Within expert e the gathered rows are ordered by source rank; tile t of e
    covers rows [t*B, min((t+1)*B, tokens_e)).  Its segment is the source-rank
    range of those rows; its stage is max over segment ranks s of (s-rank)%world.
    Sort key: (expert, stage, global tile index).
    """
    c = np.asarray(counts, dtype=np.int64)
    if c.shape != (world, n_experts):
        raise ValueError("token matrix shape mismatch")
    if (c < 0).any():
        raise ValueError("token counts must be >= 0")
    if world < 1 or lws < 1 or world % lws:
        raise ValueError("tp_size must be a multiple of local_tp_size")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if block_m < 1:
        raise ValueError("block_size_m must be >= 1")
    rows = []
    gtile = 0
    for e in range(n_experts):
        ends = np.cumsum(c[:, e])  # inclusive prefix per source rank
        total = int(ends[-1]) if world else 0
        for t in range(ceil_div(total, block_m)):
            r0 = t * block_m
            r1 = min(r0 + block_m, total)
            s0 = int(np.searchsorted(ends, r0, side="right"))
            s1 = int(np.searchsorted(ends, r1 - 1, side="right"))
            stage = max((s - rank) % world for s in range(s0, s1 + 1))
            rows.append((e, stage, gtile, s0, s1))
            gtile += 1
    rows.sort(key=lambda x: (x[0], x[1], x[2]))
    arr = np.asarray(rows, dtype=np.int64).reshape(-1, 5)
    return MoeSchedule(expert_id=arr[:, 0].copy(), tiled_m=arr[:, 2].copy(),
                       segment_start=arr[:, 3].copy(), segment_end=arr[:, 4].copy(),
                       stage=arr[:, 1].copy(), ntiles=len(rows))


def render(m: int, world: int, nnodes: int, block_m: int, mode: str) -> str:
    """Text map, one row per rank, '*' on rank-straddling tiles (swizzle.py:294-322)."""
    tiles = ceil_div(m, block_m)
    rpr = m // world

    def crosses(t):
        return (t * block_m) // rpr != (min((t + 1) * block_m, m) - 1) // rpr

    star = any(crosses(t) for t in range(tiles))
    width = len(str(tiles - 1)) + int(star)
    lines = []
    for r in range(world):
        cells = [(f"{t}*" if crosses(t) else f"{t}").rjust(width)
                 for t in tile_map(m, r, world, nnodes, block_m, mode).tolist()]
        lines.append(" ".join(cells).rstrip())
    return "\n".join(lines)
