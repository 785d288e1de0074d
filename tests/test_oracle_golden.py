"""Pin the CPU oracle against fixtures produced by running the reference itself.

The oracle (oracle/) is only trusted as a checker after these pass.
"""

import hashlib

import numpy as np
import pytest

from oracle import collectives as C
from oracle import moe as M
from oracle import swizzle as S
from tests import _golden as G


def test_render_matches_reference_golden():
    # reference tests/test_goldens.py:30-41
    text = "\n\n".join([
        S.render(16, 4, 1, 2, "gemm_rs"),
        S.render(16, 4, 1, 2, "ag_gemm"),
        S.render(4 * 997, 4, 2, 256, "gemm_rs"),
        S.render(4 * 997, 4, 2, 256, "ag_gemm"),
    ]) + "\n"
    assert text == G.swizzle_render_text()


def test_tile_maps_match_reference_matrix():
    cases = G.tile_maps()
    assert len(cases) > 2000
    for (m, w, nn, blk, r, mode), want in cases:
        got = S.tile_map(m, r, w, nn, blk, mode)
        assert np.array_equal(got, want), (m, w, nn, blk, r, mode)


def test_known_answers():
    # reference tests/test_swizzle.py:39-41, 63-70, 251-254
    assert S.grouped_pid(0, 4, 4, 2) == (0, 0)
    assert S.grouped_pid(5, 4, 4, 2) == (1, 2)
    assert S.gather_rotation(0, 8, 1, 4, 2) == 1
    assert S.scatter_rotation(0, 8, 1, 4, 2) == 2
    rows = S.render(8, 4, 1, 2, "gemm_rs").splitlines()
    assert rows == ["1 2 3 0", "2 3 0 1", "3 0 1 2", "0 1 2 3"]


def test_intranode_collapse():
    for w in (1, 2, 4, 8):
        for mpr in (24, 997):
            m = mpr * w
            for r in range(w):
                ag = S.tile_map(m, r, w, 1, 16, "ag_gemm")
                rs = S.tile_map(m, r, w, 1, 16, "gemm_rs")
                for i in range(len(ag)):
                    assert ag[i] == S.gather_rotation(i, m, r, w, 16)
                    assert rs[i] == S.scatter_rotation(i, m, r, w, 16)


def test_grouped_pid_bijective():
    for tm, tn, g in [(4, 4, 2), (5, 3, 2), (7, 2, 3), (1, 9, 4), (64, 14, 8)]:
        seen = {S.grouped_pid(p, tm, tn, g) for p in range(tm * tn)}
        assert len(seen) == tm * tn
    with pytest.raises(ValueError):
        S.grouped_pid(16, 4, 4, 2)


def test_moe_schedule_matches_reference():
    for c in G.moe_cases():
        s = S.moe_schedule(c["routing"], c["rank"], c["experts"], c["tp"], c["tp"], c["block"])
        got = np.stack([s.expert_id, s.tiled_m, s.segment_start, s.segment_end, s.stage],
                       axis=1) if s.ntiles else np.zeros((0, 5), np.int64)
        assert np.array_equal(got, c["sched"]), c["routing"]


def test_workload_oracles_match_reference_simulation():
    for c in G.workloads():
        w = c["world"]
        got = C.ref_allgather_gemm(list(c["ag_a"]), list(c["ag_b"]))
        assert all(np.array_equal(g, c["ag_c"][r]) for r, g in enumerate(got))
        got = C.ref_reduce_scatter(list(c["rs_x"]), list(c["rs_w"]))
        assert all(np.array_equal(g, c["rs_y"][r]) for r, g in enumerate(got))
        n_ar = c["ar_y"].shape[1]
        got = C.ref_allreduce(list(c["ag_a"]), [b[:n_ar] for b in c["ag_b"]])
        assert np.array_equal(got, c["ar_y"])
        routing = c["moe_routing"]
        rows = routing.sum(axis=1)
        edges = np.concatenate([[0], np.cumsum(rows)])
        toks = [c["moe_tok"][edges[r]:edges[r + 1]] for r in range(w)]
        got = C.ref_group_gemm(toks, [list(x) for x in c["moe_w"]], routing)
        assert all(np.array_equal(g, c["moe_y"][r]) for r, g in enumerate(got))


def test_config1_oracle_matches_reference_digest():
    data, meta = G.config1()
    a = [x.astype(np.int64) for x in data["a"]]
    b = [x.astype(np.int64) for x in data["b"]]
    outs = C.ref_allgather_gemm(a, b)
    for r, o in enumerate(outs):
        assert hashlib.sha256(o.astype(np.int64).tobytes()).hexdigest() == meta["sha256_per_rank"][r]


def test_compare_metric():
    assert C.compare(np.zeros(3), np.zeros(3)) == 0.0
    assert C.compare(np.array([1.0, 2.0]), np.array([1.0, 4.0])) == pytest.approx(0.5)


def test_moe_oracle_layout_matches_gather_tokens_by_expert():
    # the EP receive layout restricted to a rank's experts == the reference's
    # expert-major gather (oracles.py:38-50) of expert-sorted chunks
    rng = np.random.default_rng(5)
    world, e, t, k, h = 4, 8, 13, 3, 5
    logits = [rng.standard_normal((t, e)).astype(np.float32) for _ in range(world)]
    idx = [M.topk_route(lg, k)[0] for lg in logits]
    x = [rng.integers(-8, 8, (t, h)).astype(np.int64) for _ in range(world)]
    counts = M.routing_counts(idx, e)
    sorted_shards = [x[s][M.send_order(idx[s], e)[:, 0]] for s in range(world)]
    full = C.gather_tokens_by_expert(sorted_shards, counts)
    recv = M.dispatch(x, idx, e)
    assert np.array_equal(np.concatenate(recv), full)


def test_topk_rule_ties_to_lower_expert():
    lg = np.array([[1.0, 3.0, 3.0, 0.0]], dtype=np.float32)
    idx, w = M.topk_route(lg, 2)
    assert idx.tolist() == [[1, 2]]
    assert np.allclose(w, [[0.5, 0.5]])


def test_dispatch_layout_fast_equals_loop_oracle():
    """The vectorised layout used at full config-4 size equals the loop oracle."""
    rng = np.random.default_rng(7)
    for world, e, k, t in [(1, 8, 2, 5), (2, 8, 2, 37), (4, 16, 4, 50), (8, 64, 8, 96), (8, 256, 8, 64)]:
        idx = [np.stack([rng.choice(e, size=k, replace=False) for _ in range(t)]).astype(np.int32)
               for _ in range(world)]
        counts, recv, slot_row = M.dispatch_layout(idx, e, world)
        c2, rsrc, rtok, sr2 = M.dispatch_layout_fast(idx, e, world)
        assert np.array_equal(counts, c2)
        for d in range(world):
            assert [(s, t_) for s, t_, _ in recv[d]] == list(zip(rsrc[d].tolist(), rtok[d].tolist()))
        for s in range(world):
            assert np.array_equal(slot_row[s], sr2[s])
