"""Host side of the fused layer (config 5): planners under the reference's
builder contract, device tables, weight layout helpers and the oracle's own
consistency (CPU only)."""

import numpy as np
import pytest

from oracle import layer as OL
from oracle.collectives import compare
from paper_2605_02953_b200 import build_topology
from paper_2605_02953_b200 import layer as L
from paper_2605_02953_b200 import megakernel as MK
from paper_2605_02953_b200.errors import BuildError
from tests._layer_case import make_case


def test_registry_keeps_reference_order():
    assert MK.registered_ops()[:3] == ["linear", "add", "allreduce"]
    assert set(L.LAYER_OP_CODES) <= set(MK.registered_ops())


def test_llama_graph_dependencies():
    prog = L.llama_layer_program(build_topology(2, 1), 512, 512, 8, 2, 1024, seq_len=256)
    built = prog.build()
    by = {}
    for t in built.tasks:
        by.setdefault(t.task_id, []).append(t)
    hq = 4
    # attention (layer 2): tile (i, head pair) waits on the 256-row QKV tiles of rows <= i
    assert built.layer_configs[2]["heads_per_task"] == 2
    per_row = hq // 2
    for t in by[2]:
        i, hp = divmod(t.tile_id, per_row)
        rows = {int(lo) // 3 for p, lo, hi in built.dep_table[t.dep_start:t.dep_end] if p == 1}
        seq0 = (i // 2) * 2
        assert rows == set(range(seq0 // 2, i // 2 + 1)), (i, rows)
    # emitted shortest-first by default (position in sequence ascending)
    firsts = [t.tile_id // per_row for t in by[2]]
    assert built.layer_configs[2]["order"] == "shortest_first"
    assert firsts[0] % 2 == 0 and firsts[-1] % 2 == 1
    # o-proj tile (tm, tn) waits on every head pair of the two query tiles of its 256 rows
    for t in by[3]:
        rows = [tuple(r) for r in built.dep_table[t.dep_start:t.dep_end]]
        tm = t.tile_id // 2
        assert rows == [(2, 2 * tm * per_row, (2 * tm + 1) * per_row), (2, (2 * tm + 1) * per_row, (2 * tm + 2) * per_row)]
    # allreduce_residual rows depend on their o_part and x rows only
    for t in by[4]:
        prods = {int(r[0]) for r in built.dep_table[t.dep_start:t.dep_end]}
        assert prods == {3}
    # silu_mul output tiles are 128 wide
    assert built.layer_configs[5]["epilogue"] == "silu_mul"
    # the MLP rmsnorm is fused into the first allreduce_residual (two outputs)
    assert built.layer_ops[4] == "allreduce_residual" and built.layer_configs[4]["norm_gain"] is not None


def test_tables_and_specs():
    prog = L.llama_layer_program(build_topology(1, 1), 256, 512, 4, 2, 1024)
    built = prog.build()
    cfg, specs = L.layer_tables(prog, built)
    assert cfg.shape == (8, 16) and list(cfg[:, 0]) == [1, 2, 3, 2, 4, 2, 2, 4]
    assert cfg[1, 4] == 1 and cfg[1, 14] == 3 and cfg[1, 13] == 6 * 128
    assert cfg[5, 4] == 2 and cfg[2, 12] == 1
    g2 = next(t for t in prog.tensors if t.name == "g_mlp")
    assert cfg[4, 15] == 1 + g2.offset // 16 and cfg[7, 15] == 0
    assert specs.shape[1] == 8 and all(s[1] in (2, 3) for s in specs)
    assert all(s[0] % 16 == 0 for s in specs)


def test_planner_errors():
    p = MK.MegaProgram(build_topology(1, 1))
    bf = L.bfloat16
    x, w = p.tensor("x", (128, 100), bf), p.tensor("w", (256, 100), bf)
    y = p.tensor("y", (128, 256), bf)
    p.layer("linear", [x, w], [y])
    with pytest.raises(BuildError):
        p.build()
    p2 = MK.MegaProgram(build_topology(1, 1))
    q = p2.tensor("qkv", (256, 6 * 128), bf)
    o = p2.tensor("o", (256, 4 * 128), bf)
    p2.layer("attention", [q], [o], heads_q=4, heads_kv=2, seq_len=200)
    with pytest.raises(BuildError):
        p2.build()


def test_interleave_and_rope_table():
    g = np.arange(256 * 4, dtype=np.float32).reshape(256, 4)
    u = -g
    w = L.interleave_gate_up(g, u)
    assert np.array_equal(w[:128], g[:128]) and np.array_equal(w[128:256], u[:128])
    assert np.array_equal(w[256:384], g[128:]) and np.array_equal(w[384:], u[128:])
    t = L.rope_table(8)
    assert t.shape == (8, 128) and np.allclose(t[0, :64], 1) and np.allclose(t[0, 64:], 0)
    assert np.allclose(t[:, :64] ** 2 + t[:, 64:] ** 2, 1, atol=1e-6)


def test_oracle_tp_consistency():
    """The TP=2 sharded oracle agrees with the TP=1 oracle on the concatenated weights."""
    _, inp2, want2, _ = make_case(2, tokens=128, hidden=256, heads_q=4, heads_kv=2, ffn=512, seq=128, seed=1)
    hq, hkv = 2, 1  # per rank
    ws = inp2["w_qkv"]
    wq = [np.concatenate([w[: hq * 128] for w in ws] + [w[hq * 128:(hq + hkv) * 128] for w in ws] +
                         [w[(hq + hkv) * 128:] for w in ws])]
    blocks = lambda w: [w[b * 128:(b + 1) * 128] for b in range(w.shape[0] // 128)]
    wg = [np.concatenate([np.concatenate(blocks(w)[0::2]) for w in inp2["w_gate_up"]])]
    wu = [np.concatenate([np.concatenate(blocks(w)[1::2]) for w in inp2["w_gate_up"]])]
    wo = [np.concatenate(inp2["w_o"], axis=1)]
    w2 = [np.concatenate(inp2["w_down"], axis=1)]
    want1, _ = OL.llama_layer(inp2["x"], inp2["g_attn"], inp2["g_mlp"], inp2["rope"], wq, wo,
                              wg, wu, w2, 2 * hq, 2 * hkv, 128)
    assert compare(want1, want2) <= 2e-2


def test_oracle_attention_against_float64():
    rng = np.random.default_rng(2)
    qkv = rng.standard_normal((256, 4 * 128)).astype(np.float32)
    got = OL.causal_attention(qkv, 2, 1, 128)
    q, k, v = qkv[:, :256].reshape(256, 2, 128), qkv[:, 256:384], qkv[:, 384:]
    for s0 in (0, 128):
        for h in range(2):
            for i in (0, 5, 127):
                s = q[s0 + i, h].astype(np.float64) @ k[s0:s0 + i + 1].T.astype(np.float64) / np.sqrt(128)
                p = np.exp(s - s.max())
                p /= p.sum()
                ref = p @ v[s0:s0 + i + 1]
                assert np.allclose(got[s0 + i, h * 128:(h + 1) * 128], ref, rtol=1e-2, atol=1e-2)


def test_dataflow_order_is_topological():
    prog = L.llama_layer_program(build_topology(2, 1), 512, 512, 8, 2, 1024, seq_len=256)
    built = prog.build()
    order = L.dataflow_order(built)
    assert sorted((t.task_id, t.tile_id) for t in order) == sorted((t.task_id, t.tile_id) for t in built.tasks)
    pos = {(t.task_id, t.tile_id): i for i, t in enumerate(order)}
    for t in order:
        for p, lo, hi in built.dep_table[t.dep_start:t.dep_end]:
            for tile in range(int(lo), int(hi)):
                assert pos[(int(p), tile)] < pos[(t.task_id, t.tile_id)]
    # the final allreduce tasks are spread through the down projection, not appended
    last = [i for i, t in enumerate(order) if t.task_id == 7]
    first_down = min(i for i, t in enumerate(order) if t.task_id == 6)
    assert min(last) < max(i for i, t in enumerate(order) if t.task_id == 6)
    assert min(last) > first_down


def test_list_schedule_queues_are_topological_subsequences():
    prog = L.llama_layer_program(build_topology(2, 1), 512, 512, 8, 2, 1024, seq_len=256)
    built = prog.build()
    q, c = L.list_schedule(prog, built, 7)
    seen = []
    for cta in range(7):
        for i in range(int(c[cta])):
            seen.append((cta, i, MK.decode_task(q[i, cta])))
    assert sorted((t.task_id, t.tile_id) for _, _, t in seen) == sorted((t.task_id, t.tile_id) for t in built.tasks)
    # each queue follows the builder's topological order
    pos = {(t.task_id, t.tile_id): k for k, t in enumerate(built.tasks)}
    for cta in range(7):
        ks = [pos[(t.task_id, t.tile_id)] for cc, _, t in seen if cc == cta]
        assert ks == sorted(ks)
