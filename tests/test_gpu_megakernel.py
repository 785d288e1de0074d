"""GPU execution of reference task graphs by the persistent tcgen05 megakernel,
restating the reference's execution tests (tests/test_megakernel.py:173-384)."""

import numpy as np
import pytest
import torch

from paper_2605_02953_b200 import build_topology
from paper_2605_02953_b200 import megakernel as MK
from paper_2605_02953_b200.errors import DeadlockError, ProtocolError
from tests.test_megakernel_host import allreduce_program, mlp_program

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def mlp_inputs(rng, m=32, k=16, h=24):
    return {"x": rng.integers(-5, 5, (m, k)).astype(np.int64),
            "w1": rng.integers(-5, 5, (h, k)).astype(np.int64),
            "bias": rng.integers(-5, 5, (m, h)).astype(np.int64),
            "w2": rng.integers(-5, 5, (k, h)).astype(np.int64)}


def mlp_reference(v):
    return (v["x"] @ v["w1"].T + v["bias"]) @ v["w2"].T


def topo_order_shuffle(tasks, rng):
    by_layer = {}
    for t in tasks:
        by_layer.setdefault(t.task_id, []).append(t)
    for tiles in by_layer.values():
        rng.shuffle(tiles)
    order, cur = [], {k: 0 for k in by_layer}
    while len(order) < len(tasks):
        ready = [k for k in by_layer if cur[k] < len(by_layer[k])
                 and all(cur[j] == len(by_layer[j]) for j in by_layer if j < k)]
        k = ready[int(rng.integers(0, len(ready)))]
        order.append(by_layer[k][cur[k]])
        cur[k] += 1
    return order


def test_mlp_matches_sequential_across_sm_counts():
    rng = np.random.default_rng(31)
    prog = mlp_program(world=2)
    built = prog.build()
    vals = mlp_inputs(rng)
    want = mlp_reference(vals)
    for num_sms in (1, 2, 4, 8):
        run = MK.run_megakernel(prog, built, num_sms, inputs=vals)
        for r in range(2):
            assert np.array_equal(run.outputs["y"][r], want), num_sms


def test_mlp_schedule_independence():
    rng = np.random.default_rng(32)
    prog = mlp_program(world=2)
    built = prog.build()
    vals = mlp_inputs(rng)
    want = mlp_reference(vals)
    for _ in range(5):
        order = topo_order_shuffle(built.tasks, rng)
        nsm = int(rng.choice([1, 2, 4, 8]))
        q, c = MK.encode_work_queues(order, nsm)
        run = MK.run_megakernel(prog, built, nsm, queues=q, counts=c, inputs=vals)
        for r in range(2):
            assert np.array_equal(run.outputs["y"][r], want)


def test_scoreboard_flags_set_once_per_tile():
    rng = np.random.default_rng(33)
    prog = mlp_program(world=2)
    built = prog.build()
    run = MK.run_megakernel(prog, built, 4, inputs=mlp_inputs(rng))
    for sb in run.scoreboards:
        flags = sb.flags_view(sb.rank)
        used = [sb._slot(t.task_id, t.tile_id) for t in built.tasks]
        assert (flags[used] == 1).all()
        assert int(flags.sum()) == len(built.tasks)


def test_allreduce_task_sums_across_ranks():
    rng = np.random.default_rng(37)
    world = 4
    prog = allreduce_program(world)
    built = prog.build()
    a_vals = [rng.integers(-5, 5, (8, 6)).astype(np.int64) for _ in range(world)]
    w_val = rng.integers(-5, 5, (6, 6)).astype(np.int64)
    run = MK.run_megakernel(prog, built, 2, inputs={"a": a_vals, "w": w_val})
    want = sum(av @ w_val.T for av in a_vals)
    for r in range(world):
        assert np.array_equal(run.outputs["red"][r], want)


def test_float_mlp_larger_tiles():
    rng = np.random.default_rng(38)
    prog = MK.MegaProgram(build_topology(1, 1, num_sms=16))
    m, k, h = 300, 96, 200
    x = prog.tensor("x", (m, k), np.float32)
    w1 = prog.tensor("w1", (h, k), np.float32)
    y = prog.tensor("y", (m, h), np.float32)
    prog.layer("linear", [x, w1], [y], block_m=128, block_n=128)
    built = prog.build()
    xv = rng.standard_normal((m, k)).astype(np.float32)
    wv = rng.standard_normal((h, k)).astype(np.float32)
    run = MK.run_megakernel(prog, built, 8, inputs={"x": xv, "w1": wv})
    want = xv.astype(np.float64) @ wv.T.astype(np.float64)
    err = np.abs(run.outputs["y"][0] - want).max() / np.abs(want).max()
    assert err <= 5e-3  # tf32 operands (10-bit mantissa), fp32 accumulation


def test_consumer_first_schedule_deadlocks_with_named_slot():
    rng = np.random.default_rng(36)
    prog = mlp_program(world=1)
    built = prog.build()
    last_first = sorted(built.tasks, key=lambda t: -t.task_id)
    q, c = MK.encode_work_queues(last_first, 1)
    with pytest.raises(DeadlockError) as exc:
        MK.run_megakernel(prog, built, 1, queues=q, counts=c, inputs=mlp_inputs(rng), timeout_s=0.5)
    assert "scoreboard task" in str(exc.value)


def test_double_release_detected():
    prog = MK.MegaProgram(build_topology(1, 1))
    x = prog.tensor("x", (4, 4), np.int64)
    w = prog.tensor("w", (4, 4), np.int64)
    y = prog.tensor("y", (4, 4), np.int64)
    prog.layer("linear", [x, w], [y], block_m=4, block_n=4)
    built = prog.build()
    q, c = MK.encode_work_queues(built.tasks + built.tasks, 1)
    with pytest.raises(ProtocolError):
        MK.run_megakernel(prog, built, 1, queues=q, counts=c,
                          inputs={"x": np.ones((4, 4), np.int64), "w": np.ones((4, 4), np.int64)})


def test_zero_task_program():
    prog = MK.MegaProgram(build_topology(2, 1))
    prog.tensor("x", (4, 4), np.int64)
    built = prog.build()
    assert built.tasks == []
    run = MK.run_megakernel(prog, built, 4)
    assert run.outputs["x"][0].shape == (4, 4)
