"""Host side of the megakernel: wire format and graph building, pinned against
fixtures produced by the reference (tests/golden/make_golden.py) and restating
the reference's own encoding tests (tests/test_megakernel.py:27-168)."""

import json

import numpy as np
import pytest

from paper_2605_02953_b200 import build_topology
from paper_2605_02953_b200 import megakernel as MK
from paper_2605_02953_b200.errors import BuildError, ProtocolError
from tests._golden import GOLDEN


def mlp_program(world=2, m=32, k=16, h=24, dtype=np.int64, block=16):
    prog = MK.MegaProgram(build_topology(world, 1, num_sms=8))
    x = prog.tensor("x", (m, k), dtype)
    w1 = prog.tensor("w1", (h, k), dtype)
    h1 = prog.tensor("h1", (m, h), dtype)
    bias = prog.tensor("bias", (m, h), dtype)
    h2 = prog.tensor("h2", (m, h), dtype)
    w2 = prog.tensor("w2", (k, h), dtype)
    y = prog.tensor("y", (m, k), dtype)
    prog.layer("linear", [x, w1], [h1], block_m=block, block_n=block)
    prog.layer("add", [h1, bias], [h2], block_rows=block)
    prog.layer("linear", [h2, w2], [y], block_m=block, block_n=block)
    return prog


def allreduce_program(world=4):
    prog = MK.MegaProgram(build_topology(world, 1, num_sms=4))
    a = prog.tensor("a", (8, 6), np.int64)
    w = prog.tensor("w", (6, 6), np.int64)
    p = prog.tensor("p", (8, 6), np.int64)
    red = prog.tensor("red", (8, 6), np.int64)
    prog.layer("linear", [a, w], [p], block_m=4, block_n=3)
    prog.layer("allreduce", [p], [red], block_rows=4)
    return prog


@pytest.mark.parametrize("name,builder", [("mlp", mlp_program), ("allreduce", allreduce_program)])
def test_queues_deps_and_dag_match_reference(name, builder):
    z = np.load(GOLDEN / "megakernel.npz")
    dags = json.loads((GOLDEN / "megakernel_dags.json").read_text())
    built = builder().build()
    assert [built.max_task_id, built.max_tiles_per_op] == z[f"{name}_meta"].tolist()
    assert MK.deps_to_bytes(built.dep_table) == z[f"{name}_deps"].tobytes()
    for nsm in (1, 3, 8):
        q, c = MK.encode_work_queues(built.tasks, nsm)
        assert MK.queues_to_bytes(q) == z[f"{name}_q{nsm}"].tobytes()
        assert np.array_equal(c, z[f"{name}_c{nsm}"])
    assert MK.dump_task_graph(built.tasks, built.dep_table) == dags[name]


def test_registry_order_and_errors():
    assert MK.registered_ops()[:3] == ["linear", "add", "allreduce"]
    assert [MK.get_task_builder(o).task_type for o in ("linear", "add", "allreduce")] == [0, 1, 2]
    with pytest.raises(ProtocolError):
        MK.register_task_builder("linear", lambda io, cfg: None)
    with pytest.raises(BuildError):
        MK.get_task_builder("conv3d")


def random_task(rng):
    io = tuple(MK.IoSlot(offset=int(rng.integers(0, 2 ** 20)) * 16, dtype_tag=int(rng.integers(0, 2)),
                         dims=tuple(int(d) for d in rng.integers(1, 64, size=rng.integers(1, 5))))
               for _ in range(int(rng.integers(0, 5))))
    start = int(rng.integers(0, 1000))
    return MK.TaskRecord(int(rng.integers(0, 3)), int(rng.integers(0, 64)), int(rng.integers(0, 64)),
                         int(rng.integers(0, 4096)), start, start + int(rng.integers(0, 8)), io)


def test_encode_fetch_roundtrip_and_address_arithmetic():
    rng = np.random.default_rng(123)
    tasks = [random_task(rng) for _ in range(1000)]
    for nsm in (1, 3, 8):
        q, c = MK.encode_work_queues(tasks, nsm)
        assert int(c.sum()) == len(tasks)
        for i, t in enumerate(tasks):
            assert MK.fetch_task(q, i // nsm, i % nsm, c) == t
    q, c = MK.encode_work_queues(tasks[:5], 2)
    flat = q.reshape(-1)
    base = 1 * MK.INT_PER_TASK * 2
    assert flat[base] == tasks[2].task_type and flat[base + 3] == tasks[2].tile_id
    assert MK.INT_PER_TASK == 30 and MK.IO_TENSORS_OFFSET == 6


def test_encode_rejects_bad_fields_and_empty_queues():
    with pytest.raises(ValueError):
        MK.encode_task(MK.TaskRecord(0, 0, 0, 2 ** 31, 0, 0))
    with pytest.raises(ValueError):
        MK.encode_task(MK.TaskRecord(0, 0, 0, 0, 0, 0, io=(MK.IoSlot(0, 0, (0,)),)))
    q, c = MK.encode_work_queues([], 4)
    assert c.tolist() == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        MK.fetch_task(q, 0, 0, c)


def test_wire_roundtrip_and_runtime_scheduler_branch():
    rng = np.random.default_rng(9)
    tasks = [random_task(rng) for _ in range(7)]
    q, _ = MK.encode_work_queues(tasks, 3)
    assert np.array_equal(MK.queues_from_bytes(MK.queues_to_bytes(q), 3), q)
    d = np.array([[0, 0, 4], [1, 2, 3]], dtype=np.int32)
    assert np.array_equal(MK.deps_from_bytes(MK.deps_to_bytes(d)), d)
    flat = np.stack([MK.encode_task(t) for t in tasks])
    for i, t in enumerate(tasks):
        assert MK.fetch_task(flat, i, 0, runtime_scheduler=True) == t
    with pytest.raises(ValueError):
        MK.fetch_task(flat, len(tasks), 0, runtime_scheduler=True)


def test_dependency_structure():
    built = mlp_program().build()
    for t in (t for t in built.tasks if t.task_id == 1):
        rows = built.dep_table[t.dep_start:t.dep_end]
        assert {int(r[0]) for r in rows} == {0}
        tiles = sorted(x for r in rows for x in range(int(r[1]), int(r[2])))
        assert tiles == [t.tile_id * 2 + j for j in range(2)]
    built = allreduce_program().build()
    for t in (t for t in built.tasks if t.task_id == 1):
        rows = built.dep_table[t.dep_start:t.dep_end]
        assert len(rows) == 1 and (int(rows[0][1]), int(rows[0][2])) == (0, 4)
    with pytest.raises(BuildError):
        prog = MK.MegaProgram(build_topology(1, 1))
        x = prog.tensor("x", (4, 4), np.int64)
        prog.layer("softmax", [x], [x])


def test_api_surface_extras(tmp_path):
    """topology_from_config (topology.py:110-141), Token / consume_token (shmem.py:46-57),
    DeviceProp (runner.py:27-29)."""
    from paper_2605_02953_b200 import topology_from_config
    from paper_2605_02953_b200.errors import ConfigError
    t = topology_from_config({"world_size": 8, "profile": "b200", "num_sms": 148})
    assert t.world_size == 8 and t.num_sms == 148 and t.intra_node_bw == 900e9
    f = tmp_path / "topo.cfg"
    f.write_text("# comment\n[topology]\nworld_size = 4\nnnodes = 2\nintra_node_bw = 1e11\n")
    t2 = topology_from_config(str(f))
    assert (t2.world_size, t2.nnodes, t2.intra_node_bw) == (4, 2, 1e11)
    with pytest.raises(ConfigError):
        topology_from_config({"nnodes": 1})
    with pytest.raises(ConfigError):
        topology_from_config({"world_size": 2, "profile": "nope"})
    assert MK.DeviceProp(num_sms=8).num_sms == 8
    import importlib
    sh = importlib.import_module("paper_2605_02953_b200.shmem")
    tok = sh.Token(pe=0, slot=3, num_slots=2)
    assert sh.consume_token(41, tok) == 41
