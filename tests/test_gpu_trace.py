"""Reference protocol assertions checked on the real kernels through device
traces (reference tests/test_kernels.py:84-113)."""

import json

import numpy as np
import pytest
import torch

from tests._devices import devices_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _ctx(world, **kw):
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    args = dict(block_m=128, block_n=128, group_m=2, num_gemm_sms=0, num_comm_sms=0,
                devices=devices_for(world))
    args.update(kw)
    return WorkloadContext(topology=build_topology(world, 1), **args)


def _traced(fn):
    """Run fn with device tracing on every GPU (ranks may sit on different devices)
    and merge the rings."""
    from paper_2605_02953_b200 import trace as T
    devs = range(torch.cuda.device_count())
    for d in devs:
        T.enable(d)
    try:
        out = fn()
        for d in devs:
            torch.cuda.synchronize(d)
        events = []
        for d in devs:
            events += T.collect(d).events
        events.sort(key=lambda e: (e.t_start, e.rank, e.worker_id))
        return out, T.Trace(events)
    finally:
        for d in devs:
            T.disable(d)


def test_straddling_tiles_wait_on_both_chunks():
    # m_per_rank=96 with 128-row tiles: tiles crossing a chunk boundary wait on 2 flags
    from paper_2605_02953_b200.kernels import ag_gemm
    from oracle import collectives as O
    rng = np.random.default_rng(2)
    world = 4
    a = [rng.integers(-8, 8, (96, 64)) for _ in range(world)]
    b = [rng.integers(-8, 8, (256, 64)) for _ in range(world)]
    run, tr = _traced(lambda: ag_gemm(a, b, _ctx(world)))
    for got, want in zip(run.outputs, O.ref_allgather_gemm(a, b)):
        assert np.array_equal(got, want)
    waits = [e for e in tr.by_kind("wait") if e.payload["name"] == "wait_chunks"]
    assert waits and any(e.payload["num_slots"] == 2 for e in waits)
    assert {e.rank for e in waits} == set(range(world))


@pytest.mark.parametrize("swizzle", [True, False])
def test_gather_order_first_tile_is_local_chunk(swizzle):
    # aligned chunks: with the gather swizzle every rank's step-0 tile reads its own
    # chunk (the one that needs no transfer); without it, chunk 0
    from paper_2605_02953_b200.kernels import ag_gemm
    rng = np.random.default_rng(3)
    world = 4
    a = [rng.integers(-8, 8, (256, 64)) for _ in range(world)]
    b = [rng.integers(-8, 8, (128, 64)) for _ in range(world)]
    _, tr = _traced(lambda: ag_gemm(a, b, _ctx(world, swizzle=swizzle, num_gemm_sms=1)))
    for r in range(world):
        waits = [e for e in tr.by_kind("wait") if e.rank == r]
        first = min(waits, key=lambda e: e.t_start)
        assert first.payload["slot"] == (r if swizzle else 0)


def test_compute_events_cover_every_tile_and_chrome_schema(tmp_path):
    from paper_2605_02953_b200 import trace as T
    from paper_2605_02953_b200.kernels import gemm
    x = torch.randn(1024, 512, device="cuda").to(torch.bfloat16)
    w = torch.randn(768, 512, device="cuda").to(torch.bfloat16)
    _, tr = _traced(lambda: gemm(x, w, block_m=256, block_n=256))
    tiles = {e.payload["tile"] for e in tr.by_kind("compute")}
    assert tiles == set(range(4 * 3))
    assert len(tr.by_kind("store")) == 12 * 2  # one drain per CTA of each pair
    assert all(e.t_end >= e.t_start for e in tr.events)
    path = tmp_path / "t.json"
    T.export_chrome_trace(tr, path)
    events = json.loads(path.read_text())
    assert events and {"name", "cat", "ph", "ts", "dur", "pid", "tid", "args"} <= set(events[0])


@pytest.mark.parametrize("fuse", [True, False])
def test_gemm_rs_counter_protocol_fires_on_fourth_tile(fuse):
    """ovs tests/test_kernels.py:164-191 on the real kernels: 2 row tiles x 2 column
    tiles feed each owner row block (world 2, 128-row blocks, block_n 128); the
    counter reaches exactly 4 through bumps 1, 2, 3, 4, and the owner's reduce sees
    the block ready no earlier than the 4th bump (%globaltimer)."""
    from oracle import collectives as O
    from paper_2605_02953_b200.kernels import gemm_rs
    rng = np.random.default_rng(6)
    world = 2
    m, n, k = world * 256, 256, 64
    inp = [rng.integers(-8, 8, (m, k)) for _ in range(world)]
    w = [rng.integers(-8, 8, (n, k)) for _ in range(world)]
    run, tr = _traced(lambda: gemm_rs(inp, w, _ctx(world, fuse_scatter=fuse, num_gemm_sms=4)))
    for got, want in zip(run.outputs, O.ref_reduce_scatter(inp, w)):
        assert np.array_equal(got, want)
    sig = tr.by_kind("signal")
    bumps, ready = {}, {}
    for e in sig:
        key = (e.payload["pe"], e.payload["slot"])
        if e.payload["name"] == "atomic_add":
            bumps.setdefault(key, []).append((e.t_start, e.payload["value"]))
        else:
            ready.setdefault(key, []).append((e.t_start, e.payload["value"]))
    blocks = {(r, b) for r in range(world) for b in range(r * 2, r * 2 + 2)}
    assert set(bumps) == blocks and set(ready) == blocks
    for key, hist in bumps.items():
        assert sorted(v for _, v in hist) == [1, 2, 3, 4], key
        fourth = max(t for t, v in hist if v == 4)
        assert all(t >= fourth for t, _ in ready[key]), key
        assert all(v == 4 for _, v in ready[key]), key
