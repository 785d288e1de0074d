"""GEMM+ReduceScatter summation order = the reference's (ovs/kernels/gemm_rs.py).

Integer fixtures cannot see the order of a sum.  Here each rank's partial is a
column of order-sensitive float32 values (+-2^24 next to small integers), exact
through the GEMM (k = 1 against a ones weight, fp32 6-term split path), so the
fp32 reduction must reproduce the reference's tree bit for bit:
  fused   : one fold over the world in reduce_visit_order (_fused_reducer)
  unfused : per node a fold in reduce_visit_order -- or the neighbour ring of
            _scatter_ring when assume_full_mesh_links=False -- then a fold of the
            node partials in reduce_visit_order over nodes (_hier_reducer).
Also the reference's multi-node exact test (tests/test_kernels.py:150-160)."""

import numpy as np
import pytest
import torch

from oracle import collectives as OC
from tests._devices import devices_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _visit(begin, n, order):  # ovs/kernels/context.py:77-81
    return list(range(n)) if order == "ascending" else [(begin + 1 + i) % n for i in range(n)]


def _fold(vals):
    acc = vals[0].copy()
    for v in vals[1:]:
        acc = (acc + v).astype(np.float32)
    return acc


def _reference_rows(parts, owner, world, nnodes, order, fused, full_mesh):
    """Rows of `owner` summed in the reference's order (float32)."""
    mpr = parts[0].shape[0] // world
    rows = [p[owner * mpr:(owner + 1) * mpr].astype(np.float32) for p in parts]
    if fused:
        return _fold([rows[s] for s in _visit(owner, world, order)])
    lws = world // nnodes
    node, local = owner // lws, owner % lws
    intra = _visit(local, lws, "ring" if (not full_mesh and lws > 1) else order)
    node_parts = [_fold([rows[nd * lws + j] for j in intra]) for nd in range(nnodes)]
    return _fold([node_parts[nd] for nd in _visit(node, nnodes, order)])


@pytest.mark.parametrize("world,nnodes", [(4, 1), (4, 2), (8, 2), (8, 4)])
@pytest.mark.parametrize("order", ["ascending", "ring"])
@pytest.mark.parametrize("mode", ["fused", "unfused_mesh", "unfused_ring"])
def test_rs_summation_order_matches_reference(world, nnodes, order, mode):
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    from paper_2605_02953_b200.kernels import gemm_rs
    rng = np.random.default_rng(world * 10 + nnodes)
    m, n = world * 128, 64
    big = np.float32(2.0 ** 24)
    choices = np.array([big, -big, 1.0, 3.0, -1.0, 0.5], dtype=np.float32)
    inp = [rng.choice(choices, size=(m, 1)).astype(np.float32) for _ in range(world)]
    w = [np.ones((n, 1), dtype=np.float32) for _ in range(world)]
    fused = mode == "fused"
    ctx = WorkloadContext(topology=build_topology(world, nnodes), block_m=128, block_n=128,
                          fuse_scatter=fused, reduce_order=order, devices=devices_for(world))
    run = gemm_rs(inp, w, ctx, assume_full_mesh_links=(mode != "unfused_ring"))
    parts = [np.repeat(x, n, axis=1) for x in inp]
    for r in range(world):
        want = _reference_rows(parts, r, world, nnodes, order, fused, mode != "unfused_ring")
        assert run.outputs[r].dtype == np.float32
        assert np.array_equal(run.outputs[r].view(np.uint32), want.view(np.uint32)), (r, mode, order)


def test_gemm_rs_multinode_exact():
    """ovs tests/test_kernels.py:150-160 on the device."""
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    from paper_2605_02953_b200.kernels import gemm_rs
    rng = np.random.default_rng(5)
    for world, nnodes in ((4, 2), (8, 2), (8, 4)):
        inp = [rng.integers(-8, 8, (world * 4, 5)) for _ in range(world)]
        w = [rng.integers(-8, 8, (6, 5)) for _ in range(world)]
        ref = OC.ref_reduce_scatter(inp, w)
        for mesh in (True, False):
            ctx = WorkloadContext(topology=build_topology(world, nnodes), block_m=128, block_n=128,
                                  devices=devices_for(world))
            run = gemm_rs(inp, w, ctx, assume_full_mesh_links=mesh)
            for r in range(world):
                assert np.array_equal(run.outputs[r], ref[r])
