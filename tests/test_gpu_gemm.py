"""GPU parity: the tcgen05 GEMM and the fused AG-GEMM / GEMM-RS against the oracle.

Exact mode (reference tests/test_kernels.py:31-32): integer-lattice inputs in
[-8, 8) are exact in bf16 and every partial sum stays below 2^24, so the fp32
results must be bit-identical to the int64 oracle / reference fixtures.
Production mode: N(0,1) bf16 inputs, bf16 outputs, max-norm relative error
<= 2e-2 vs the fp32 oracle on the same bf16-rounded inputs (north_star).
"""

import hashlib

import numpy as np
import pytest
import torch

from tests._devices import devices_for

from oracle import collectives as O
from tests import _golden as G

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _k():
    from paper_2605_02953_b200 import kernels
    return kernels


def _ctx(world, **kw):
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    args = dict(block_m=128, block_n=256, block_k=64, group_m=4, num_gemm_sms=0,
                num_comm_sms=0, devices=devices_for(world))
    args.update(kw)
    return WorkloadContext(topology=build_topology(world, 1), **args)


def _bf16(rng, shape, scale=1.0):
    return (torch.from_numpy(rng.standard_normal(shape).astype(np.float32)) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("bm", [128, 256, 512])
@pytest.mark.parametrize("m,n,k,bn", [(128, 256, 64, 256), (256, 512, 1024, 256),
                                      (300, 200, 136, 128), (1000, 1000, 520, 256),
                                      (2048, 1536, 4096, 256), (64, 40, 8, 128)])
def test_core_gemm_vs_torch_fp32(m, n, k, bn, bm):
    K = _k()
    if bm == 512 and bn != 256:
        pytest.skip("the 512-row pair tile is built for block_n 256")
    rng = np.random.default_rng(m * 7 + n)
    a = _bf16(rng, (m, k)).cuda()
    b = _bf16(rng, (n, k)).cuda()
    out = K.gemm(a, b, block_n=bn, block_m=bm)
    ref = a.float() @ b.float().T
    torch.cuda.synchronize()
    err = O.compare(out.float().cpu().numpy(), ref.cpu().numpy())
    assert err <= TOL_BF16, err


@pytest.mark.parametrize("bm", [128, 256, 512])
@pytest.mark.parametrize("bn", [128, 256])
def test_core_gemm_exact_lattice_fp32_out(bn, bm):
    K = _k()
    if bm == 512 and bn != 256:
        pytest.skip("the 512-row pair tile is built for block_n 256")
    rng = np.random.default_rng(bn)
    m, n, k = 512, 768, 2048
    a = rng.integers(-8, 8, (m, k))
    b = rng.integers(-8, 8, (n, k))
    ta = torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).cuda()
    tb = torch.from_numpy(b.astype(np.float32)).to(torch.bfloat16).cuda()
    out = K.gemm(ta, tb, out_dtype=torch.float32, block_n=bn, block_m=bm)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.int64), a @ b.T)


def test_core_gemm_persistent_grid_and_tile_map_order_irrelevant():
    K = _k()
    rng = np.random.default_rng(3)
    m, n, k = 1024, 512, 256
    a = _bf16(rng, (m, k)).cuda()
    b = _bf16(rng, (n, k)).cuda()
    base = K.gemm(a, b)
    for bm in (128, 256, 512):
        tm = K.tile_map_tensor(m, 3, 8, 1, "ag_gemm", "cuda", bm)
        for sms in (1, 3, 148):
            out = K.gemm(a, b, num_sms=sms, tile_map=tm, group_m=3, block_m=bm)
            torch.cuda.synchronize()
            assert torch.equal(out, base)


def test_sm_die_map_and_die_ranked_grid():
    """tf_sm_die_map: every SM in one of two L2 partitions (B200: two dies); the
    die-ranked cluster ids (default TF_GEMM_DIE=1) give bit-identical results for
    full waves, partial waves and repeated launches (self-resetting counter slots)."""
    import ctypes as C
    from paper_2605_02953_b200 import _lib
    out = (C.c_uint8 * 256)()
    n = C.c_int()
    _lib.call("tf_sm_die_map", 0, out, 256, C.byref(n))
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    dies = np.frombuffer(out, np.uint8)[: n.value]
    if n.value:
        assert n.value == nsm
        assert set(dies.tolist()) == {0, 1} and min((dies == 0).sum(), (dies == 1).sum()) >= nsm // 4
    K = _k()
    rng = np.random.default_rng(5)
    m, n_, k = 4096, 2304, 512
    a = _bf16(rng, (m, k)).cuda()
    b = _bf16(rng, (n_, k)).cuda()
    want = a.float() @ b.float().T
    for sms in (148, 100, 7):
        for _ in range(3):
            out = K.gemm(a, b, num_sms=sms, block_m=512, group_m=8)
            torch.cuda.synchronize()
            assert torch.equal(out, K.gemm(a, b, num_sms=sms, block_m=512, group_m=8))
            assert (out.float() - want).abs().max().item() <= 2e-2 * want.abs().max().item()


@pytest.mark.parametrize("bm", [128, 256, 512])
@pytest.mark.parametrize("case", range(12))
def test_ag_gemm_exact_vs_reference_fixture(case, bm):
    K = _k()
    c = G.workloads()[case]
    w = c["world"]
    run = K.ag_gemm(list(c["ag_a"]), list(c["ag_b"]), _ctx(w, block_m=bm))
    for r in range(w):
        assert run.outputs[r].dtype == np.int64
        assert np.array_equal(run.outputs[r], c["ag_c"][r]), (case, r)


@pytest.mark.parametrize("case", range(12))
@pytest.mark.parametrize("variant", ["fused_asc", "fused_ring", "unfused", "fused_pair", "fused_pair512"])
def test_gemm_rs_exact_vs_reference_fixture(case, variant):
    K = _k()
    c = G.workloads()[case]
    w = c["world"]
    ctx = _ctx(w, fuse_scatter=variant.startswith("fused"),
               reduce_order="ring" if variant == "fused_ring" else "ascending",
               block_m={"fused_pair": 256, "fused_pair512": 512}.get(variant, 128))
    run = K.gemm_rs(list(c["rs_x"]), list(c["rs_w"]), ctx)
    for r in range(w):
        assert np.array_equal(run.outputs[r], c["rs_y"][r]), (case, variant, r)
    for r in range(w):
        assert not run.heap.sig_view(run.handles["counters"], r).any()


def test_config1_ag_gemm_world2_1024_exact_digest():
    """BASELINE config 1 restated on the GPU: world=2, M=N=K=1024."""
    K = _k()
    data, meta = G.config1()
    a = [x.astype(np.int64) for x in data["a"]]
    b = [x.astype(np.int64) for x in data["b"]]
    run = K.ag_gemm(a, b, _ctx(2))
    for r, o in enumerate(run.outputs):
        assert hashlib.sha256(o.astype(np.int64).tobytes()).hexdigest() == meta["sha256_per_rank"][r]


@pytest.mark.parametrize("bm", [128, 256, 512])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_ag_gemm_bf16_production_tolerance(world, bm):
    K = _k()
    rng = np.random.default_rng(world)
    mpr, n, k = 256, 384, 1024
    a = [_bf16(rng, (mpr, k)).cuda() for _ in range(world)]
    b = [_bf16(rng, (n, k), 1 / 32).cuda() for _ in range(world)]
    run = K.ag_gemm(a, b, _ctx(world, block_m=bm))
    ref = O.ref_allgather_gemm([x.float().cpu().numpy() for x in a],
                               [x.float().cpu().numpy() for x in b])
    for r in range(world):
        assert run.outputs[r].dtype == torch.bfloat16
        assert O.compare(run.outputs[r].float().cpu().numpy(), ref[r]) <= TOL_BF16


@pytest.mark.parametrize("bm", [128, 256, 512])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fused", [True, False])
def test_gemm_rs_bf16_production_tolerance(world, fused, bm):
    K = _k()
    rng = np.random.default_rng(world + 10 * fused)
    m, n, k = world * 128, 512, 768
    x = [_bf16(rng, (m, k)).cuda() for _ in range(world)]
    w = [_bf16(rng, (n, k), 1 / 32).cuda() for _ in range(world)]
    run = K.gemm_rs(x, w, _ctx(world, fuse_scatter=fused, block_m=bm))
    ref = O.ref_reduce_scatter([t.float().cpu().numpy() for t in x],
                               [t.float().cpu().numpy() for t in w])
    for r in range(world):
        assert O.compare(run.outputs[r].float().cpu().numpy(), ref[r]) <= TOL_BF16


def test_validation_errors_match_reference():
    K = _k()
    rng = np.random.default_rng(4)
    ctx = _ctx(2)
    ga = [rng.integers(-8, 8, (4, 4)).astype(np.int64) for _ in range(2)]
    gb = [rng.integers(-8, 8, (4, 4)).astype(np.int64) for _ in range(2)]
    with pytest.raises(ValueError):
        K.ag_gemm(ga[:1], gb, ctx)
    with pytest.raises(ValueError):
        K.ag_gemm(ga, [gb[0], rng.integers(-8, 8, (4, 5)).astype(np.int64)], ctx)
    with pytest.raises(ValueError):
        K.ag_gemm(ga, [gb[0], gb[1].astype(np.float32)], ctx)
    with pytest.raises(ValueError):
        K.ag_gemm([x.astype(np.int32) for x in ga], gb, ctx)
    with pytest.raises(ValueError):
        K.gemm_rs([rng.integers(-8, 8, (7, 4)).astype(np.int64) for _ in range(2)], gb, ctx)


# -- GEMM + AllReduce (ovs/kernels/gemm_ar.py; reference tests/test_kernels.py:229-282) --------


@pytest.mark.parametrize("case", range(12))
@pytest.mark.parametrize("two_shot", [False, True])
@pytest.mark.parametrize("bm", [128, 512])
def test_gemm_ar_exact_vs_reference_fixture(case, two_shot, bm):
    K = _k()
    c = G.workloads()[case]
    w = c["world"]
    n_ar = c["ar_y"].shape[1]
    b = [x[:n_ar] for x in c["ag_b"]]
    run = K.gemm_allreduce(list(c["ag_a"]), b, _ctx(w, block_m=bm, block_n=4 if n_ar % 4 == 0 else 1),
                           use_multimem_st=two_shot)
    for r in range(w):
        assert np.array_equal(run.outputs[r], c["ar_y"]), (case, two_shot, r)


def test_gemm_ar_paths_agree_and_flags_reset():
    K = _k()
    rng = np.random.default_rng(10)
    world = 4
    a = [rng.integers(-8, 8, (300, 40)) for _ in range(world)]
    b = [rng.integers(-8, 8, (264, 40)) for _ in range(world)]
    runs = [K.gemm_allreduce(a, b, _ctx(world, block_n=8), use_multimem_st=ts) for ts in (False, True)]
    want = O.ref_allreduce(a, b)
    for run in runs:
        for r in range(world):
            assert np.array_equal(run.outputs[r], want)
            assert not run.heap.sig_view(run.handles["tile_ready"], r).any()
            assert not run.heap.sig_view(run.handles["mst_sig"], r).any()


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("two_shot", [False, True])
def test_gemm_ar_bf16_tolerance(world, two_shot):
    K = _k()
    rng = np.random.default_rng(world)
    m, n, k = 1000, 768, 512
    a = [_bf16(rng, (m, k)).cuda() for _ in range(world)]
    b = [_bf16(rng, (n, k), 1 / 32).cuda() for _ in range(world)]
    run = K.gemm_allreduce(a, b, _ctx(world, block_n=256), use_multimem_st=two_shot)
    want = O.ref_allreduce([x.float().cpu().numpy() for x in a], [x.float().cpu().numpy() for x in b])
    for r in range(world):
        assert O.compare(run.outputs[r].float().cpu().numpy(), want) <= TOL_BF16


def test_gemm_ar_validation():
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    K = _k()
    rng = np.random.default_rng(12)
    a = [rng.integers(-8, 8, (4, 4)) for _ in range(2)]
    b = [rng.integers(-8, 8, (6, 4)) for _ in range(2)]
    with pytest.raises(ValueError):
        K.gemm_allreduce(a, b, _ctx(2, block_n=4))  # N=6 not divisible by block_n=4
    multi = WorkloadContext(topology=build_topology(4, 2), devices=devices_for(4))
    with pytest.raises(ValueError):
        K.gemm_allreduce([rng.integers(-8, 8, (4, 4))] * 4, [rng.integers(-8, 8, (4, 4))] * 4, multi)


def _norm_rel_err(got, want):
    # the reference's metric (tests/test_kernels.py:43-46): max-abs error / max-abs value
    diff = np.abs(np.asarray(got, np.float64) - np.asarray(want, np.float64)).max(initial=0.0)
    scale = np.abs(np.asarray(want, np.float64)).max(initial=0.0) or 1.0
    return float(diff / scale)


def test_float_fractional_tolerance_unordered():
    """Reference tests/test_kernels.py:365-381: fractional float32 gemm_rs (ring
    order) and gemm_allreduce (one- and two-shot) within norm-relative 1e-5 of the
    fp32 oracle -- the float32 contract, met with the 6-term bf16 split (tf_prep.cu)."""
    K = _k()
    rng = np.random.default_rng(18)
    world = 4
    frac = lambda shape: rng.standard_normal(shape).astype(np.float32)
    inp = [frac((world * 8, 16)) for _ in range(world)]
    w = [frac((12, 16)) for _ in range(world)]
    ref = O.ref_reduce_scatter(inp, w)
    run = K.gemm_rs(inp, w, _ctx(world, reduce_order="ring"))
    for got, want in zip(run.outputs, ref):
        assert got.dtype == np.float32
        assert _norm_rel_err(got, want) <= 1e-5
    a = [frac((8, 16)) for _ in range(world)]
    b = [frac((8, 16)) for _ in range(world)]
    want = O.ref_allreduce(a, b)
    for ts in (False, True):
        run = K.gemm_allreduce(a, b, _ctx(world, block_m=4, block_n=4, block_k=4), use_multimem_st=ts)
        for got in run.outputs:
            assert _norm_rel_err(got, want) <= 1e-5


@pytest.mark.parametrize("world,mpr,n,k", [(2, 256, 384, 512), (4, 100, 136, 1000)])
def test_float32_ag_gemm_fp32_accuracy(world, mpr, n, k):
    """float32 AG-GEMM at non-trivial K: error vs the float64 product stays at the
    level of the tensor core's fp32 accumulation (measured 6.5e-6 at K=512; the
    accumulator adds truncate, so it grows ~linearly in K/16), two orders of
    magnitude below plain bf16 rounding of the operands (~3e-3)."""
    K = _k()
    rng = np.random.default_rng(world * 31 + k)
    a = [rng.standard_normal((mpr, k)).astype(np.float32) for _ in range(world)]
    b = [rng.standard_normal((n, k)).astype(np.float32) for _ in range(world)]
    run = K.ag_gemm(a, b, _ctx(world))
    full = np.concatenate(a).astype(np.float64)
    for r in range(world):
        want = full @ b[r].astype(np.float64).T
        assert run.outputs[r].dtype == np.float32
        assert _norm_rel_err(run.outputs[r], want) <= 3e-5


def test_drop_in_team_cache_reuse_is_exact():
    """Repeated drop-in calls of one shape reuse a cached team (heap, flags, workspaces);
    alternating fused / unfused GEMM-RS and interleaved AG-GEMM calls stay bit-exact."""
    K = _k()
    rng = np.random.default_rng(21)
    world, mpr, n, k = 4, 128, 256, 192
    for it in range(3):
        a = [rng.integers(-8, 8, (mpr, k)).astype(np.int64) for _ in range(world)]
        b = [rng.integers(-8, 8, (n, k)).astype(np.int64) for _ in range(world)]
        run = K.ag_gemm(a, b, _ctx(world))
        for got, want in zip(run.outputs, O.ref_allgather_gemm(a, b)):
            assert np.array_equal(got, want), it
        x = [rng.integers(-8, 8, (world * mpr, k)).astype(np.int64) for _ in range(world)]
        w = [rng.integers(-8, 8, (n, k)).astype(np.int64) for _ in range(world)]
        for fused in (True, False):
            ctx = _ctx(world)
            ctx.fuse_scatter = fused
            run = K.gemm_rs(x, w, ctx)
            for got, want in zip(run.outputs, O.ref_reduce_scatter(x, w)):
                assert np.array_equal(got, want), (it, fused)
    assert len(K._TEAM_CACHE) <= K._TEAM_CACHE_MAX


@pytest.mark.parametrize("case", range(12))
@pytest.mark.parametrize("comm", [1, 8])
def test_ag_gemm_in_kernel_pull_exact_vs_reference_fixture(case, comm):
    """ag_pull="sm": the gather runs inside the GEMM launch (pull-engine CTAs), bit-exact
    with the reference's outputs on its fixtures."""
    c = G.workloads()[case]
    K = _k()
    w = c["world"]
    ctx = _ctx(w, ag_pull="sm", num_comm_sms=comm, block_m=256)
    run = K.ag_gemm(list(c["ag_a"]), list(c["ag_b"]), ctx)
    for r in range(w):
        assert run.outputs[r].dtype == np.int64
        assert np.array_equal(run.outputs[r], c["ag_c"][r]), (case, r)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_all_gather_gemm_in_kernel_pull_bf16(world):
    """Persistent AllGatherGemm with num_comm_sms > 0 (in-kernel pulls) vs the fp32 reference."""
    from paper_2605_02953_b200.kernels import AllGatherGemm
    from paper_2605_02953_b200.shmem import Team
    rng = np.random.default_rng(world)
    m, k, n = 512 * world, 512, 768
    team = Team(world, devices_for(world), heap_bytes=4 * m * k * 2 + (8 << 20), signal_slots=1024)
    op = AllGatherGemm(team, m, k, n, num_comm_sms=4)
    a = [_bf16(rng, (m // world, k)).cuda() for _ in range(world)]
    b = [_bf16(rng, (n, k), k ** -0.5).cuda() for _ in range(world)]
    for _ in range(2):  # second call: next epoch of the same workspace
        outs = op.forward(a, b)
        torch.cuda.synchronize()
        team.check()
        full = torch.cat(a).float()
        for r in range(world):
            want = full @ b[r].float().T
            err = (outs[r].float() - want).abs().max().item() / want.abs().max().item()
            assert err <= 2e-2, (r, err)
    team.close()
