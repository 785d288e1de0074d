"""GPU parity of the fused AllGather + grouped GEMM (ag_moe_group_gemm,
ovs/kernels/ag_moe.py:20-142).

One launch per rank: pull-engine CTAs gather the peers' dynamic-size chunks
into expert-major rows while the grouped tcgen05 GEMM walks the swizzle_ag_moe
schedule, waiting per tile on the source ranks its rows come from.  Checked
against a float64 restatement of ag_moe.py's output (expert-major rows of the
gathered tokens times each rank's expert shard) at the bf16 tolerance of
north_star (max-norm relative 2e-2), exactly on the integer lattice, and
through the device trace (each tile's waits cover exactly its
[segment_start, segment_end] sources).  The reference's own exact-mode fixtures
run through the drop-in in tests/test_gpu_moe.py.
"""

import numpy as np
import pytest
import torch

from oracle import swizzle as OS
from tests._devices import devices_for

pytestmark = pytest.mark.gpu
TOL_BF16 = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _reference(routing, toks, wts):
    """ag_moe.py:120-142 restated: out[expert_base[e] + j] = gathered_e[j] @ W[e].T,
    gathered_e = rows of expert e from ranks 0..w-1 in rank order."""
    world, E = routing.shape
    edges = np.concatenate([np.zeros((world, 1), np.int64), np.cumsum(routing, axis=1)], axis=1)
    rows = []
    for e in range(E):
        for s in range(world):
            rows.append(toks[s][edges[s, e]:edges[s, e + 1]])
    g = np.concatenate(rows) if rows else np.zeros((0, toks[0].shape[1]))
    ebase = np.concatenate([[0], np.cumsum(routing.sum(axis=0))])
    outs = []
    for r in range(world):
        o = np.zeros((g.shape[0], wts[r].shape[1]))
        for e in range(E):
            o[ebase[e]:ebase[e + 1]] = g[ebase[e]:ebase[e + 1]] @ wts[r][e].T
        outs.append(o)
    return outs


def _run(world, E, n, k, routing, *, block_m=128, block_n=256, comm=0, swizzle=True, seed=0,
         lattice=False, trace=False):
    from paper_2605_02953_b200 import moe as M
    from paper_2605_02953_b200.shmem import Team
    rng = np.random.default_rng(seed)
    devs = devices_for(world)
    total = int(routing.sum())
    if lattice:
        toks = [rng.integers(-4, 5, (int(routing[r].sum()), k)).astype(np.float64) for r in range(world)]
        wts = [rng.integers(-4, 5, (E, n, k)).astype(np.float64) for _ in range(world)]
    else:
        toks = [rng.standard_normal((int(routing[r].sum()), k)) for r in range(world)]
        wts = [rng.standard_normal((E, n, k)) / np.sqrt(k) for _ in range(world)]
    # the kernel's inputs are bf16: compare against the product of the rounded inputs
    tb = [torch.from_numpy(t).to(torch.bfloat16) for t in toks]
    wb = [torch.from_numpy(w).to(torch.bfloat16) for w in wts]
    want = _reference(routing, [t.double().numpy() for t in tb], [w.double().numpy() for w in wb])
    team = Team(world, devs, M._agmoe_heap_bytes(max(total, 1), k, E, world, block_m), 4 * world + 64)
    odt = torch.float32 if lattice else torch.bfloat16
    op = M.AgMoeGroupGemm(team, E, n, k, max(total, 1), block_m=block_m, block_n=block_n,
                          num_comm_sms=comm, swizzle=swizzle, out_dtype=odt)
    tt = [tb[r].to(f"cuda:{devs[r]}") if tb[r].shape[0] else None for r in range(world)]
    ww = [wb[r].to(f"cuda:{devs[r]}").contiguous() for r in range(world)]
    if trace:
        from paper_2605_02953_b200 import trace as T
        T.enable(devs[0], 1 << 16)
    outs = op(routing, tt, ww)
    for d in sorted(set(devs)):
        torch.cuda.synchronize(d)
    events = None
    if trace:
        from paper_2605_02953_b200 import trace as T
        events = T.collect(devs[0], 1 << 16)
        T.disable(devs[0])
    team.check()
    got = [o.double().cpu().numpy() for o in outs]
    team.close()
    return got, want, events


def _check(got, want, exact=False):
    for r, (g, w) in enumerate(zip(got, want)):
        assert g.shape == w.shape, (r, g.shape, w.shape)
        if exact:
            assert np.array_equal(g, w), r
        elif w.size:
            err = np.abs(g - w).max() / max(np.abs(w).max(), 1e-30)
            assert err <= TOL_BF16, (r, err)


def _routing(rng, world, E, lo=0, hi=300, zero_frac=0.2):
    r = rng.integers(lo, hi, size=(world, E))
    r[rng.random((world, E)) < zero_frac] = 0
    return r.astype(np.int64)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("block_m,block_n", [(128, 256), (256, 256), (128, 128)])
def test_ag_moe_bf16_vs_reference(world, block_m, block_n):
    rng = np.random.default_rng(world * 7 + block_m + block_n)
    E, n, k = 12, 384, 512
    routing = _routing(rng, world, E)
    got, want, _ = _run(world, E, n, k, routing, block_m=block_m, block_n=block_n)
    _check(got, want)


@pytest.mark.parametrize("world,swizzle,comm", [(2, False, 2), (4, True, 4), (8, True, 16), (8, False, 8)])
def test_ag_moe_exact_lattice(world, swizzle, comm):
    """Integer-lattice inputs: the fp32-accumulated bf16 product is exact, so the
    output must equal the float64 reference bit for bit (any ordering, any pull
    split or missed wait would show)."""
    rng = np.random.default_rng(100 + world)
    E, n, k = 9, 256, 256
    routing = _routing(rng, world, E, 0, 200, 0.3)
    got, want, _ = _run(world, E, n, k, routing, comm=comm, swizzle=swizzle, lattice=True)
    _check(got, want, exact=True)


def test_ag_moe_empty_ranks_and_experts():
    """A rank with no rows, experts with no tokens, a single-row expert."""
    world, E, n, k = 4, 6, 128, 128
    routing = np.array([[0, 0, 0, 0, 0, 0],
                        [5, 0, 1, 0, 300, 0],
                        [0, 0, 0, 0, 129, 0],
                        [0, 0, 0, 1, 0, 0]], dtype=np.int64)
    got, want, _ = _run(world, E, n, k, routing, lattice=True)
    _check(got, want, exact=True)


def test_ag_moe_deepseek_like_shapes():
    """DeepSeek-V3-like expert shapes (256 experts, hidden 7168) at EP=8 emulated,
    512 tokens per rank routed top-8 (4096 rows per rank), N = 256 per rank."""
    world, E, n, k = 8, 256, 256, 7168
    rng = np.random.default_rng(3)
    routing = np.zeros((world, E), dtype=np.int64)
    for r in range(world):
        idx = np.argsort(rng.standard_normal((512, E)), axis=1)[:, :8]
        routing[r] = np.bincount(idx.ravel(), minlength=E)
    got, want, _ = _run(world, E, n, k, routing, block_m=128, seed=5)
    _check(got, want)


def test_ag_moe_waits_follow_segments():
    """Every tile's recorded waits (trace kind 1) name exactly the source ranks
    [segment_start, segment_end] of its schedule slot that were not yet known
    to have arrived, and each source is waited for at most once per CTA."""
    world, E, n, k = 4, 5, 256, 256
    rng = np.random.default_rng(11)
    routing = _routing(rng, world, E, 50, 400, 0.0)
    got, want, ev = _run(world, E, n, k, routing, lattice=True, trace=True)
    _check(got, want, exact=True)
    waits = ev.by_kind("wait")
    assert waits, "no wait events recorded"
    num_pid_n = -(-n // 256)
    for r in range(world):
        sched = OS.moe_schedule(routing, r, E, world, world, 128)
        mine = [x for x in waits if x.rank == r]
        assert mine or world == 1
        for e in mine:
            slot = e.payload["tile"] // num_pid_n
            s0, cnt = e.payload["slot"], e.payload["num_slots"]
            assert int(sched.segment_start[slot]) <= s0
            assert s0 + cnt - 1 <= int(sched.segment_end[slot])


def test_ag_moe_validation_errors():
    from paper_2605_02953_b200 import moe as M
    from paper_2605_02953_b200.shmem import Team
    team = Team(2, devices_for(2), 1 << 22, 64)
    with pytest.raises(ValueError):
        M.AgMoeGroupGemm(team, 4, 100, 64, 128)  # n % 8
    op = M.AgMoeGroupGemm(team, 4, 64, 64, 16)
    routing = np.full((2, 4), 4, dtype=np.int64)  # total 32 > max_rows 16
    toks = [torch.zeros((16, 64), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    wts = [torch.zeros((4, 64, 64), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    with pytest.raises(Exception):
        op(routing, toks, wts)
    team.close()
