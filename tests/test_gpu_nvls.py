"""NVLS multicast region: multimem_ld_reduce / multimem_st as
multimem.ld_reduce / multimem.st through a multicast object (tf_nvls.cu), and the
two-shot GEMM+AllReduce through the switch.

NVLS needs one GPU per PE on an NVSwitch box; on a single-GPU lease the multicast
object cannot be created, so the NVLS tests skip and the fallback test checks
that the same API keeps working over the P2P heap."""

import numpy as np
import pytest
import torch

from oracle import collectives as OC
from tests._devices import devices_for, distinct

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _nvls_team(world, nbytes=64 << 20):
    from paper_2605_02953_b200.shmem import SymmetricHeap, Team
    from paper_2605_02953_b200.topology import build_topology
    if not distinct(world):
        pytest.skip(f"NVLS needs {world} GPUs")
    team = Team(world, devices_for(world), 1 << 24, 256)
    if not team.enable_nvls(nbytes):
        team.close()
        pytest.skip("multicast objects unavailable on this box")
    return team, SymmetricHeap(build_topology(world, 1), team=team)


def test_probe_reports_support():
    from paper_2605_02953_b200.shmem import Team
    assert Team.nvls_supported(0) in (True, False)


def test_fallback_without_nvls():
    """Shared device: enable_nvls declines, alloc_multimem lands on the P2P heap and
    multimem_ld_reduce / multimem_st keep the reference semantics."""
    from paper_2605_02953_b200.shmem import SymmetricHeap, Team
    from paper_2605_02953_b200.topology import build_topology
    world = 2
    team = Team(world, [0, 0], 1 << 20, 64)
    assert team.enable_nvls(1 << 20) is False and not team.nvls_enabled
    heap = SymmetricHeap(build_topology(world, 1), team=team)
    h = heap.alloc_multimem(4096)
    assert h.space == "heap"
    for r in range(world):
        heap.view(h, r, torch.int64)[:].copy_(torch.arange(512, device="cuda") * (r + 1))
    got = heap.multimem_ld_reduce(h, 0, torch.int64, 512, 0)
    assert torch.equal(got.cpu(), torch.arange(512) * 3)
    heap.multimem_st(h, 0, torch.full((512,), 7, dtype=torch.int64), 1)
    for r in range(world):
        assert torch.equal(heap.view(h, r, torch.int64).cpu(), torch.full((512,), 7, dtype=torch.int64))
    team.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multimem_reduce_and_store(world):
    team, heap = _nvls_team(world)
    n = 1 << 16
    h = heap.alloc_multimem(n * 8)
    assert h.space == "nvls"
    rng = np.random.default_rng(world)
    vals = [rng.integers(-64, 64, n) for _ in range(world)]
    for dt in (torch.int64, torch.float32, torch.bfloat16):
        for r in range(world):
            heap.view(h, r, dt)[:n].copy_(torch.from_numpy(vals[r]).to(dt))
        torch.cuda.synchronize()
        want = np.sum(vals, axis=0)
        for pe in range(world):
            got = heap.multimem_ld_reduce(h, 0, dt, n, pe).cpu().to(torch.float64).numpy()
            torch.cuda.synchronize()
            assert np.array_equal(got, want.astype(np.float64)), (dt, pe)  # lattice: exact
    vec = torch.arange(n, dtype=torch.float32)
    heap.multimem_st(h, 0, vec, 0)
    torch.cuda.synchronize()
    for r in range(world):
        assert torch.equal(heap.view(h, r, torch.float32)[:n].cpu(), vec)
    team.close()


@pytest.mark.parametrize("world", [2, 8])
def test_gemm_allreduce_two_shot_over_nvls(world):
    """Two-shot GEMM+AR with the NVLS region: integer lattice exact vs the oracle."""
    from paper_2605_02953_b200 import WorkloadContext, build_topology
    from paper_2605_02953_b200.kernels import gemm_allreduce
    if not distinct(world):
        pytest.skip(f"NVLS needs {world} GPUs")
    from paper_2605_02953_b200.shmem import Team
    probe = Team(world, devices_for(world), 1 << 20, 64)
    ok = probe.enable_nvls(1 << 21)
    probe.close()
    if not ok:
        pytest.skip("multicast objects unavailable on this box")
    rng = np.random.default_rng(5)
    m, n, k = 512, 512, 256
    a = [rng.integers(-8, 8, (m, k)).astype(np.int64) for _ in range(world)]
    b = [rng.integers(-8, 8, (n, k)).astype(np.int64) for _ in range(world)]
    ctx = WorkloadContext(topology=build_topology(world, 1), block_m=128, block_n=256,
                          devices=devices_for(world), use_multimem_st=True)
    run = gemm_allreduce(a, b, ctx)
    want = OC.ref_allreduce(a, b)
    for r in range(world):
        assert np.array_equal(run.outputs[r], want[r] if isinstance(want, list) else want)
