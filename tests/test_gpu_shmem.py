"""GPU tests of the symmetric-heap primitives, mirroring the reference's
tests/test_shmem.py semantics (alloc symmetry, put-then-signal visibility,
all-of wait, atomics, barrier_all, views) on real device memory.  Several PEs
share cuda:0 (single-device team)."""

import numpy as np
import pytest
import torch

from tests._devices import devices_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _heap(world=4, data=1 << 20, slots=256):
    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200.shmem import SymmetricHeap
    return SymmetricHeap(build_topology(world, 1), data_bytes=data, signal_slots=slots,
                         devices=devices_for(world))


def test_alloc_symmetric_aligned_and_disjoint():
    h = _heap()
    a = h.alloc(100)
    b = h.alloc(7, align=64)
    z = h.alloc(0)
    assert a.offset % 16 == 0 and b.offset % 64 == 0
    assert b.offset >= a.offset + 100
    assert z.nbytes == 0
    for pe in range(4):  # same offset on every PE, distinct memory
        h.view(a, pe, np.uint8)[:] = pe
    torch.cuda.synchronize()
    for pe in range(4):
        assert (h.view(a, pe, np.uint8).cpu().numpy() == pe).all()


def test_alloc_exhaustion_and_collective_mismatch():
    from paper_2605_02953_b200.errors import AllocationError, ProtocolError
    h = _heap(data=4096, slots=8)
    with pytest.raises(AllocationError):
        h.alloc(1 << 20)
    with pytest.raises(AllocationError):
        h.alloc_signals(1 << 12)
    with pytest.raises(ProtocolError):
        h.alloc_collective([16, 32, 16, 16])
    assert h.alloc_collective([16] * 4).nbytes == 16


def test_put_then_signal_visible_and_wait():
    h = _heap()
    buf = h.alloc(4096)
    sig = h.alloc_signals(4)
    src = torch.arange(1024, dtype=torch.float32, device="cuda")
    h.putmem_signal(h.symm_at(buf, 2), 0, src, sig, 1, 7, from_pe=0)
    h.wait(sig, 1, 1, pe=2, value=7)
    got = h.view(buf, 2, np.float32, (1024,))
    torch.cuda.synchronize()
    assert torch.equal(got, src)
    assert h.sig_view(sig, 2).tolist() == [0, 7, 0, 0]


def test_signal_add_and_all_of_wait():
    h = _heap()
    sig = h.alloc_signals(3)
    for _ in range(5):
        h.atomic_add(sig, 0, 2, pe=1)
    h.st(sig, 1, 10, pe=1)
    h.notify(sig, 2, pe=1, value=10)
    h.wait(sig, 1, 2, pe=1, value=10)  # all-of over slots 1..2
    torch.cuda.synchronize()
    assert h.sig_view(sig, 1).tolist() == [10, 10, 10]
    h.reset_signals(sig, 1)
    torch.cuda.synchronize()
    assert not h.sig_view(sig, 1).any()


def test_getmem_and_barrier_all():
    h = _heap()
    buf = h.alloc(256)
    for pe in range(4):
        h.view(buf, pe, np.int32)[:] = 100 + pe
    h.barrier_all()
    dst = torch.empty(64, dtype=torch.int32, device="cuda")
    h.getmem(dst, h.symm_at(buf, 3), 0, from_pe=0)
    torch.cuda.synchronize()
    assert (dst.cpu().numpy() == 103).all()
    h.team.check()


def test_range_and_scope_validation():
    h = _heap()
    buf = h.alloc(64)
    sig = h.alloc_signals(2)
    with pytest.raises(ValueError):
        h.putmem(h.symm_at(buf, 0), 32, torch.zeros(64, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        h.st(sig, 2, 1, pe=0)
    with pytest.raises(ValueError):
        h.st(sig, 0, 1, pe=0, scope="cta")
    with pytest.raises(ValueError):
        h.symm_at(buf, 4)


# -- node-team collectives: multimem_ld_reduce / multimem_st (ovs/shmem.py:335-385) -------


@pytest.mark.parametrize("world", [1, 2, 4])
def test_multimem_reduce_and_broadcast(world):
    import numpy as np
    import torch
    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200.shmem import SymmetricHeap
    heap = SymmetricHeap(build_topology(world, 1), data_bytes=1 << 22, signal_slots=64,
                         devices=devices_for(world))
    rng = np.random.default_rng(world)
    h = heap.alloc(4096 * 8)
    # int64: exact ascending sum
    vals = [rng.integers(-1000, 1000, 4096) for _ in range(world)]
    for r in range(world):
        heap.view(h, r, np.int64, (4096,)).copy_(torch.from_numpy(vals[r]))
    got = heap.multimem_ld_reduce(h, 0, np.int64, 4096, pe=world - 1)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), np.sum(vals, axis=0))
    # fp32: ascending-rank fp32 sum, bit-exact with the same order on the host
    f = [rng.standard_normal(1000).astype(np.float32) for _ in range(world)]
    for r in range(world):
        heap.view(h, r, np.float32, (1000,)).copy_(torch.from_numpy(f[r]))
    want = f[0].copy()
    for r in range(1, world):
        want = want + f[r]
    got = heap.multimem_ld_reduce(h, 0, np.float32, 1000, pe=0)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy(), want)
    # bf16 block reduce
    shape = (16, 24)
    bl = [torch.randn(shape).to(torch.bfloat16) for _ in range(world)]
    for r in range(world):
        heap.view(h, r, torch.bfloat16, shape).copy_(bl[r])
    blk = heap.multimem_ld_reduce_block(h, 0, torch.bfloat16, shape, 2, 5, 3, 7)
    acc = bl[0].float()
    for r in range(1, world):
        acc = acc + bl[r].float()
    assert torch.equal(blk.cpu(), acc.to(torch.bfloat16)[2:7, 3:10])
    # broadcast (vector and block) lands in every PE's copy
    v = torch.arange(300, dtype=torch.float32)
    heap.multimem_st(h, 64, v, pe=world - 1)
    for r in range(world):
        assert torch.equal(heap.view(h, r, torch.float32, (316,))[16:].cpu(), v)
    b = torch.full((2, 3), 7, dtype=torch.int64)
    heap.multimem_st_block(h, 0, b, (8, 8), 5, 4)
    for r in range(world):
        assert torch.equal(heap.view(h, r, torch.int64, (8, 8))[5:7, 4:7].cpu(), b)
    with pytest.raises(ValueError):
        heap.multimem_ld_reduce(h, 0, np.int8, 4, pe=0)
    heap.team.close()


def test_atomic_cas_and_putmem_strided():
    import numpy as np
    import torch
    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200.shmem import SymmetricHeap
    world = 2
    heap = SymmetricHeap(build_topology(world, 1), data_bytes=1 << 20, signal_slots=64,
                         devices=devices_for(world))
    sig = heap.alloc_signals(4)
    assert heap.atomic_cas(sig, 1, 0, 7, pe=1) == 0       # swaps
    assert heap.atomic_cas(sig, 1, 0, 9, pe=1) == 7       # mismatch: unchanged
    assert heap.atomic_cas(sig, 1, 7, 11, pe=1) == 7
    assert int(heap.sig_view(sig, 1)[1]) == 11 and int(heap.sig_view(sig, 0)[1]) == 0
    h = heap.alloc(64 * 64 * 4)
    region = heap.view(h, 1, torch.float32, (64, 64))
    region.zero_()
    block = torch.arange(5 * 7, dtype=torch.float32, device="cuda").view(5, 7)
    heap.putmem_strided(heap.symm_at(h, 1), 3 * 64 * 4 + 2 * 4, block, 64 * 4)
    torch.cuda.synchronize()
    assert torch.equal(region[3:8, 2:9], block)
    assert float(region.sum()) == float(block.sum())
    heap.sync_all(0)
    heap.node_barrier(1)
    torch.cuda.synchronize()
    heap.team.close()


def test_wait_equality_and_fetch_add_old_value():
    """Reference semantics: wait() is all-of '== value' (shmem.py:223-224) and
    atomic_add returns the old value (shmem.py:184-194)."""
    h = _heap()
    sig = h.alloc_signals(2)
    assert h.atomic_add(sig, 0, 3, pe=1) == 0
    assert h.atomic_add(sig, 0, 4, pe=1) == 3
    assert h.atomic_add(sig, 0, 1, pe=1, fetch=False) is None
    torch.cuda.synchronize()
    assert h.sig_view(sig, 1).tolist() == [8, 0]
    h.wait(sig, 0, 1, pe=1, value=8)          # == passes
    h.wait(sig, 0, 1, pe=1, value=5, cmp="ge")  # >= passes
    h.wait(sig, 1, 1, pe=1, value=0)          # == 0 passes on a fresh slot
    torch.cuda.synchronize()
    h.team.check()
    with pytest.raises(ValueError):
        h.wait(sig, 0, 1, pe=1, value=8, cmp="gt")
