"""GPU tests of the symmetric-heap primitives, mirroring the reference's
tests/test_shmem.py semantics (alloc symmetry, put-then-signal visibility,
all-of wait, atomics, barrier_all, views) on real device memory.  Several PEs
share cuda:0 (single-device team)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _heap(world=4, data=1 << 20, slots=256):
    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200.shmem import SymmetricHeap
    return SymmetricHeap(build_topology(world, 1), data_bytes=data, signal_slots=slots,
                         devices=[0] * world)


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
