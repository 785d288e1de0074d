"""CPU tests of the C-ABI library: it loads, exports every symbol the public
header declares, and its host-side tile tables equal the reference fixtures."""

import ctypes as C
import os

import numpy as np
import pytest

from paper_2605_02953_b200 import _lib
from tests import _golden as G


def test_library_exports_header_symbols():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib._SIGS), "every header symbol must have a ctypes signature"


def test_version_string():
    assert b"sm_100a" in _lib.lib().tf_version()


def _cmap(m, w, nn, blk, r, mode):
    tiles = (m + blk - 1) // blk
    buf = (C.c_int32 * tiles)()
    _lib.call("tf_tile_map", m, r, w, nn, blk, 0 if mode == "ag_gemm" else 1, buf, tiles)
    return np.frombuffer(bytes(buf), dtype=np.int32).astype(np.int64)


def test_c_tile_maps_match_reference_fixtures():
    for (m, w, nn, blk, r, mode), want in G.tile_maps():
        assert np.array_equal(_cmap(m, w, nn, blk, r, mode), want), (m, w, nn, blk, r, mode)


def test_c_swizzle_2d_known_answers():
    pm, pn = C.c_int64(), C.c_int64()
    _lib.call("tf_swizzle_2d", 5, 4, 4, 2, C.byref(pm), C.byref(pn))
    assert (pm.value, pn.value) == (1, 2)
    for tm, tn, g in [(4, 4, 2), (5, 3, 2), (7, 2, 3), (64, 14, 8)]:
        seen = set()
        for p in range(tm * tn):
            _lib.call("tf_swizzle_2d", p, tm, tn, g, C.byref(pm), C.byref(pn))
            seen.add((pm.value, pn.value))
        assert len(seen) == tm * tn
    with pytest.raises(ValueError):
        _lib.call("tf_swizzle_2d", 16, 4, 4, 2, C.byref(pm), C.byref(pn))


def _cmoe(routing, rank, tp, block):
    routing = np.ascontiguousarray(routing, dtype=np.int64)
    w, e = routing.shape
    nt = C.c_int64()
    cp = routing.ctypes.data_as(C.POINTER(C.c_int64))
    _lib.call("tf_moe_schedule", cp, w, e, rank, tp, block, C.byref(nt), None, None, None, None, None)
    n = nt.value
    arrs = [np.zeros(max(n, 1), np.int64) for _ in range(5)]
    ptrs = [a.ctypes.data for a in arrs]
    _lib.call("tf_moe_schedule", cp, w, e, rank, tp, block, C.byref(nt), *ptrs)
    eid, tiled, s0, s1, st = (a[:n] for a in arrs)
    return np.stack([eid, tiled, s0, s1, st], axis=1) if n else np.zeros((0, 5), np.int64)


def test_c_moe_schedule_matches_reference_fixtures():
    for c in G.moe_cases():
        assert np.array_equal(_cmoe(c["routing"], c["rank"], c["tp"], c["block"]), c["sched"])


def test_c_tile_map_validation_errors():
    buf = (C.c_int32 * 8)()
    with pytest.raises(ValueError):
        _lib.call("tf_tile_map", 10, 0, 4, 1, 2, 0, buf, 8)   # M not divisible by world
    with pytest.raises(ValueError):
        _lib.call("tf_tile_map", 8, 0, 4, 3, 2, 0, buf, 8)    # world % nnodes
    with pytest.raises(ValueError):
        _lib.call("tf_tile_map", 8, 4, 4, 1, 2, 0, buf, 8)    # rank out of range


def test_sass_has_blackwell_and_multimem_instructions():
    """The built library carries tcgen05 MMAs, TMA, and the NVLS multimem loads
    (LDGMC = multimem.ld_reduce; multimem.st lowers to a STG.*.STRONG.SYS on the
    multicast address, so it has no mnemonic of its own)."""
    import shutil
    import subprocess
    from paper_2605_02953_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for op in ("UTCHMMA", "UTMALDG", "LDGMC.E.HPADD.BF16", "LDGMC.E.ADD.F32"):
        assert op in sass, op
