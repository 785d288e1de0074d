"""ctypes binding of libtilefuse.so (the C ABI declared in include/tilefuse.h).

There is deliberately no fallback: if the library is missing or fails to load,
every operator raises.  Build it with `python -m paper_2605_02953_b200._build`
(or __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes as C
import pathlib
import re

from .errors import STATUS_EXC

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libtilefuse.so"
HEADER = pathlib.Path(__file__).resolve().parent.parent / "include" / "tilefuse.h"

TF_DTYPE_BF16, TF_DTYPE_F32 = 0, 1
TF_REDUCE_RING, TF_REDUCE_ASCENDING = 0, 1
PHASE_PRE, PHASE_MAIN, PHASE_POST, PHASE_FINAL = 1, 2, 4, 8  # FINAL: gemm_ar two-shot gather
PHASE_ALL = 15
MAX_WORLD = 16

vp = C.c_void_p
i32, i64, u64, sz = C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
ci = C.c_int


class GemmArgs(C.Structure):
    _fields_ = [
        ("a", vp), ("b", vp), ("c", vp),
        ("m", i64), ("n", i64), ("k", i64), ("lda", i64), ("ldb", i64), ("ldc", i64),
        ("out_dtype", i32), ("block_m", i32), ("block_n", i32), ("block_k", i32),
        ("group_m", i32), ("num_gemm_sms", i32), ("num_comm_sms", i32), ("swizzle", i32),
        ("fuse_scatter", i32), ("reduce_order", i32), ("tile_map", vp),
        ("nnodes", i32), ("ring_links", i32),
    ]


class MoeArgs(C.Structure):
    _fields_ = [
        ("tokens", i64), ("hidden", i64), ("k", i32), ("n_experts", i32), ("max_recv", i64),
        ("x", vp), ("topk_idx", vp), ("topk_w", vp), ("out", vp), ("counts", vp),
        ("sorted_pos", vp), ("dest_row", vp), ("recv_rows", vp), ("logits", vp),
    ]


class AttnArgs(C.Structure):
    _fields_ = [
        ("q", vp), ("k", vp), ("scores", vp), ("s_local", i64), ("hq", i64), ("hkv", i64),
        ("d", i64), ("out_dtype", i32), ("block_m", i32), ("block_n", i32), ("group_m", i32),
        ("num_gemm_sms", i32), ("swizzle", i32), ("key_tile_map", vp),
    ]


class AttnFwdArgs(C.Structure):
    _fields_ = [
        ("q", vp), ("k", vp), ("v", vp), ("out", vp), ("s_local", i64), ("hq", i64),
        ("hkv", i64), ("d", i64), ("scale", C.c_float),
    ]


class AgMoeArgs(C.Structure):
    _fields_ = [
        ("tokens", vp), ("weights", vp), ("out", vp), ("routing", vp),
        ("n_experts", i64), ("n", i64), ("k", i64), ("max_rows", i64), ("lda", i64), ("ldo", i64),
        ("out_dtype", i32), ("block_m", i32), ("block_n", i32), ("num_gemm_sms", i32),
        ("num_comm_sms", i32), ("swizzle", i32),
    ]


_SIGS = {
    "tf_last_error": (C.c_char_p, []),
    "tf_version": (C.c_char_p, []),
    "tf_tile_map": (ci, [i64, ci, ci, ci, ci, ci, C.POINTER(i32), i64]),
    "tf_swizzle_2d": (ci, [i64, i64, i64, ci, C.POINTER(i64), C.POINTER(i64)]),
    "tf_moe_schedule": (ci, [C.POINTER(i64), ci, ci, ci, ci, ci, C.POINTER(i64), vp, vp, vp, vp, vp]),
    "tf_team_create_local": (ci, [ci, C.POINTER(ci), sz, sz, C.POINTER(vp)]),
    "tf_team_create_ipc": (ci, [ci, ci, ci, sz, sz, C.POINTER(vp)]),
    "tf_team_export_handle": (ci, [vp, vp, sz]),
    "tf_team_open_peers": (ci, [vp, vp, sz]),
    "tf_team_destroy": (ci, [vp]),
    "tf_team_world": (ci, [vp, C.POINTER(ci)]),
    "tf_team_device": (ci, [vp, ci, C.POINTER(ci)]),
    "tf_team_check": (ci, [vp]),
    "tf_heap_alloc": (ci, [vp, sz, sz, C.POINTER(u64)]),
    "tf_signal_alloc": (ci, [vp, sz, C.POINTER(u64)]),
    "tf_heap_ptr": (ci, [vp, ci, u64, C.POINTER(vp)]),
    "tf_signal_ptr": (ci, [vp, ci, u64, C.POINTER(vp)]),
    "tf_signal_read": (ci, [vp, ci, u64, sz, C.POINTER(u64)]),
    "tf_signal_reset": (ci, [vp, ci, u64, sz, vp]),
    "tf_putmem": (ci, [vp, ci, u64, vp, sz, vp]),
    "tf_getmem": (ci, [vp, ci, u64, vp, sz, vp]),
    "tf_putmem_signal": (ci, [vp, ci, u64, vp, sz, u64, u64, ci, vp]),
    "tf_signal_op": (ci, [vp, ci, u64, u64, ci, vp]),
    "tf_team_reduce": (ci, [vp, ci, u64, ci, i64, vp, vp]),
    "tf_signal_cas": (ci, [vp, ci, u64, u64, u64, C.POINTER(u64), vp]),
    "tf_putmem_strided": (ci, [vp, ci, u64, sz, vp, sz, sz, sz, vp]),
    "tf_team_broadcast": (ci, [vp, ci, u64, vp, sz, vp]),
    "tf_signal_wait": (ci, [vp, ci, u64, sz, u64, vp]),
    "tf_signal_wait_cmp": (ci, [vp, ci, u64, sz, u64, ci, vp]),
    "tf_split_f32_bf16x3": (ci, [vp, i64, i64, i64, vp, i64, ci, vp]),
    "tf_signal_fetch_add": (ci, [vp, ci, u64, u64, C.POINTER(u64), vp]),
    "tf_barrier_arrive": (ci, [vp, ci, vp]),
    "tf_barrier_wait": (ci, [vp, ci, vp]),
    "tf_barrier_all": (ci, [vp, ci, vp]),
    "tf_gemm": (ci, [C.POINTER(GemmArgs), vp]),
    "tf_ag_gemm": (ci, [vp, ci, C.POINTER(GemmArgs), ci, vp, vp]),
    "tf_gemm_rs": (ci, [vp, ci, C.POINTER(GemmArgs), ci, vp, vp]),
    "tf_ag_kv_scores": (ci, [vp, ci, C.POINTER(AttnArgs), ci, vp, vp]),
    "tf_gemm_ar": (ci, [vp, ci, C.POINTER(GemmArgs), ci, ci, vp, vp]),
    "tf_ag_kv_attention": (ci, [vp, ci, C.POINTER(AttnFwdArgs), ci, vp, vp]),
    "tf_megakernel_run": (ci, [vp, vp, vp]),
    "tf_layer_megakernel_run": (ci, [vp, ci, vp, vp]),
    "tf_trace_enable": (ci, [ci, i64]),
    "tf_trace_disable": (ci, [ci]),
    "tf_trace_read": (ci, [ci, vp, i64, C.POINTER(i64)]),
    "tf_sm_die_map": (ci, [ci, vp, ci, C.POINTER(ci)]),
    "tf_moe_topk": (ci, [vp, i64, ci, ci, vp, vp, vp]),
    "tf_moe_count_scratch_bytes": (i64, [i64, ci]),
    "tf_moe_count": (ci, [vp, i64, ci, ci, vp, vp, vp, vp]),
    "tf_moe_buffers": (ci, [vp, ci, C.POINTER(MoeArgs), C.POINTER(vp), C.POINTER(vp)]),
    "tf_moe_dispatch": (ci, [vp, ci, C.POINTER(MoeArgs), ci, vp]),
    "tf_moe_combine": (ci, [vp, ci, C.POINTER(MoeArgs), ci, vp]),
    "tf_ag_moe_group_gemm": (ci, [vp, ci, C.POINTER(AgMoeArgs), ci, vp]),
    "tf_nvls_supported": (ci, [ci, C.POINTER(ci)]),
    "tf_team_nvls_create": (ci, [vp, sz, C.POINTER(ci)]),
    "tf_team_nvls_import": (ci, [vp, sz, ci]),
    "tf_team_nvls_add_device": (ci, [vp]),
    "tf_team_nvls_bind": (ci, [vp]),
    "tf_nvls_enabled": (ci, [vp, C.POINTER(ci), C.POINTER(sz)]),
    "tf_nvls_alloc": (ci, [vp, sz, sz, C.POINTER(u64)]),
    "tf_nvls_ptr": (ci, [vp, ci, u64, C.POINTER(vp), C.POINTER(vp)]),
    "tf_nvls_reduce": (ci, [vp, ci, u64, ci, i64, vp, vp]),
    "tf_nvls_broadcast": (ci, [vp, ci, u64, vp, sz, vp]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(tf_\w+)\s*\(", text, re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"libtilefuse.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2605_02953_b200._build` (there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().tf_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        exc = STATUS_EXC.get(rc, RuntimeError)
        raise exc(f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
