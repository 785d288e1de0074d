"""world_size-2 gloo tests of the multi-process (torchrun) host logic, on CPU.

The N>1 path is one process per GPU.  Its host side -- IPC handle exchange,
per-rank tile tables that must agree across ranks, max-over-ranks timing and
rank-0-only reporting -- is exercised here with the gloo backend; the device
side is covered by the GPU tests (several ranks emulated on one GPU).
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        from oracle import swizzle as S
        from paper_2605_02953_b200.kernels import tile_map_host
        from paper_2605_02953_b200.shmem import HANDLE_BLOB, exchange_handles
        # 1) handle exchange: rank-ordered concatenation of fixed-size blobs
        blob = bytes([rank + 1]) * HANDLE_BLOB
        allb = exchange_handles(blob)
        ok_blob = allb == b"".join(bytes([r + 1]) * HANDLE_BLOB for r in range(world))
        # 2) per-rank tile tables (C library, host) agree with the oracle and form
        #    the collective structure: gather step 0 = own chunk, scatter step 0 = successor
        m, bm = 8192, 256
        ag = tile_map_host(m, rank, world, 1, bm, "ag_gemm")
        rs = tile_map_host(m, rank, world, 1, bm, "gemm_rs")
        ok_maps = (np.array_equal(ag, S.tile_map(m, rank, world, 1, bm, "ag_gemm"))
                   and np.array_equal(rs, S.tile_map(m, rank, world, 1, bm, "gemm_rs")))
        firsts = [None] * world
        dist.all_gather_object(firsts, (int(ag[0]), int(rs[0])))
        mpr = m // world
        ok_first = all(f[0] * bm == r * mpr and f[1] * bm == ((r + 1) % world) * mpr
                       for r, f in enumerate(firsts))
        # 3) max-over-ranks timing reduction used by bench.py
        t = torch.tensor([1.0 + rank, 5.0 - rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok_max = t.tolist() == [float(world), 5.0]
        # 4) the TP=world layer megakernel program (one launch per rank): every rank
        #    builds byte-identical task queues, dependency rows and device tables,
        #    and the two-shot allreduce tiles are split evenly by owner
        import hashlib

        from paper_2605_02953_b200 import build_topology
        from paper_2605_02953_b200 import layer as L
        from paper_2605_02953_b200 import megakernel as MK
        prog = L.llama_layer_program(build_topology(world, 1), 1024, 1024, 8, 2, 2048, seq_len=512)
        built = prog.build()
        qs, cs = MK.encode_work_queues(built.tasks, 16)
        cfg, specs = L.layer_tables(prog, built)
        h = hashlib.sha256(MK.queues_to_bytes(qs) + MK.deps_to_bytes(built.dep_table) + cfg.tobytes()
                           + specs.tobytes()).hexdigest()
        hs = [None] * world
        dist.all_gather_object(hs, h)
        owners = [t.tile_id % world for t in built.tasks if built.layer_ops[t.layer_id] == "allreduce_residual"]
        ok_layer = len(set(hs)) == 1 and all(owners.count(o) == owners.count(0) for o in range(world))
        q.put((rank, ok_blob, ok_maps, ok_first, ok_max, ok_layer))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    for rank, *oks in res:
        assert all(oks), (rank, oks)


def test_reference_arm_rank_gating():
    """--impl reference under torchrun: rank 0 prints one JSON line, others exit 0 silently."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1", OPENBLAS_NUM_THREADS="2")
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                         "--gpus", "2", "--steps", "1", "--warmup", "0"],
                        capture_output=True, text=True, env=env, timeout=300)
    assert r1.returncode == 0 and r1.stdout.strip() == ""
    env.update(RANK="0", LOCAL_RANK="0")
    r0 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                         "--gpus", "2", "--steps", "1", "--warmup", "0"],
                        capture_output=True, text=True, env=env, timeout=300)
    assert r0.returncode == 0, r0.stderr
    line = json.loads(r0.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "TFLOP/s"
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["e2e"]["h2d_bytes_per_step"] == 0


def _fd_worker(rank, world, port, q):
    """share_fd (the NVLS handle transport): rank 0's pipe read end reaches every
    rank over SCM_RIGHTS, and each rank reads rank 0's bytes through its copy."""
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_02953_b200.shmem import share_fd
        r_fd = w_fd = None
        if rank == 0:
            r_fd, w_fd = os.pipe()
            os.write(w_fd, b"x" * (world - 1))
        got = share_fd(r_fd)
        ok = True
        if rank != 0:
            ok = os.read(got, 1) == b"x" and got != r_fd
            os.close(got)
        dist.barrier()
        if rank == 0:
            os.close(r_fd)
            os.close(w_fd)
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_over_unix_socket(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_fd_worker, args=(world, port, q), nprocs=world, join=True, start_method="spawn")
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(ok for _, ok in res), res
