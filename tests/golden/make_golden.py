"""Regenerate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `overlapsim` read-only from /root/reference/pkg/src and writes small
fixtures next to this file.  The GPU box never runs this script; the tests only
read the committed outputs.

Fixtures
  swizzle_maps.txt   reference render_swizzle_map output (tests/test_goldens.py:30-41)
  tile_maps.npz      ag_gemm_tile_map / gemm_rs_tile_map over the reference's
                     validation matrix (tests/test_swizzle.py:20-22) plus the
                     BASELINE shapes (M=8192, BM=128/256, world 1..8)
  moe_sched.npz      swizzle_ag_moe for the 25 random routings of
                     tests/test_swizzle.py:198-213 and the 60-expert case (:216-231)
  workloads.npz      exact-mode (int64) inputs/outputs of the reference simulated
                     ag_gemm, gemm_rs (4 variants), gemm_allreduce, ag_moe_group_gemm
                     for SHAPES x WORLDS of tests/test_kernels.py:18-21
  config1.npz        BASELINE config 1 (AG+GEMM, world=2, M=N=K=1024) in exact
                     mode: int8 inputs + sha256/row/col checksums of the reference
                     simulated ag_gemm outputs
"""

from __future__ import annotations

import hashlib
import json
import pathlib
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = pathlib.Path(__file__).resolve().parent


def _import_ref():
    sys.path.insert(0, REF_SRC)
    import overlapsim  # noqa: F401
    from overlapsim import kernels, swizzle, topology
    return kernels, swizzle, topology


def make_render(swz):
    perfect = swz.SwizzleParams(m=16, n=8, k=8, block_size_m=2, block_size_n=2,
                                block_size_k=2, group_size_m=1, rank=0, world_size=4)
    imperfect = swz.SwizzleParams(m=4 * 997, n=256, k=64, block_size_m=256,
                                  block_size_n=256, block_size_k=64, group_size_m=4,
                                  rank=0, world_size=4, nnodes=2)
    text = "\n\n".join([
        swz.render_swizzle_map(perfect, "gemm_rs"),
        swz.render_swizzle_map(perfect, "ag_gemm"),
        swz.render_swizzle_map(imperfect, "gemm_rs"),
        swz.render_swizzle_map(imperfect, "ag_gemm"),
    ]) + "\n"
    (OUT / "swizzle_maps.txt").write_text(text)


def make_tile_maps(swz):
    cases = []
    for w in (1, 2, 4, 8, 16, 32):
        for nn in (1, 2, 4):
            if w % nn:
                continue
            for mpr in (256, 997, 1024):
                for blk in (64, 256):
                    cases.append((w * mpr, w, nn, blk))
    for w in (1, 2, 4, 8):
        for blk in (128, 256):
            cases.append((8192, w, 1, blk))
    # small shapes used by the GPU parity tests (tests/test_kernels.py:18-21 style)
    for w in (1, 2, 4, 8):
        for mpr in (4, 5, 6, 128, 200, 512):
            for blk in (2, 4, 128):
                cases.append((w * mpr, w, 1, blk))
    meta, flat = [], []
    for m, w, nn, blk in cases:
        for r in range(w):
            for mode, fn in (("ag_gemm", swz.ag_gemm_tile_map), ("gemm_rs", swz.gemm_rs_tile_map)):
                mp = fn(m, r, w, nn, blk).astype(np.int32)
                meta.append((m, w, nn, blk, r, 0 if mode == "ag_gemm" else 1, len(flat), mp.size))
                flat.extend(mp.tolist())
    np.savez_compressed(OUT / "tile_maps.npz", meta=np.asarray(meta, dtype=np.int64),
                        maps=np.asarray(flat, dtype=np.int32))
    return len(meta)


def _moe_case_arrays(swz, routing, rank, tp, block):
    s = swz.swizzle_ag_moe(routing, rank, routing.shape[1], tp, tp, block)
    return np.stack([s.expert_id, s.tiled_m, s.segment_start, s.segment_end, s.stage],
                    axis=1).astype(np.int64) if s.ntiles else np.zeros((0, 5), np.int64)


def make_moe(swz):
    rng = np.random.default_rng(17)
    routings, meta, rows = [], [], []
    for _ in range(25):
        tp = int(rng.choice([1, 2, 4, 8]))
        experts = int(rng.integers(1, 7))
        block = int(rng.choice([1, 2, 3, 8]))
        routing = rng.integers(0, 9, size=(tp, experts))
        rank = int(rng.integers(0, tp))
        routings.append(routing)
        meta.append((tp, experts, block, rank))
    rng = np.random.default_rng(42)
    tp, experts, topk, tpr = 8, 60, 4, 1024
    routing = np.zeros((tp, experts), dtype=np.int64)
    for r in range(tp):
        for _ in range(tpr):
            for e in rng.choice(experts, size=topk, replace=False):
                routing[r, e] += 1
    for rank in range(tp):
        routings.append(routing)
        meta.append((tp, experts, 128, rank))
    out = {}
    for i, ((tp, experts, block, rank), routing) in enumerate(zip(meta, routings)):
        out[f"routing_{i}"] = np.asarray(routing, dtype=np.int64)
        out[f"sched_{i}"] = _moe_case_arrays(swz, np.asarray(routing), rank, tp, block)
    out["meta"] = np.asarray(meta, dtype=np.int64)
    np.savez_compressed(OUT / "moe_sched.npz", **out)
    return len(meta)


WORLDS = (1, 2, 4, 8)
SHAPES = ((4, 8, 8), (6, 9, 5), (5, 7, 33))


def make_workloads(kern, topo_mod):
    rng = np.random.default_rng(20260101)
    out = {}
    idx = []

    def ctx(world, **kw):
        t = topo_mod.build_topology(world, 1, num_sms=8)
        args = dict(block_m=4, block_n=4, block_k=16, group_m=2, num_gemm_sms=2, num_comm_sms=2)
        args.update(kw)
        return kern.WorkloadContext(topology=t, **args)

    def ints(shape):
        return rng.integers(-8, 8, size=shape).astype(np.int64)

    case = 0
    for world in WORLDS:
        for mpr, n, k in SHAPES:
            a = [ints((mpr, k)) for _ in range(world)]
            b = [ints((n, k)) for _ in range(world)]
            run = kern.ag_gemm(a, b, ctx(world))
            out[f"ag_{case}_a"] = np.stack(a)
            out[f"ag_{case}_b"] = np.stack(b)
            out[f"ag_{case}_c"] = np.stack(run.outputs)
            m = mpr * world
            x = [ints((m, k)) for _ in range(world)]
            w = [ints((n, k)) for _ in range(world)]
            out[f"rs_{case}_x"] = np.stack(x)
            out[f"rs_{case}_w"] = np.stack(w)
            results = []
            for variant in ("ring", "ascending", "fused", "ring_links"):
                c = ctx(world, reduce_order="ascending" if variant == "ascending" else "ring",
                        fuse_scatter=variant == "fused")
                r = kern.gemm_rs(x, w, c, assume_full_mesh_links=variant != "ring_links")
                results.append(np.stack(r.outputs))
            for v in results[1:]:
                assert np.array_equal(v, results[0])
            out[f"rs_{case}_y"] = results[0]
            n_ar = n - n % 4 or 4
            b_ar = [bb[:n_ar] for bb in b]
            ar = kern.gemm_allreduce(a, b_ar, ctx(world), use_multimem_st=False)
            out[f"ar_{case}_y"] = ar.outputs[0]
            routing = rng.integers(0, 5, size=(world, 3)).astype(np.int64)
            toks = [ints((int(routing[r].sum()), k)) for r in range(world)]
            wts = [[ints((n, k)) for _ in range(3)] for _ in range(world)]
            moe = kern.ag_moe_group_gemm(toks, wts, routing, ctx(world, block_m=2))
            out[f"moe_{case}_routing"] = routing
            out[f"moe_{case}_tok"] = np.concatenate(toks) if toks else np.zeros((0, k), np.int64)
            out[f"moe_{case}_w"] = np.asarray(wts)
            out[f"moe_{case}_y"] = np.stack(moe.outputs)
            idx.append((case, world, mpr, n, k))
            case += 1
    out["index"] = np.asarray(idx, dtype=np.int64)
    np.savez_compressed(OUT / "workloads.npz", **out)
    return case


def make_config1(kern, topo_mod):
    rng = np.random.default_rng(1)
    world, m, n, k = 2, 1024, 1024, 1024
    a = [rng.integers(-8, 8, size=(m // world, k)).astype(np.int64) for _ in range(world)]
    b = [rng.integers(-8, 8, size=(n // world, k)).astype(np.int64) for _ in range(world)]
    t = topo_mod.build_topology(world, 1, num_sms=8)
    ctx = kern.WorkloadContext(topology=t, block_m=128, block_n=128, block_k=64, group_m=4,
                               num_gemm_sms=4, num_comm_sms=1)
    run = kern.ag_gemm(a, b, ctx)
    digests = [hashlib.sha256(np.ascontiguousarray(o, dtype=np.int64).tobytes()).hexdigest()
               for o in run.outputs]
    np.savez_compressed(
        OUT / "config1.npz",
        a=np.stack(a).astype(np.int8), b=np.stack(b).astype(np.int8),
        row_sums=np.stack([o.sum(axis=1) for o in run.outputs]),
        col_sums=np.stack([o.sum(axis=0) for o in run.outputs]),
        corner=np.stack([o[:8, :8] for o in run.outputs]))
    (OUT / "config1_sha256.json").write_text(json.dumps(
        {"world": world, "m": m, "n": n, "k": k, "dtype": "int64",
         "sha256_per_rank": digests}, indent=1) + "\n")


def make_megakernel(topo_mod):
    """Reference task graphs: queue bytes, dependency tables and DAG text."""
    from overlapsim.megakernel import (MegaProgram, dump_task_graph, encode_work_queues,
                                       queues_to_bytes, deps_to_bytes)
    out, texts = {}, {}
    progs = {}
    # the MLP of tests/test_megakernel.py:48-61 and the allreduce graph of :374-384
    topo = topo_mod.build_topology(2, 1, num_sms=8)
    prog = MegaProgram(topo)
    x = prog.tensor("x", (32, 16), np.int64)
    w1 = prog.tensor("w1", (24, 16), np.int64)
    h1 = prog.tensor("h1", (32, 24), np.int64)
    bias = prog.tensor("bias", (32, 24), np.int64)
    h2 = prog.tensor("h2", (32, 24), np.int64)
    w2 = prog.tensor("w2", (16, 24), np.int64)
    y = prog.tensor("y", (32, 16), np.int64)
    prog.layer("linear", [x, w1], [h1], block_m=16, block_n=16)
    prog.layer("add", [h1, bias], [h2], block_rows=16)
    prog.layer("linear", [h2, w2], [y], block_m=16, block_n=16)
    progs["mlp"] = prog
    topo = topo_mod.build_topology(4, 1, num_sms=4)
    prog = MegaProgram(topo)
    a = prog.tensor("a", (8, 6), np.int64)
    w = prog.tensor("w", (6, 6), np.int64)
    pp = prog.tensor("p", (8, 6), np.int64)
    red = prog.tensor("red", (8, 6), np.int64)
    prog.layer("linear", [a, w], [pp], block_m=4, block_n=3)
    prog.layer("allreduce", [pp], [red], block_rows=4)
    progs["allreduce"] = prog
    for name, prog in progs.items():
        built = prog.build()
        for nsm in (1, 3, 8):
            q, c = encode_work_queues(built.tasks, nsm)
            out[f"{name}_q{nsm}"] = np.frombuffer(queues_to_bytes(q), dtype=np.uint8)
            out[f"{name}_c{nsm}"] = c
        out[f"{name}_deps"] = np.frombuffer(deps_to_bytes(built.dep_table), dtype=np.uint8)
        out[f"{name}_meta"] = np.array([built.max_task_id, built.max_tiles_per_op], np.int64)
        texts[name] = dump_task_graph(built.tasks, built.dep_table)
    np.savez_compressed(OUT / "megakernel.npz", **out)
    (OUT / "megakernel_dags.json").write_text(json.dumps(texts, indent=1) + "\n")


def main():
    kern, swz, topo_mod = _import_ref()
    make_megakernel(topo_mod)
    make_render(swz)
    nmaps = make_tile_maps(swz)
    nmoe = make_moe(swz)
    nwl = make_workloads(kern, topo_mod)
    make_config1(kern, topo_mod)
    print(f"wrote {nmaps} tile maps, {nmoe} moe schedules, {nwl} workload cases to {OUT}")


if __name__ == "__main__":
    main()
