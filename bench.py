"""Benchmark of the fused-collective hot path (BASELINE.json config 2).

One step = one tensor-parallel Llama-3-70B MLP pass through the fused ops:
    h_r = AllGather+GEMM(x_r, W1_r)      x_r [8192/TP, 8192], W1_r [28672/TP, 8192]
    y_r = GEMM+ReduceScatter(h_r, W2_r)  h_r [8192, 28672/TP], W2_r [8192, 28672/TP]
bf16 inputs, fp32 accumulation, bf16 outputs; TP = number of GPUs (one process
per GPU under torchrun, IPC symmetric heap).  At N=1 both ops degenerate to the
local GEMM (no exchange), which is what the round-end 1-GPU bench measures.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement): value = total
TFLOP/s over all ranks (max-over-ranks device time), roofline of the dominant
kernel (the tcgen05 GEMM) against MEASURED_PEAKS.json, e2e through the public
API with pinned host buffers, cuBLAS comparator, clocks sampled during the timed
region, and the CPU baseline (the numpy oracle on a bounded sample).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AG-GEMM/GEMM-RS TFLOPS at 1/2/4/8 B200 vs roofline; MoE a2a GB/s"
TOKENS, HIDDEN, FFN = 8192, 8192, 28672
# NVLink roofline: north_star's "link bandwidth" = NVLink 5 nominal 900 GB/s per direction;
# the measured peer copy (B200_PROFILING.md) is reported beside it
NVLINK_GBS, NVLINK_MEASURED_GBS = 900.0, 770.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--group-m", type=int, default=int(os.environ.get("TF_GROUP_M", "8")))
    p.add_argument("--no-moe", action="store_true")
    p.add_argument("--no-attn", action="store_true")
    p.add_argument("--no-layer", action="store_true")
    p.add_argument("--only-layer", action="store_true")
    p.add_argument("--only-attn", action="store_true")
    p.add_argument("--only-agmoe", action="store_true")
    p.add_argument("--only-moe", action="store_true")
    return p.parse_args()


def _committed_traffic():
    """DRAM bytes per launch of the GEMM kernel from the committed ncu --set full
    capture (profiles/gemm_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"dram_bytes_per_launch": d["dram_bytes_per_launch"],
                "algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"], "source": d["source"]}
    except (OSError, KeyError, ValueError):
        return None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def wait_first(self, timeout=3.0):
        """Block until nvidia-smi has produced a sample (its start-up takes ~0.3 s)."""
        t_end = time.time() + timeout
        while self.proc is not None and not self.lines and time.time() < t_end:
            time.sleep(0.01)

    def stop(self, t0=None, t1=None):
        """Summarise the samples taken inside [t0, t1] (the timed region; the
        nearest later sample if none fell inside)."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        lines = [ln for ts, ln in self.lines if t0 is None or (t0 <= ts <= t1 + 0.05)]
        if not lines and t0 is not None:
            later = [ln for ts, ln in self.lines if ts >= t0]
            lines = later[:1]
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None,
                "sm_max_mhz": max(maxes) if maxes else None,
                "reasons": sorted(reasons), "samples": len(sms)}


# ------------------------------------------------------------------ CPU baseline / reference arm
CPU_ROWS = 1024  # the bounded sample both CPU legs use: 1024 of the 8192 tokens


def _ref_package():
    """The unmodified reference (overlapsim) installed in baseline/_ref, or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "overlapsim")) and path not in sys.path:
        sys.path.insert(0, path)
    try:
        import overlapsim  # noqa: F401
        return path
    except ImportError:
        return None


def cpu_sample(tp: int, rows: int = CPU_ROWS, steps: int = 1, min_seconds: float = 0.0):
    """One config-2 MLP step of the reference's CPU path on a bounded sample
    (`rows` tokens, TP=tp ranks simulated, hidden 8192, ffn 28672, fp32, all host
    threads).  With baseline/_ref installed this is the reference's own public
    operators -- overlapsim ag_gemm + gemm_rs (ovs/kernels/ag_gemm.py:20,
    gemm_rs.py:31) with block 128x256x64 and num_gemm_sms=144 --
    kind "reference"; otherwise the numpy oracle port, kind "port".  Returns a dict
    with TFLOP/s, seconds per step, cores, kind, sample text and the reference
    oracle (ref_allgather_gemm + ref_reduce_scatter) on the same sample."""
    import numpy as np

    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)
    f_tp = FFN // tp
    mpr = max(rows // tp, 1)
    x = [rng.standard_normal((mpr, HIDDEN), dtype=np.float32) for _ in range(tp)]
    w1 = [rng.standard_normal((f_tp, HIDDEN), dtype=np.float32) for _ in range(tp)]
    w2 = [rng.standard_normal((HIDDEN, f_tp), dtype=np.float32) for _ in range(tp)]
    flops = 2 * 2 * (mpr * tp) * HIDDEN * FFN
    if _ref_package():
        from overlapsim import build_topology
        from overlapsim.kernels.ag_gemm import ag_gemm
        from overlapsim.kernels.context import WorkloadContext
        from overlapsim.kernels.gemm_rs import gemm_rs
        from overlapsim.kernels.oracles import ref_allgather_gemm, ref_reduce_scatter
        topo = build_topology(tp, 1, num_sms=148)
        kw = dict(topology=topo, block_m=128, block_n=256, block_k=64, num_gemm_sms=144, num_comm_sms=4)
        ctx_ag, ctx_rs = WorkloadContext(**kw), WorkloadContext(fuse_scatter=True, **kw)

        def step():
            h = ag_gemm(x, w1, ctx_ag).outputs
            gemm_rs(h, w2, ctx_rs)
        kind = "reference"
        what = ("reference overlapsim ag_gemm + gemm_rs (baseline/_ref, unmodified; block 128x256x64, "
                "num_gemm_sms=144, fuse_scatter)")
    else:
        from oracle import collectives as O
        ref_allgather_gemm, ref_reduce_scatter = O.ref_allgather_gemm, O.ref_reduce_scatter

        def step():
            ref_reduce_scatter(ref_allgather_gemm(x, w1), w2)
        kind = "port"
        what = "oracle port of ref_allgather_gemm + ref_reduce_scatter (baseline/_ref not installed)"
    t0 = time.perf_counter()
    done = 0
    while done < steps or time.perf_counter() - t0 < min_seconds:
        step()
        done += 1
    dt = (time.perf_counter() - t0) / done
    t1 = time.perf_counter()
    ref_reduce_scatter(ref_allgather_gemm(x, w1), w2)
    dt_oracle = time.perf_counter() - t1
    sample = (f"{what}, numpy fp32 (OpenBLAS, {cores} threads) on {mpr * tp} of {TOKENS} tokens, "
              f"TP={tp} simulated ranks, hidden {HIDDEN}, ffn {FFN}")
    return {"value": flops / dt / 1e12, "seconds_per_step": dt, "cores": cores, "kind": kind,
            "sample": sample, "oracle_tflops": flops / dt_oracle / 1e12, "steps": done}


def cpu_sample_1thread(tp: int, rows: int = CPU_ROWS):
    """The same step with one host thread (OPENBLAS_NUM_THREADS=1 must be set
    before numpy loads, hence a subprocess)."""
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
    code = (f"import json,sys; sys.path.insert(0, {ROOT!r}); import bench; "
            f"print(json.dumps(bench.cpu_sample({tp}, {rows})))")
    try:
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                             timeout=600)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        return {"value": round(d["value"], 6), "seconds_per_step": round(d["seconds_per_step"], 3),
                "oracle_tflops": round(d["oracle_tflops"], 6), "cores": 1}
    except Exception as exc:  # noqa: BLE001
        return {"error": f"{type(exc).__name__}: {exc}"[:200]}


def run_reference(args):
    """--impl reference: the reference's own CPU path (baseline/_ref overlapsim
    ag_gemm + gemm_rs, else the oracle port) on the host cores, each step the
    bounded 1024-token sample of config 2 at TP = --gpus (the same sample as the
    GPU arm's cpu_baseline).  Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    tp = args.gpus
    runs = []
    for i in range(args.warmup + args.steps):
        d = cpu_sample(tp)
        if i >= args.warmup:
            runs.append(d)
    value = statistics.median(d["value"] for d in runs)
    ms = statistics.median(d["seconds_per_step"] for d in runs) * 1e3
    last = runs[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"llama3-70b MLP AG-GEMM+GEMM-RS, TP={tp}, sampled on {CPU_ROWS} tokens",
                   "tokens": TOKENS, "hidden": HIDDEN, "ffn": FFN, "tp": tp, "sample_tokens": CPU_ROWS},
        "cpu_baseline": {"value": round(value, 6), "unit": "TFLOP/s", "cores": last["cores"],
                         "kind": last["kind"], "sample": last["sample"],
                         "oracle_tflops": round(statistics.median(d["oracle_tflops"] for d in runs), 6)},
        "e2e": {"value": round(value, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_over_ranks(vals, dev, distributed):
    """Element-wise max over ranks (device tensor for NCCL, host tensor for gloo)."""
    import torch
    import torch.distributed as dist
    if not distributed:
        return [float(v) for v in vals]
    if dist.get_backend() == "nccl":
        t = torch.tensor(vals, dtype=torch.float64, device=f"cuda:{dev}")
    else:
        t = torch.tensor(vals, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


# ------------------------------------------------------------------ MoE EP (config 4)
MOE_E, MOE_K, MOE_H, MOE_T = 256, 8, 7168, 4096


def bench_moe(team, dev, world, rank, steps, warmup, flush, stream, distributed, peaks):
    """DeepSeek-V3-like EP dispatch + combine: 256 experts, top-8, hidden 7168,
    4096 tokens/rank, EP = number of GPUs.  Routing from N(0,1) logits through
    the device top-k; expert compute excluded (expert outputs = received rows)."""
    import torch
    import torch.distributed as dist

    from paper_2605_02953_b200 import moe as M
    g = torch.Generator(device="cpu").manual_seed(4321 + rank)
    x = torch.randn(MOE_T, MOE_H, generator=g).to(torch.bfloat16).to(f"cuda:{dev}")
    logits = torch.randn(MOE_T, MOE_E, generator=g).to(f"cuda:{dev}")
    ep = M.ExpertParallelMoE(team, MOE_E, MOE_H, MOE_K, max_tokens=MOE_T)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    with torch.cuda.stream(stream):
        for i in range(warmup + steps):
            if i >= warmup:
                flush.zero_()
                ev[i - warmup][0].record(stream)
            recv, idx, w = ep.route_dispatch(x, logits)  # top-k fused into the dispatch launch
            if i >= warmup:
                ev[i - warmup][1].record(stream)
            if i == 0:
                torch.cuda.synchronize()
                n = ep.recv_rows()
                ep.expert_out()[:n].copy_(recv[:n])
            ep.combine(idx, w)
            if i >= warmup:
                ev[i - warmup][2].record(stream)
        torch.cuda.synchronize()
        # the same dispatch with the routing given (ExpertParallelMoE.dispatch(x, topk_idx),
        # the reference's split of routing and dispatch): no top-k, no grid-wide barrier
        evg = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        idx_given = idx.clone()
        for i in range(warmup + steps):
            if i >= warmup:
                flush.zero_()
                evg[i - warmup][0].record(stream)
            ep.dispatch(x, idx_given)
            if i >= warmup:
                evg[i - warmup][1].record(stream)
        torch.cuda.synchronize()
    team.check()
    d_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    c_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    g_ms = sum(e[0].elapsed_time(e[1]) for e in evg) / steps
    d_ms, c_ms, g_ms = max_over_ranks([d_ms, c_ms, g_ms], dev, distributed)
    rows = MOE_T * MOE_K
    row_b = MOE_H * 2
    moved = rows * row_b  # token rows delivered by dispatch (and pulled back by combine), per rank
    remote = moved * (world - 1) / world
    hbm = (MOE_T * row_b + moved)  # per phase: unique x read + routed rows written (or the mirror)
    peak_hbm = peaks.get("hbm_gbs", 6550.1)
    out = {
        "workload": f"EP={world}: {MOE_E} experts, top-{MOE_K}, hidden {MOE_H}, {MOE_T} tokens/rank, "
                    "bf16, routing from N(0,1) logits (device top-k); expert compute excluded",
        "dispatch_ms": round(d_ms, 4), "combine_ms": round(c_ms, 4),
        "dispatch_given_routing_ms": round(g_ms, 4),
        "gbps": round(world * 2 * moved / ((d_ms + c_ms) * 1e-3) / 1e9, 2),
        "unit": "GB/s (routed token bytes moved by dispatch + combine, all ranks)",
        "nvlink_bytes_per_rank_per_phase": remote,
    }
    if world == 1:
        ach = 2 * hbm / ((d_ms + c_ms) * 1e-3) / 1e9
        out["roofline"] = {"bound": "hbm", "achieved": round(ach, 1), "peak": peak_hbm,
                           "unit": "GB/s", "frac": round(ach / peak_hbm, 4),
                           "bytes_per_phase": hbm}
    else:
        ach = remote / (max(d_ms, c_ms) * 1e-3) / 1e9
        out["roofline"] = {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_GBS,
                           "unit": "GB/s per rank per direction (NVLink 5 link bandwidth)",
                           "frac": round(ach / NVLINK_GBS, 4),
                           "frac_vs_measured_p2p": round(ach / NVLINK_MEASURED_GBS, 4)}
    return out


# ------------------------------------------------------------------ AG + grouped GEMM (ag_moe_group_gemm)
AGM_TP, AGM_N = 8, 512  # W13 of a DeepSeek-V3 expert (2 x 2048) sharded over TP=8: 512 columns per rank


def _agm_counts(rng_seed, ranks, dev):
    """[ranks, E] routed-row counts: top-8 of N(0,1) logits for MOE_T tokens per rank."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(rng_seed)
    out = []
    for _ in range(ranks):
        idx = torch.randn(MOE_T, MOE_E, generator=g).to(f"cuda:{dev}").topk(MOE_K, dim=1).indices
        out.append(torch.bincount(idx.flatten(), minlength=MOE_E).cpu().numpy())
    import numpy as np
    return np.stack(out).astype(np.int64)


def bench_ag_moe(dev, world, rank, steps, warmup, flush, stream, distributed, peaks):
    """The reference's MoE operator (ag_moe_group_gemm, ovs/kernels/ag_moe.py:20) with
    expert compute: DeepSeek-V3-like 256 experts, top-8, hidden 7168, 4096 tokens per
    source rank, W13 shard N=512 per rank (TP=8).  N=1: one rank's work of the TP=8
    job (all 8 sources' rows gathered: 262144 rows), no exchange; N>1: a real
    AllGather over the team with `world` sources.  Comparators: cuBLAS per-expert
    GEMMs (torch.matmul loop) and torch._grouped_mm on the same expert-major rows."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_02953_b200 import moe as M
    from paper_2605_02953_b200.shmem import Team
    if world == 1:
        routing = _agm_counts(777, AGM_TP, dev).sum(axis=0, keepdims=True)
    else:
        routing = _agm_counts(777, world, dev)
    total = int(routing.sum())
    rows_r = int(routing[rank].sum())
    k, n, E = MOE_H, AGM_N, MOE_E
    heap = M._agmoe_heap_bytes(total, k, E, world, 128)  # 128-row slots bound every block_m
    team = (Team.from_process_group(heap_bytes=heap, signal_slots=256) if distributed
            else Team(1, [dev], heap_bytes=heap, signal_slots=256))
    g = torch.Generator(device="cpu").manual_seed(99 + rank)
    tok = torch.empty(rows_r, k, dtype=torch.bfloat16, device=f"cuda:{dev}")
    for i in range(0, rows_r, 16384):  # generate in slices (host RAM)
        j = min(rows_r, i + 16384)
        tok[i:j] = torch.randn(j - i, k, generator=g).to(torch.bfloat16)
    wts = (torch.randn(E, n, k, generator=g) * k ** -0.5).to(torch.bfloat16).to(f"cuda:{dev}")
    out = torch.empty(total, n, dtype=torch.bfloat16, device=f"cuda:{dev}")
    bm = int(os.environ.get("TF_AGM_BM", "256"))  # CTA pair: 1.777 vs 1.796 ms for 128 (same box, after the relaxed arrives)
    op = M.AgMoeGroupGemm(team, E, n, k, total, block_m=bm, block_n=256, num_comm_sms=8)

    def timed(fn, n_steps, n_warm):
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n_steps)]
        with torch.cuda.stream(stream):
            for i in range(n_warm + n_steps):
                if i >= n_warm:
                    flush.zero_()
                    ev[i - n_warm][0].record(stream)
                fn()
                if i >= n_warm:
                    ev[i - n_warm][1].record(stream)
            torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / n_steps

    if distributed:
        dist.barrier()
    ms = timed(lambda: op(routing, tok, wts, out=out), steps, warmup)
    ms = max_over_ranks([ms], dev, distributed)[0]
    team.check()
    flops = 2.0 * total * n * k
    peak = peaks.get("bf16_tflops", 1590.0)
    hbm = peaks.get("hbm_gbs", 6550.1)
    bytes_ = total * k * 2 + E * n * k * 2 + total * n * 2
    t_tensor, t_hbm = flops / (peak * 1e12) * 1e3, bytes_ / (hbm * 1e9) * 1e3
    res = {
        "workload": (f"ag_moe_group_gemm: {E} experts, top-{MOE_K}, hidden {k}, {MOE_T} tokens per source "
                     f"rank, W13 shard N={n} (TP={AGM_TP}); " +
                     (f"one rank's work of the TP={AGM_TP} job ({total} gathered rows), no exchange"
                      if world == 1 else f"AllGather over {world} ranks ({total} gathered rows)")),
        "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 2), "block_m": bm,
        "roofline": {"bound": "tensor" if t_tensor >= t_hbm else "hbm",
                     "t_roof_ms": round(max(t_tensor, t_hbm), 4),
                     "frac": round(max(t_tensor, t_hbm) / ms, 4), "peak_tflops": peak,
                     "algorithmic_bytes": bytes_},
    }
    if world == 1 and rank == 0:
        ebase = np.concatenate([[0], np.cumsum(routing.sum(axis=0))])
        segs = [(int(ebase[e]), int(ebase[e + 1])) for e in range(E)]
        out2 = torch.empty_like(out)

        def per_expert():
            for e, (lo, hi) in enumerate(segs):
                if hi > lo:
                    torch.matmul(tok[lo:hi], wts[e].t(), out=out2[lo:hi])
        c_ms = timed(per_expert, max(3, steps // 2), 2)
        cmp_ = {"cublas_per_expert": {"ms": round(c_ms, 4), "speedup": round(c_ms / ms, 4)}}
        err = (out.float() - out2.float()).abs().max().item() / max(out2.float().abs().max().item(), 1e-30)
        cmp_["max_rel_err_vs_cublas"] = round(err, 5)
        try:
            offs = torch.tensor(ebase[1:], dtype=torch.int32, device=f"cuda:{dev}")
            wt = wts.transpose(1, 2)
            gm_ms = timed(lambda: torch._grouped_mm(tok, wt, offs=offs), max(3, steps // 2), 2)
            cmp_["torch_grouped_mm"] = {"ms": round(gm_ms, 4), "speedup": round(gm_ms / ms, 4)}
        except Exception as exc:  # noqa: BLE001
            cmp_["torch_grouped_mm"] = {"error": f"{type(exc).__name__}: {exc}"[:160]}
        res["comparator"] = cmp_
    team.close()
    del tok, wts, out
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ SP attention scores (config 3)
ATT_S, ATT_SP, ATT_HQ, ATT_HKV, ATT_D = 32768, 8, 64, 8, 128


def bench_attention(dev, steps, peaks):
    """Config 3 per SP rank: fused AG-KV flash-attention forward, Q [4096, 64, 128]
    against K/V gathered to [32768, 8, 128] (GQA 8:1, non-causal, bf16).  On one
    GPU the 8 SP ranks are emulated by a local team whose PEs share the device;
    their fused calls run back to back and the per-rank time is total / 8."""
    import ctypes as C

    import torch

    from paper_2605_02953_b200 import _lib
    from paper_2605_02953_b200.attention import _fwd_args
    from paper_2605_02953_b200.shmem import Team
    sl = ATT_S // ATT_SP
    g = torch.Generator(device="cpu").manual_seed(99)
    team = Team(ATT_SP, [dev] * ATT_SP, 4 * ATT_S * ATT_HKV * ATT_D * 2 + (16 << 20), 256)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).to(f"cuda:{dev}")
    qs = [mk(sl, ATT_HQ, ATT_D) for _ in range(ATT_SP)]
    ks = [mk(sl, ATT_HKV, ATT_D) for _ in range(ATT_SP)]
    vs = [mk(sl, ATT_HKV, ATT_D) for _ in range(ATT_SP)]
    outs = [torch.empty_like(q) for q in qs]
    args = [_fwd_args(qs[r], ks[r], vs[r], outs[r], sl, ATT_HQ, ATT_HKV, ATT_D, ATT_D ** -0.5)
            for r in range(ATT_SP)]
    stream = torch.cuda.current_stream(dev)

    def step():
        for phase in (_lib.PHASE_PRE, _lib.PHASE_MAIN, _lib.PHASE_POST):
            for r in range(ATT_SP):
                _lib.call("tf_ag_kv_attention", team.handle, r, C.byref(args[r]), phase,
                          stream.cuda_stream, None)

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    team.check()
    per_rank_ms = e0.elapsed_time(e1) / steps / ATT_SP
    flops = 4.0 * sl * ATT_S * ATT_D * ATT_HQ  # QK^T + PV
    t_tc = flops / (peaks.get("bf16_tflops", 1622.7) * 1e12)
    team.close()
    # library comparator on one rank's problem (K/V already gathered): torch SDPA, cuDNN backend
    comparator = None
    try:
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel
        qt = qs[0].transpose(0, 1).unsqueeze(0)
        kt = torch.cat(ks).transpose(0, 1).unsqueeze(0)
        vt = torch.cat(vs).transpose(0, 1).unsqueeze(0)
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            for _ in range(2):
                F.scaled_dot_product_attention(qt, kt, vt, enable_gqa=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                F.scaled_dot_product_attention(qt, kt, vt, enable_gqa=True)
            e1.record(stream)
            torch.cuda.synchronize()
        c_ms = e0.elapsed_time(e1) / steps
        comparator = {"impl": "torch SDPA, cuDNN backend, K/V pre-gathered (no AllGather)",
                      "ms": round(c_ms, 4), "speedup": round(c_ms / per_rank_ms, 4)}
    except Exception as e:  # noqa: BLE001
        comparator = {"impl": "torch SDPA (cuDNN)", "error": str(e).splitlines()[0][:160]}
    return {"comparator": comparator,
            "workload": "config 3 per SP rank: fused AG-KV flash-attention forward, Q[4096,64,128] vs "
                        "K/V[32768,8,128] (GQA 8:1, non-causal, bf16); SP=8 emulated on one GPU "
                        "(per-rank = total / 8)",
            "ms_per_rank": round(per_rank_ms, 4),
            "tflops_per_rank": round(flops / (per_rank_ms * 1e-3) / 1e12, 2),
            "roofline": {"bound": "tensor", "t_roof_ms": round(t_tc * 1e3, 4),
                         "frac": round(t_tc / (per_rank_ms * 1e-3), 4),
                         "peak": peaks.get("bf16_tflops", 1622.7), "unit": "TFLOP/s"}}


# ------------------------------------------------------------------ fused layer (config 5)
LAY_T, LAY_H, LAY_HQ, LAY_HKV, LAY_F = 8192, 8192, 64, 8, 28672


def layer_flops(tokens, hidden, hq, hkv, ffn, tp=1):
    """Algorithmic FLOPs of one Llama layer shard (causal attention counted at T^2/2)."""
    hq, hkv, f = hq // tp, hkv // tp, ffn // tp
    qkv = 2.0 * tokens * hidden * (hq + 2 * hkv) * 128
    att = 4.0 * tokens * tokens * 128 * hq / 2
    o = 2.0 * tokens * hq * 128 * hidden
    mlp = 2.0 * tokens * hidden * 2 * f + 2.0 * tokens * f * hidden
    return qkv + att + o + mlp


def bench_layer(dev, steps, warmup, peaks, flush, tp_emulated=1):
    """Config 5 on one GPU: the Llama-3-70B layer (8192 tokens, hidden 8192, 64/8
    heads, ffn 28672, one causal sequence) as ONE persistent megakernel launch
    (rmsnorm -> QKV+RoPE -> attention -> O -> allreduce+residual -> rmsnorm ->
    gate/up+SiLU -> down -> allreduce+residual).  TP=1 here (the allreduce tasks
    reduce a single partial); the unfused comparator is cuBLAS GEMMs + cuDNN/flash
    SDPA + torch elementwise on the same bf16 tensors."""
    import torch
    import torch.nn.functional as F

    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200 import layer as L
    T, H, HQ, HKV, FF = LAY_T, LAY_H, LAY_HQ, LAY_HKV, LAY_F
    prog = L.llama_layer_program(build_topology(1, 1), T, H, HQ, HKV, FF, seq_len=T)
    runner = L.LayerRunner(prog, device=dev)
    g = torch.Generator(device="cpu").manual_seed(55)
    mk = lambda *s, sc=1.0: (torch.randn(*s, generator=g) * sc).to(torch.bfloat16).to(f"cuda:{dev}")
    qkv_n = (HQ + 2 * HKV) * 128
    x = mk(T, H)
    w = {"w_qkv": mk(qkv_n, H, sc=H ** -0.5), "w_o": mk(H, HQ * 128, sc=(HQ * 128) ** -0.5),
         "w_gate_up": mk(2 * FF, H, sc=H ** -0.5), "w_down": mk(H, FF, sc=FF ** -0.5)}
    g1 = (1 + 0.1 * torch.randn(1, H, generator=g)).to(torch.bfloat16).to(f"cuda:{dev}")
    g2 = (1 + 0.1 * torch.randn(1, H, generator=g)).to(torch.bfloat16).to(f"cuda:{dev}")
    rope = torch.from_numpy(L.rope_table(T)).to(f"cuda:{dev}")
    for name, val in [("x", x), ("g_attn", g1), ("g_mlp", g2), ("rope", rope), *w.items()]:
        runner.view(name).copy_(val)
    stream = torch.cuda.current_stream(dev)
    flops = layer_flops(T, H, HQ, HKV, FF)

    # ---- unfused comparator on the same tensors (gate/up de-interleaved for torch)
    wgu = w["w_gate_up"].view(FF // 128, 2, 128, H)
    wg, wu = wgu[:, 0].reshape(FF, H).contiguous(), wgu[:, 1].reshape(FF, H).contiguous()
    cos = rope[:, :64].to(torch.float32)
    sin = rope[:, 64:].to(torch.float32)

    def rms(t, gg):
        tf = t.float()
        return (tf * torch.rsqrt(tf.pow(2).mean(-1, keepdim=True) + 1e-5) * gg.float()).to(torch.bfloat16)

    def rot(t):  # [T, heads, 128]
        tf = t.float()
        a1, a2 = tf[..., :64], tf[..., 64:]
        c, s_ = cos[:, None, :], sin[:, None, :]
        return torch.cat([a1 * c - a2 * s_, a2 * c + a1 * s_], -1).to(torch.bfloat16)

    def unfused():
        xn = rms(x, g1)
        qkv = xn @ w["w_qkv"].t()
        q = rot(qkv[:, :HQ * 128].view(T, HQ, 128))
        k = rot(qkv[:, HQ * 128:(HQ + HKV) * 128].view(T, HKV, 128))
        v = qkv[:, (HQ + HKV) * 128:].view(T, HKV, 128)
        att = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                             v.transpose(0, 1)[None], is_causal=True, enable_gqa=True)
        att = att[0].transpose(0, 1).reshape(T, HQ * 128)
        h = att @ w["w_o"].t() + x
        hn = rms(h, g2)
        act = F.silu(hn @ wg.t()) * (hn @ wu.t())
        return act @ w["w_down"].t() + h

    # warm both, then alternate fused / unfused steps so both see the same clocks and
    # temperature (the launch is energy-bound at the 1 kW cap); L2 flushed before each
    for _ in range(warmup):
        runner.run(stream)
        ref = unfused()
    torch.cuda.synchronize(dev)
    runner.check()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    cevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for (e0, e1), (c0, c1) in zip(evs, cevs):
        flush.zero_()
        e0.record(stream)
        runner.run(stream)
        e1.record(stream)
        flush.zero_()
        c0.record(stream)
        unfused()
        c1.record(stream)
    torch.cuda.synchronize(dev)
    runner.check()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    cms = sum(a.elapsed_time(b) for a, b in cevs) / steps
    out_fused = runner.view("out").clone()
    ref = unfused()
    torch.cuda.synchronize(dev)
    rel = float((out_fused.float() - ref.float()).abs().max() / ref.float().abs().max())
    n_tasks = len(runner.built.tasks)
    runner.close()
    del runner
    torch.cuda.empty_cache()

    # ---- the TP=8 graph of the same layer, all 8 ranks co-scheduled on this GPU
    # (8 x 18 CTAs in one launch; peers' partials are HBM-local here, so this checks
    # the TP8 protocol -- two-shot allreduce, per-rank scoreboards -- at full size,
    # not NVLink scaling)
    tp = 8
    prog8 = L.llama_layer_program(build_topology(tp, 1), T, H, HQ, HKV, FF, seq_len=T)
    r8 = L.LayerRunner(prog8, device=dev)
    for pe in range(tp):
        for t in prog8.tensors:
            v = r8.view(t.name, pe)
            if t.name == "rope":
                v.copy_(rope)
            elif t.name in ("g_attn", "g_mlp"):
                v.copy_(g1)
            else:
                sc = (t.shape[1] ** -0.5) if t.name.startswith("w_") else 1.0
                v.copy_((torch.randn(v.shape, generator=g) * sc).to(v.dtype))
    for _ in range(2):
        r8.run(stream)
    torch.cuda.synchronize(dev)
    r8.check()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        r8.run(stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    r8.check()
    ms8 = e0.elapsed_time(e1) / 3
    flops8 = tp * layer_flops(T, H, HQ, HKV, FF, tp)
    tp8 = {"ms_all_8_ranks": round(ms8, 4), "tflops": round(flops8 / (ms8 * 1e-3) / 1e12, 2),
           "tasks_per_rank": len(r8.built.tasks), "ctas_per_rank": r8.num_sms,
           "note": "TP=8 graph, 8 ranks co-resident on one GPU (18 CTAs each); protocol at full "
                   "size, not NVLink scaling"}
    r8.close()
    peak = peaks.get("bf16_tflops", 1622.7)
    return {"workload": f"config 5: Llama-3-70B layer, {T} tokens (one causal sequence), hidden {H}, "
                        f"{HQ}/{HKV} heads, ffn {FF}, TP=1, bf16, one persistent megakernel launch",
            "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 2),
            "flops": flops, "tasks": n_tasks,
            "roofline": {"bound": "tensor", "frac": round(flops / (ms * 1e-3) / 1e12 / peak, 4),
                         "peak": peak, "unit": "TFLOP/s"},
            "comparator": {"impl": "unfused cuBLAS GEMMs + torch SDPA (causal, GQA) + torch elementwise",
                           "ms": round(cms, 4), "speedup": round(cms / ms, 4)},
            "max_rel_err_vs_unfused": round(rel, 5), "tp8_emulated": tp8}


def bench_layer_dist(dev, world, rank, steps, warmup, flush, peaks, shared_gpus, tokens=LAY_T):
    """Config 5 at TP = world, one process per GPU: every rank launches its own
    persistent megakernel over an IPC team (two-shot allreduce tasks over NVLink P2P).
    Comparator: the same rank's shard unfused -- cuBLAS GEMMs, SDPA, torch elementwise
    and two NCCL all_reduce calls.  Fused and unfused steps alternate; times are
    max over ranks."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    from paper_2605_02953_b200 import build_topology
    from paper_2605_02953_b200 import layer as L
    from paper_2605_02953_b200.shmem import Team
    T, H, HQ, HKV, FF = tokens, LAY_H, LAY_HQ, LAY_HKV, LAY_F
    hq, hkv, f = HQ // world, HKV // world, FF // world
    prog = L.llama_layer_program(build_topology(world, 1), T, H, HQ, HKV, FF, seq_len=T)
    built = prog.build()
    nslots = (built.max_task_id + 1) * built.max_tiles_per_op
    team = Team.from_process_group(heap_bytes=prog._top + 4096, signal_slots=nslots + 64)
    runner = L.LayerRunner(prog, built, team=team)
    gs = torch.Generator(device="cpu").manual_seed(77)              # shared across ranks
    gr = torch.Generator(device="cpu").manual_seed(1000 + rank)     # this rank's shard
    mk = lambda gen, *sh, sc=1.0: (torch.randn(*sh, generator=gen) * sc).to(torch.bfloat16).to(f"cuda:{dev}")
    x = mk(gs, T, H)
    g1 = (1 + 0.1 * torch.randn(1, H, generator=gs)).to(torch.bfloat16).to(f"cuda:{dev}")
    g2 = (1 + 0.1 * torch.randn(1, H, generator=gs)).to(torch.bfloat16).to(f"cuda:{dev}")
    rope = torch.from_numpy(L.rope_table(T)).to(f"cuda:{dev}")
    w = {"w_qkv": mk(gr, (hq + 2 * hkv) * 128, H, sc=H ** -0.5), "w_o": mk(gr, H, hq * 128, sc=(HQ * 128) ** -0.5),
         "w_gate_up": mk(gr, 2 * f, H, sc=H ** -0.5), "w_down": mk(gr, H, f, sc=FF ** -0.5)}
    for name, val in [("x", x), ("g_attn", g1), ("g_mlp", g2), ("rope", rope), *w.items()]:
        runner.view(name).copy_(val)
    stream = torch.cuda.current_stream(dev)
    wgu = w["w_gate_up"].view(f // 128, 2, 128, H)
    wg, wu = wgu[:, 0].reshape(f, H).contiguous(), wgu[:, 1].reshape(f, H).contiguous()
    cos, sin = rope[:, :64], rope[:, 64:]

    def rms(t, gg):
        tf = t.float()
        return (tf * torch.rsqrt(tf.pow(2).mean(-1, keepdim=True) + 1e-5) * gg.float()).to(torch.bfloat16)

    def rot(t):
        tf = t.float()
        a1, a2 = tf[..., :64], tf[..., 64:]
        c, s_ = cos[:, None, :], sin[:, None, :]
        return torch.cat([a1 * c - a2 * s_, a2 * c + a1 * s_], -1).to(torch.bfloat16)

    def unfused():
        qkv = rms(x, g1) @ w["w_qkv"].t()
        q = rot(qkv[:, :hq * 128].view(T, hq, 128))
        k = rot(qkv[:, hq * 128:(hq + hkv) * 128].view(T, hkv, 128))
        v = qkv[:, (hq + hkv) * 128:].view(T, hkv, 128)
        att = F.scaled_dot_product_attention(q.transpose(0, 1)[None], k.transpose(0, 1)[None],
                                             v.transpose(0, 1)[None], is_causal=True, enable_gqa=True)
        o = att[0].transpose(0, 1).reshape(T, hq * 128) @ w["w_o"].t()
        dist.all_reduce(o)
        h = o + x
        hn = rms(h, g2)
        d = (F.silu(hn @ wg.t()) * (hn @ wu.t())) @ w["w_down"].t()
        dist.all_reduce(d)
        return d + h

    do_cmp = not shared_gpus  # NCCL needs one GPU per rank
    for _ in range(warmup):
        runner.run(stream)
        if do_cmp:
            unfused()
    torch.cuda.synchronize(dev)
    runner.check()
    dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    cevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for (e0, e1), (c0, c1) in zip(evs, cevs):
        flush.zero_()
        e0.record(stream)
        runner.run(stream)
        e1.record(stream)
        if do_cmp:
            flush.zero_()
            c0.record(stream)
            unfused()
            c1.record(stream)
    torch.cuda.synchronize(dev)
    runner.check()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    cms = sum(a.elapsed_time(b) for a, b in cevs) / steps if do_cmp else 0.0
    ms, cms = max_over_ranks([ms, cms], dev, True)
    flops = world * layer_flops(T, H, HQ, HKV, FF, world)
    out = {"workload": f"config 5 at TP={world}: Llama-3-70B layer, {T} tokens (one causal sequence), "
                       "one persistent megakernel per rank, two-shot allreduce tasks over NVLink P2P",
           "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 2), "flops": flops,
           "tasks_per_rank": len(built.tasks)}
    if do_cmp:
        out["comparator"] = {"impl": "unfused per rank: cuBLAS GEMMs + SDPA + torch elementwise + "
                                     "2 x NCCL all_reduce", "ms": round(cms, 4), "speedup": round(cms / ms, 4)}
    dist.barrier()
    runner.close()
    return out


def bench_attention_dist(dev, world, rank, steps, flush, peaks, shared_gpus):
    """Config 3 at SP = world, one process per GPU: the fused AG-KV flash attention
    (K/V chunks pulled from the peers while the tensor cores start on the local
    chunk) against NCCL all_gather of K and V + SDPA on the same shard."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    from paper_2605_02953_b200.attention import AllGatherKVAttention
    from paper_2605_02953_b200.shmem import Team
    S, HQ, HKV, D = int(os.environ.get("TF_BENCH_ATT_S", ATT_S)), ATT_HQ, ATT_HKV, ATT_D
    sl = S // world
    team = Team.from_process_group(heap_bytes=4 * S * HKV * D * 2 + (16 << 20), signal_slots=256)
    g = torch.Generator(device="cpu").manual_seed(500 + rank)
    mk = lambda *sh: torch.randn(*sh, generator=g).to(torch.bfloat16).to(f"cuda:{dev}")
    q, k, v = mk(sl, HQ, D), mk(sl, HKV, D), mk(sl, HKV, D)
    out = torch.empty_like(q)
    op = AllGatherKVAttention(team, sl, HQ, HKV, D)
    kall = torch.empty(S, HKV, D, dtype=torch.bfloat16, device=f"cuda:{dev}")
    vall = torch.empty_like(kall)
    stream = torch.cuda.current_stream(dev)

    def unfused():
        dist.all_gather_into_tensor(kall, k)
        dist.all_gather_into_tensor(vall, v)
        return F.scaled_dot_product_attention(q.transpose(0, 1)[None], kall.transpose(0, 1)[None],
                                              vall.transpose(0, 1)[None], enable_gqa=True)

    do_cmp = not shared_gpus
    for _ in range(2):
        op(q, k, v, out)
        if do_cmp:
            unfused()
    torch.cuda.synchronize(dev)
    team.check()
    dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    cevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for (e0, e1), (c0, c1) in zip(evs, cevs):
        flush.zero_()
        e0.record(stream)
        op(q, k, v, out)
        e1.record(stream)
        if do_cmp:
            flush.zero_()
            c0.record(stream)
            unfused()
            c1.record(stream)
    torch.cuda.synchronize(dev)
    team.check()
    ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    cms = sum(a.elapsed_time(b) for a, b in cevs) / steps if do_cmp else 0.0
    ms, cms = max_over_ranks([ms, cms], dev, True)
    flops = 4.0 * sl * S * D * HQ
    nv = (world - 1) / world * S * HKV * D * 2 * 2  # K and V bytes pulled per rank
    res = {"workload": f"config 3 at SP={world}: fused AG-KV flash attention, Q[{sl},64,128] per rank vs "
                       f"K/V[{S},8,128] gathered over NVLink (non-causal, GQA 8:1, bf16)",
           "ms_per_rank": round(ms, 4), "tflops_per_rank": round(flops / (ms * 1e-3) / 1e12, 2),
           "tflops_total": round(world * flops / (ms * 1e-3) / 1e12, 2),
           "roofline": {"bound": "tensor", "t_roof_ms": round(max(flops / (peaks.get("bf16_tflops", 1622.7) * 1e12),
                                                                   nv / (NVLINK_GBS * 1e9)) * 1e3, 4),
                        "frac": round(max(flops / (peaks.get("bf16_tflops", 1622.7) * 1e12), nv / (NVLINK_GBS * 1e9))
                                      / (ms * 1e-3), 4)}}
    if do_cmp:
        res["comparator"] = {"impl": "NCCL all_gather(K), all_gather(V) + torch SDPA", "ms": round(cms, 4),
                             "speedup": round(cms / ms, 4)}
    dist.barrier()
    team.close()
    return res


# ------------------------------------------------------------------ GPU arm
def main_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_02953_b200 import kernels as K
    from paper_2605_02953_b200.shmem import Team

    if args.only_attn:  # probe: config 3 only
        torch.cuda.set_device(0)
        print(json.dumps(bench_attention(0, max(args.steps, 3), load_peaks()[0])), flush=True)
        return
    if args.only_agmoe:  # probe: ag_moe_group_gemm only
        torch.cuda.set_device(0)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
        print(json.dumps(bench_ag_moe(0, 1, 0, args.steps, args.warmup, flush, torch.cuda.Stream(), False,
                                      load_peaks()[0])), flush=True)
        return
    if args.only_moe:  # probe: config 4 dispatch/combine only
        torch.cuda.set_device(0)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
        team = Team(1, [0], heap_bytes=2 * MOE_T * MOE_K * MOE_H * 2 + (64 << 20), signal_slots=4096)
        print(json.dumps(bench_moe(team, 0, 1, 0, args.steps, args.warmup, flush, torch.cuda.Stream(), False,
                                   load_peaks()[0])), flush=True)
        return
    if args.only_layer:  # probe: config 5 only
        torch.cuda.set_device(0)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
        print(json.dumps(bench_layer(0, args.steps, args.warmup, load_peaks()[0], flush)), flush=True)
        return
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    distributed = world_env > 1
    shared_gpus = False
    if distributed:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        ndev = torch.cuda.device_count()
        shared_gpus = ndev < world_env  # test mode: several ranks per GPU (NCCL refuses that)
        dev0 = local % ndev
        torch.cuda.set_device(dev0)
        if shared_gpus:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev0}"))
        rank, world = dist.get_rank(), dist.get_world_size()
    else:
        torch.cuda.set_device(0)
        rank, world = 0, 1
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev = torch.cuda.current_device()
    tp = world
    if shared_gpus and rank == 0:
        print(f"[bench] {world} ranks share {torch.cuda.device_count()} GPU(s): functional run "
              "only, numbers are not GPU-scaling measurements", file=sys.stderr)
    m, f_tp = TOKENS, FFN // tp
    mpr = m // tp
    peaks, peaks_kind = load_peaks()

    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    def rnd(*shape, scale=1.0):
        return (torch.randn(*shape, generator=g) * scale).to(torch.bfloat16).to(f"cuda:{dev}")
    x = rnd(mpr, HIDDEN)
    w1 = rnd(f_tp, HIDDEN, scale=HIDDEN ** -0.5)
    w2 = rnd(HIDDEN, f_tp, scale=f_tp ** -0.5)
    h = torch.empty(m, f_tp, dtype=torch.bfloat16, device=f"cuda:{dev}")
    y = torch.empty(mpr, HIDDEN, dtype=torch.bfloat16, device=f"cuda:{dev}")

    heap = 2 * m * HIDDEN * 2 + m * ((HIDDEN + 7) // 8 * 8) * 2 + (64 << 20)
    heap += 2 * m * HIDDEN * 2 + (16 << 20)  # in-kernel-pull AG variant (ag_sm_pull below)
    if not args.no_moe:  # EP receive + expert-output buffers (worst case: every token to one rank)
        heap += 2 * MOE_T * MOE_K * world * MOE_H * 2 + (8 << 20)
    if distributed:
        team = Team.from_process_group(heap_bytes=heap, signal_slots=4096)
    else:
        team = Team(1, [dev], heap_bytes=heap, signal_slots=4096)
    # ranks sharing one GPU (functional test mode): each rank's persistent GEMM takes its
    # share of the SMs, so every rank's kernels are co-resident and their flags can move
    gemm_sms = 0
    if shared_gpus:
        per_gpu = -(-world // torch.cuda.device_count())
        gemm_sms = max(2, (torch.cuda.get_device_properties(dev).multi_processor_count // per_gpu - 8) & ~1)
    ag = K.AllGatherGemm(team, m, HIDDEN, f_tp, block_n=256, group_m=args.group_m, num_gemm_sms=gemm_sms)
    rs = K.GemmReduceScatter(team, m, f_tp, HIDDEN, block_n=256, group_m=args.group_m, num_comm_sms=8,
                             num_gemm_sms=gemm_sms,
                             fuse_scatter=True, reduce_order="ascending")
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    def barrier():
        if distributed:
            dist.barrier()



    def step():
        ag(x, w1, h)
        rs(h, w2, y)

    # ---- cuBLAS comparator (same GEMMs, torch.matmul; unfused NCCL at N>1)
    xg = torch.empty(m, HIDDEN, dtype=torch.bfloat16, device=f"cuda:{dev}")
    hp = torch.empty(m, HIDDEN, dtype=torch.bfloat16, device=f"cuda:{dev}")

    def cublas_step():
        if distributed:
            dist.all_gather_into_tensor(xg, x)
            hh = torch.matmul(xg, w1.t())
            torch.matmul(hh, w2.t(), out=hp)
            dist.reduce_scatter_tensor(y, hp)
        else:
            hh = torch.matmul(x, w1.t())
            torch.matmul(hh, w2.t())

    def time_cublas(n):
        # same protocol as our timed loop: flush, event, step, event -- no host syncs
        with torch.cuda.stream(stream):
            for _ in range(3):
                cublas_step()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(n)]
            for e0, e1 in evs:
                flush.zero_()
                e0.record(stream)
                cublas_step()
                e1.record(stream)
            torch.cuda.synchronize()
        return sum(e0.elapsed_time(e1) for e0, e1 in evs) / n

    cub_before = None if shared_gpus else time_cublas(args.steps)
    n_events = args.steps
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_events)]
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(dev)
        clocks.start()
        clocks.wait_first()
        t_clk0 = time.time()
        for i in range(args.steps):
            flush.zero_()  # evict L2 between steps (outside the per-step events)
            ev[i][0].record(stream)
            ag(x, w1, h)
            ev[i][1].record(stream)
            rs(h, w2, y)
            ev[i][2].record(stream)
        torch.cuda.synchronize()
        t_clk1 = time.time()
        barrier()
        torch.cuda.synchronize()
        clk = clocks.stop(t_clk0, t_clk1)
    team.check()
    # AG-GEMM with the gather inside the GEMM launch (16 pull-engine CTAs; copy-engine
    # pulls above): same flush/event protocol, reported beside the main line
    ag_sm = None
    try:
        ag_pull = K.AllGatherGemm(team, m, HIDDEN, f_tp, block_n=256, num_comm_sms=16, num_gemm_sms=gemm_sms)
        h2 = torch.empty_like(h)
        with torch.cuda.stream(stream):
            for _ in range(2):
                ag_pull.forward(x, w1, h2)
            torch.cuda.synchronize()
            barrier()
            evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(max(3, args.steps // 2))]
            for e0, e1 in evp:
                flush.zero_()
                e0.record(stream)
                ag_pull.forward(x, w1, h2)
                e1.record(stream)
            torch.cuda.synchronize()
        team.check()
        sm_ms = max_over_ranks([sum(a.elapsed_time(b) for a, b in evp) / len(evp)], dev, distributed)[0]
        ag_sm = {"impl": "AllGatherGemm(num_comm_sms=16): gather by pull-engine CTAs inside the GEMM launch",
                 "ms": round(sm_ms, 4), "tflops_per_rank": round(2.0 * m * f_tp * HIDDEN / (sm_ms * 1e-3) / 1e12, 2)}
    except Exception as exc:  # noqa: BLE001
        ag_sm = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    ag_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(n_events)]
    rs_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in range(n_events)]
    step_ms = sum(a + b for a, b in zip(ag_ms, rs_ms)) / n_events
    gemm_flops = 2.0 * m * f_tp * HIDDEN  # per GEMM per rank
    # max over ranks
    step_ms, ag_avg, rs_avg = max_over_ranks(
        [step_ms, sum(ag_ms) / n_events, sum(rs_ms) / n_events], dev, distributed)
    total_flops = 2 * gemm_flops * world
    value = total_flops / (step_ms * 1e-3) / 1e12

    cub_ms = None
    overlap = None
    if not shared_gpus:  # NCCL cannot run with several ranks on one GPU
        cub_ms = 0.5 * (cub_before + time_cublas(args.steps)) if cub_before else time_cublas(args.steps)
        cub_ms = max_over_ranks([cub_ms], dev, distributed)[0]
        if distributed:
            # overlap efficiency, the reference's formula (simengine.py:346-352):
            # hidden = 1 - (t_fused - t_gemm_alone) / t_comm_alone, with the GEMMs alone
            # (cuBLAS, on the pre-gathered operand) and the collectives alone (NCCL)
            def time_fn(fn, n):
                with torch.cuda.stream(stream):
                    for _ in range(2):
                        fn()
                    torch.cuda.synchronize()
                    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                           for _ in range(n)]
                    for e0, e1 in evs:
                        flush.zero_()
                        e0.record(stream)
                        fn()
                        e1.record(stream)
                    torch.cuda.synchronize()
                return sum(a.elapsed_time(b) for a, b in evs) / n

            def gemms_only():
                hh = torch.matmul(xg, w1.t())
                torch.matmul(hh, w2.t(), out=hp)

            def comm_only():
                dist.all_gather_into_tensor(xg, x)
                dist.reduce_scatter_tensor(y, hp)

            t_gemm = max_over_ranks([time_fn(gemms_only, args.steps)], dev, distributed)[0]
            t_comm = max_over_ranks([time_fn(comm_only, args.steps)], dev, distributed)[0]
            hidden = 1.0 - (step_ms - t_gemm) / t_comm if t_comm > 0 else 0.0
            overlap = {"t_fused_ms": round(step_ms, 4), "t_gemm_alone_ms": round(t_gemm, 4),
                       "t_comm_alone_ms": round(t_comm, 4),
                       "hidden_fraction": round(min(max(hidden, 0.0), 1.0), 4),
                       "speedup_vs_serial": round((t_gemm + t_comm) / step_ms, 4),
                       "formula": "1 - (t_fused - t_gemm_alone) / t_comm_alone (simengine.py:346-352); "
                                  "gemm = cuBLAS, comm = NCCL all_gather + reduce_scatter"}

    # ---- e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # Every step: H2D of its activations from pinned host memory, the fused
        # AG-GEMM -> GEMM-RS, D2H of its result.  Copies run on copy-engine
        # streams double-buffered against the compute stream, so step i+1's upload
        # and step i-1's download overlap step i's GEMMs (as a serving loop would).
        nb = 2
        x_host = [x.cpu().pin_memory() for _ in range(nb)]
        y_host = [torch.empty(mpr, HIDDEN, dtype=torch.bfloat16).pin_memory() for _ in range(nb)]
        x_dev = [torch.empty_like(x) for _ in range(nb)]
        y_dev = [torch.empty_like(y) for _ in range(nb)]
        h2d_s = torch.cuda.Stream(device=dev)
        d2h_s = torch.cuda.Stream(device=dev)
        n_e2e = 3 * args.steps + 2  # a pipelined serving loop: fill/drain amortised over the steps

        def run_e2e(n):
            ev_h2d = [torch.cuda.Event() for _ in range(n)]
            ev_cmp = [torch.cuda.Event() for _ in range(n)]
            ev_d2h = [torch.cuda.Event() for _ in range(n)]
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(h2d_s)
            for i in range(n):
                b = i % nb
                if i >= nb:
                    h2d_s.wait_event(ev_cmp[i - nb])       # x_dev[b] free again
                with torch.cuda.stream(h2d_s):
                    x_dev[b].copy_(x_host[b], non_blocking=True)
                ev_h2d[i].record(h2d_s)
                stream.wait_event(ev_h2d[i])
                if i >= nb:
                    stream.wait_event(ev_d2h[i - nb])      # y_dev[b] downloaded
                with torch.cuda.stream(stream):
                    ag(x_dev[b], w1, h)
                    rs(h, w2, y_dev[b])
                ev_cmp[i].record(stream)
                d2h_s.wait_event(ev_cmp[i])
                with torch.cuda.stream(d2h_s):
                    y_host[b].copy_(y_dev[b], non_blocking=True)
                ev_d2h[i].record(d2h_s)
            t1.record(d2h_s)
            torch.cuda.synchronize()
            return t0.elapsed_time(t1) / n

        run_e2e(3)
        barrier()
        e2e_ms = max_over_ranks([run_e2e(n_e2e)], dev, distributed)[0]
        e2e = {"value": round(total_flops / (e2e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(e2e_ms, 4), "steps": n_e2e,
               "h2d_bytes_per_step": x.numel() * 2, "d2h_bytes_per_step": y.numel() * 2,
               "note": "pinned host buffers; H2D/D2H on copy streams overlapped with the "
                       "previous/next step's GEMMs (double-buffered)"}

    # ---- roofline of the dominant kernel (the tcgen05 GEMM; one launch per op at N=1)
    # achieved = algorithmic FLOPs per launch / the MEAN event-timed duration of the two
    # fused ops (each is one launch of the GEMM kernel at N=1; at N>1 the op's time
    # includes its exchange); per-op rooflines use the north_star definition
    # t_roof = max(FLOPs / tensor peak, NVLink bytes / 900 GB/s link bandwidth)
    peak = peaks.get("bf16_tflops", 1622.7)
    peak_sus = peaks.get("bf16_tflops_sustained", peak)
    nv_bytes = (world - 1) / world * m * HIDDEN * 2 if world > 1 else 0
    mean_ms = 0.5 * (ag_avg + rs_avg)
    achieved = gemm_flops / (mean_ms * 1e-3) / 1e12

    def op_roof(ms):
        t_tc, t_nv = gemm_flops / (peak * 1e12), nv_bytes / NVLINK_GBS / 1e9
        t_nv_meas = nv_bytes / NVLINK_MEASURED_GBS / 1e9
        return {"ms": round(ms, 4), "tflops": round(gemm_flops / (ms * 1e-3) / 1e12, 2),
                "t_roof_ms": round(max(t_tc, t_nv) * 1e3, 4), "frac": round(max(t_tc, t_nv) / (ms * 1e-3), 4),
                "frac_vs_measured_p2p": round(max(t_tc, t_nv_meas) / (ms * 1e-3), 4),
                "nvlink_bytes": nv_bytes}
    roof = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "frac_of_sustained": round(achieved / peak_sus, 4),
            "peak_kind": f"{peaks_kind} burst bf16 (MEASURED_PEAKS.json bf16_tflops)",
            "achieved_def": "2*M*N*K per launch / mean(ag_gemm ms, gemm_rs ms)",
            "traffic": _committed_traffic(), "kernel": "gemm_sm100_kernel<CG=2,MH=2,BN=256,bf16> (512x256 tile per CTA pair)",
            "group_m": args.group_m, "flops_per_launch": gemm_flops,
            "nvlink_gbs": {"link": NVLINK_GBS, "measured_p2p": NVLINK_MEASURED_GBS},
            "per_op": {"ag_gemm": op_roof(ag_avg), "gemm_rs": op_roof(rs_avg)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))
        # the same bounded sample as the reference arm, repeated for >= 10 s of timed CPU work
        d = cpu_sample(tp, min_seconds=10.0)
        cpu = {"value": round(d["value"], 6), "unit": "TFLOP/s", "cores": d["cores"], "kind": d["kind"],
               "sample": d["sample"] + f"; {d['steps']} steps, >= 10 s of timed CPU work",
               "seconds_per_step": round(d["seconds_per_step"], 3),
               "oracle_tflops": round(d["oracle_tflops"], 6),
               "one_thread": cpu_sample_1thread(tp)}

    moe = None
    if not args.no_moe and shared_gpus:
        # the fused dispatch keeps one CTA per SM co-resident per rank (grid-wide waits):
        # two ranks' launches cannot share one GPU at this size (tests/test_gpu_ipc.py covers
        # the protocol with ranks sharing a GPU at sizes whose grids fit together)
        moe = {"skipped": "ranks share a GPU: the fused dispatch grid needs every SM per rank"}
    elif not args.no_moe:
        moe = bench_moe(team, dev, world, rank, args.steps, args.warmup, flush, stream,
                        distributed, peaks)

    agmoe = None
    if not args.no_moe:
        try:
            agmoe = bench_ag_moe(dev, world, rank, max(3, args.steps // 2), 2, flush, stream, distributed, peaks)
        except Exception as exc:  # noqa: BLE001
            agmoe = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    attn = None
    if not args.no_attn and world == 1:
        attn = bench_attention(dev, 3, peaks)
    elif not args.no_attn:
        try:  # failure-isolated, like the layer section
            attn = bench_attention_dist(dev, world, rank, 3, flush, peaks, shared_gpus)
        except Exception as exc:  # noqa: BLE001
            attn = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    layer = None
    if not args.no_layer and world == 1:
        layer = bench_layer(dev, max(3, args.steps // 4), 2, peaks, flush)
    elif not args.no_layer:
        try:  # a failure here must not cost the config-2 / MoE line of the scaling run
            layer = bench_layer_dist(dev, world, rank, max(3, args.steps // 4), 2, flush, peaks, shared_gpus,
                                     tokens=int(os.environ.get("TF_BENCH_LAYER_TOKENS", LAY_T)))
        except Exception as exc:  # noqa: BLE001
            layer = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    # our kernels per timed step: N=1 -> AG GEMM + its split-K tail fix-up (1792 pair tiles leave a
    # partial last wave) + RS GEMM (profiles/r01_launches_v2.txt); N>1 adds the barrier
    # arrive/wait kernels of both ops and the RS owner-reduce kernel
    launches_per_step = 3 if world == 1 else (3 + 2 + 2 + 1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded N(0,1) activations, 1/sqrt(K)-scaled weights)",
            "config": {"workload": f"llama3-70b MLP: AG-GEMM(M={m},N={f_tp},K={HIDDEN}) + "
                                   f"GEMM-RS(M={m},N={HIDDEN},K={f_tp}), TP={tp}",
                       "tokens": TOKENS, "hidden": HIDDEN, "ffn": FFN, "tp": tp,
                       "parallelism": f"tp{tp}", "l2": "flushed between steps (256 MiB memset), "
                       "outside the per-step events"},
            "roofline": roof,
            "comparator": None if cub_ms is None else {
                "impl": "cuBLAS (torch.matmul)" + (" + NCCL all_gather/reduce_scatter"
                                                   if distributed else ""),
                "ms_per_step": round(cub_ms, 4),
                "tflops": round(total_flops / (cub_ms * 1e-3) / 1e12, 3),
                "speedup": round(cub_ms / step_ms, 4)},
            "overlap": overlap,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "moe": moe, "ag_moe": agmoe, "attention": attn, "layer": layer,
            "ag_sm_pull": ag_sm,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    main_ours(args)


if __name__ == "__main__":
    main()
