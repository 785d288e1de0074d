"""torchrun worker: the one-process-per-GPU (IPC team) path of AG-GEMM, GEMM-RS
and MoE dispatch/combine, checked against the oracle.  When there are fewer
GPUs than ranks, ranks share devices (CUDA IPC works across processes on one
device; contexts time-slice), which exercises the same code as a real box.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tests/dist/ipc_worker.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from oracle import collectives as OC
    from oracle import moe as OM
    from paper_2605_02953_b200 import kernels as K
    from paper_2605_02953_b200 import moe as M
    from paper_2605_02953_b200.shmem import Team

    team = Team.from_process_group(heap_bytes=256 << 20, signal_slots=1024)
    rng = np.random.default_rng(7)  # same stream on every rank: everyone knows all shards
    mpr, n, k = 256, 384, 512
    m = mpr * world
    a_all = [rng.integers(-8, 8, (mpr, k)) for _ in range(world)]
    b_all = [rng.integers(-8, 8, (n, k)) for _ in range(world)]
    x_all = [rng.integers(-8, 8, (m, k)) for _ in range(world)]
    w_all = [rng.integers(-8, 8, (n, k)) for _ in range(world)]

    def bf(x):
        return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).cuda()

    ok = True
    for bm in (128, 256, 512):
        ag = K.AllGatherGemm(team, m, k, n, out_dtype=torch.float32, block_m=bm)
        for it in range(3):  # repeated calls exercise the epoch / double-buffer protocol
            c = ag(bf(a_all[rank]), bf(b_all[rank]))
            torch.cuda.synchronize()
            want = OC.ref_allgather_gemm(a_all, b_all)[rank]
            ok &= np.array_equal(c.cpu().numpy().astype(np.int64), want)
        for fused in (True, False):
            rs = K.GemmReduceScatter(team, m, k, n, out_dtype=torch.float32, block_m=bm,
                                     fuse_scatter=fused, num_comm_sms=4)
            for it in range(3):
                y = rs(bf(x_all[rank]), bf(w_all[rank]))
                torch.cuda.synchronize()
                want = OC.ref_reduce_scatter(x_all, w_all)[rank]
                ok &= np.array_equal(y.cpu().numpy().astype(np.int64), want)
        for two_shot in (False, True):
            ar = K.GemmAllReduce(team, mpr, k, n, out_dtype=torch.float32, block_m=bm,
                                 two_shot=two_shot, num_comm_sms=2)
            for it in range(3):
                y = ar(bf(a_all[rank]), bf(b_all[rank]))
                torch.cuda.synchronize()
                ok &= np.array_equal(y.cpu().numpy().astype(np.int64), OC.ref_allreduce(a_all, b_all))
    team.check()

    # MoE EP dispatch / combine
    e, topk, t, h = 16, 4, 64, 256
    xs = [rng.standard_normal((t, h)).astype(np.float32) for _ in range(world)]
    logits = [rng.standard_normal((t, e)).astype(np.float32) for _ in range(world)]
    ep = M.ExpertParallelMoE(team, e, h, topk, max_tokens=t)
    idx, w = M.moe_route(torch.from_numpy(logits[rank]).cuda(), topk)
    xb = torch.from_numpy(xs[rank]).to(torch.bfloat16).cuda()
    recv = ep.dispatch(xb, idx)
    torch.cuda.synchronize()
    idx_all = [OM.topk_route(lg, topk)[0] for lg in logits]
    counts, want_recv, slot_row = OM.dispatch_layout(idx_all, e, world)
    ok &= np.array_equal(ep.counts().cpu().numpy(), counts)
    nrow = ep.recv_rows()
    xs_bf = [torch.from_numpy(x).to(torch.bfloat16).float().numpy() for x in xs]
    want = np.stack([xs_bf[s][tok] for s, tok, _ in want_recv[rank]]) if nrow else np.zeros((0, h))
    ok &= nrow == len(want_recv[rank]) and np.array_equal(recv[:nrow].float().cpu().numpy(), want)
    ep.expert_out()[:nrow] = recv[:nrow]
    out = ep.combine(idx, w)
    torch.cuda.synchronize()
    w_all = [OM.topk_route(lg, topk)[1] for lg in logits]
    ys = []
    # every rank's expert outputs equal its received rows: rebuild them from the oracle layout
    for d in range(world):
        rows = [xs_bf[s][tok] for s, tok, _ in want_recv[d]]
        ys.append(np.stack(rows) if rows else np.zeros((0, h), np.float32))
    want_out = OM.combine(ys, idx_all, w_all, e)[rank]
    ok &= OC.compare(out.float().cpu().numpy(), want_out) <= 2e-2
    team.check()

    res = torch.tensor([1 if ok else 0])
    dist.all_reduce(res, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("IPC_OK" if res.item() == 1 else "IPC_FAIL", flush=True)
    dist.barrier()
    team.close()
    dist.destroy_process_group()
    sys.exit(0 if res.item() == 1 else 1)


if __name__ == "__main__":
    main()
