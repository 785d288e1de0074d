"""torchrun worker: the fused AG-KV flash attention with one process per rank over
an IPC team (K/V chunks pulled from the peer), checked against the oracle.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29513 tests/dist/attn_ipc_worker.py
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
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from oracle import attention as OA
    from oracle.collectives import compare
    from paper_2605_02953_b200.attention import AllGatherKVAttention
    from paper_2605_02953_b200.shmem import Team

    sl, hq, hkv, d = (int(os.environ.get("ATTN_SL", "256")), int(os.environ.get("ATTN_HQ", "4")),
                      int(os.environ.get("ATTN_HKV", "2")), 128)
    rng = np.random.default_rng(5)  # same stream everywhere: every rank knows all shards
    qs = [rng.standard_normal((sl, hq, d)).astype(np.float32) for _ in range(world)]
    ks = [rng.standard_normal((sl, hkv, d)).astype(np.float32) for _ in range(world)]
    vs = [rng.standard_normal((sl, hkv, d)).astype(np.float32) for _ in range(world)]
    bf = lambda a: torch.from_numpy(a).to(torch.bfloat16).cuda()
    team = Team.from_process_group(heap_bytes=4 * sl * world * hkv * d * 2 + (8 << 20), signal_slots=256)
    op = AllGatherKVAttention(team, sl, hq, hkv, d)
    q, k, v = bf(qs[rank]), bf(ks[rank]), bf(vs[rank])
    want = OA.ref_ag_kv_attention([bf(x).float().cpu().numpy() for x in qs],
                                  [bf(x).float().cpu().numpy() for x in ks],
                                  [bf(x).float().cpu().numpy() for x in vs], hkv, d ** -0.5)[rank]
    ok = True
    for _ in range(3):
        out = op(q, k, v)
        torch.cuda.synchronize()
        team.check()
        ok &= compare(out.float().cpu().numpy(), want) <= 2e-2
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("ATTN_IPC_OK" if int(flag) else "ATTN_IPC_FAIL", flush=True)
    dist.barrier()
    team.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
