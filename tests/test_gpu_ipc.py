"""GPU test of the one-process-per-GPU (torchrun, CUDA IPC) path.  With a
single GPU both ranks share cuda:0 -- the IPC mapping, epoch flags, barriers and
fused kernels are the same code as on an 8-GPU box."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc", [2])
def test_torchrun_ipc_team_parity(nproc):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "dist", "ipc_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "IPC_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


def test_torchrun_layer_megakernel_ipc():
    """Config-5 layer, one process per rank (IPC team), allreduce over P2P."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "dist", "layer_ipc_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "LAYER_IPC_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("shape", [None, (2048, 64, 8)])
def test_torchrun_attention_ipc(shape):
    """Config-3 fused AG-KV attention, one process per rank (IPC team).  The big
    shape launches more CTAs than one GPU holds for both ranks at once: it only
    finishes because K/V tiles are read straight from each owner's chunk (no
    device-side pull that waits on co-resident CTAs of the other rank)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    env = dict(os.environ)
    if shape:
        env.update(ATTN_SL=str(shape[0]), ATTN_HQ=str(shape[1]), ATTN_HKV=str(shape[2]))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "dist", "attn_ipc_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "ATTN_IPC_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
