"""Device placement for multi-rank GPU tests.

Each rank gets its own GPU when the box has at least `world` of them, so that
the .sys-scope release/acquire between devices, copy-engine peer pulls with
stream-written flags, and peer access / IPC mappings run over NVLink.  With
fewer GPUs (a 1-GPU lease) the ranks share cuda:0 (single-device emulation).
TF_TEST_SHARED_GPU=1 forces the shared mode."""

import os

import torch


def devices_for(world: int) -> list[int]:
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if os.environ.get("TF_TEST_SHARED_GPU") == "1" or n < world:
        return [0] * world
    return list(range(world))


def distinct(world: int) -> bool:
    d = devices_for(world)
    return len(set(d)) == len(d)
