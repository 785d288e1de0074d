"""Run configuration and result bundle (mirrors ovs/kernels/context.py:18-81).

The reference fields keep their meaning:
  block_m / block_n / block_k / group_m  tile shape and swizzle_2d group.  The
      tensor-core tile is fixed at 128 x {128, 256} x 64 on sm_100a; block_m is
      still validated like the reference, the device tile uses 128 rows and
      block_n > 128 selects the 256-column variant.
  num_gemm_sms   persistent GEMM CTAs (the reference's compute workers stride
      tiles by this count, ag_gemm.py:81 -- so does the kernel); 0 = all SMs.
  num_comm_sms   CTAs reserved for reduce / pack kernels.
  fuse_scatter, swizzle, reduce_order   as in the reference.
B200 additions: `devices` (CUDA device per rank; repeats allowed = several ranks
emulated on one GPU) and `out_dtype` ("bf16" | "f32" | None = follow inputs).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .topology import Topology

SUPPORTED_NUMPY = (np.dtype(np.float32), np.dtype(np.int64))
REDUCE_ORDERS = ("ring", "ascending")


@dataclass
class WorkloadContext:
    topology: Topology
    block_m: int = 16
    block_n: int = 16
    block_k: int = 16
    group_m: int = 4
    num_gemm_sms: int = 2
    num_comm_sms: int = 1
    fuse_scatter: bool = False
    use_multimem_st: bool = False
    swizzle: bool = True
    reduce_order: str = "ring"
    seed: int = 0
    devices: list | None = None
    out_dtype: str | None = None
    # B200 extension: how ag_gemm gathers -- "ce" (copy-engine pulls on a side stream,
    # flags per row slice) or "sm" (num_comm_sms pull-engine CTAs inside the GEMM launch)
    ag_pull: str = "ce"

    def __post_init__(self):
        if min(self.block_m, self.block_n, self.block_k, self.group_m) < 1:
            raise ConfigError("block and group sizes must be >= 1")
        if self.num_gemm_sms < 0 or self.num_comm_sms < 0:
            raise ConfigError("SM counts must be >= 0")
        if self.num_gemm_sms + self.num_comm_sms > self.topology.num_sms:
            raise ConfigError(f"{self.num_gemm_sms}+{self.num_comm_sms} workers exceed "
                              f"{self.topology.num_sms} SMs per rank")
        if self.reduce_order not in REDUCE_ORDERS:
            raise ConfigError(f"reduce_order must be one of {REDUCE_ORDERS}")
        if self.ag_pull not in ("ce", "sm"):
            raise ConfigError("ag_pull must be 'ce' or 'sm'")
        if self.out_dtype not in (None, "bf16", "f32"):
            raise ConfigError("out_dtype must be None, 'bf16' or 'f32'")
        if self.devices is not None and len(self.devices) != self.topology.world_size:
            raise ConfigError("devices must list one CUDA device per rank")

    @property
    def hw_block_n(self) -> int:
        return 128 if self.block_n <= 128 else 256

    @property
    def hw_block_m(self) -> int:
        # 512 / 256 = CTA pair per tile (tcgen05 cta_group::2, two or one M=256
        # MMA per k-step); smaller = one CTA, 128 rows
        if self.block_m >= 512 and self.hw_block_n == 256:
            return 512
        return 256 if self.block_m >= 256 else 128


@dataclass
class WorkloadRun:
    """Outputs plus what is needed to inspect the run (context.py:57-64).
    `trace` is None: there is no simulated timeline on hardware."""

    outputs: list
    trace: object
    heap: object
    handles: dict = field(default_factory=dict)


def reduce_visit_order(begin: int, n: int, order: str) -> list[int]:
    """context.py:77-81 -- ascending, or ring starting at begin+1."""
    if order == "ascending":
        return list(range(n))
    return [(begin + 1 + i) % n for i in range(n)]
