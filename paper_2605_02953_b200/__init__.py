"""B200-native (sm_100a) fused collectives behind the overlapsim operator API.

Hot path (BASELINE.json north_star): AllGather+GEMM, GEMM+ReduceScatter and the
MoE expert-parallel dispatch/combine, on a symmetric-memory runtime with
device-side flags.  See DESIGN.md.
"""

from .context import WorkloadContext, WorkloadRun, reduce_visit_order
from .errors import (AllocationError, BuildError, ConfigError, DeadlockError, ProtocolError,
                     VerificationError)
from .topology import (LINK_PROFILES, LinkConfig, Topology, build_topology, local_rank_of, node_of,
                       topology_from_config)

__all__ = [
    "WorkloadContext", "WorkloadRun", "reduce_visit_order", "AllocationError", "BuildError",
    "ConfigError", "DeadlockError", "ProtocolError", "VerificationError", "LINK_PROFILES",
    "LinkConfig", "Topology", "build_topology", "local_rank_of", "node_of", "topology_from_config",
    "Token", "consume_token",
    "ag_gemm", "gemm_rs", "gemm", "gemm_allreduce", "AllGatherGemm", "GemmReduceScatter",
    "SymmetricHeap", "Team", "ag_moe_group_gemm", "ExpertParallelMoE", "moe_route", "ag_kv_scores",
]


def __getattr__(name):
    # the operator modules import torch + the CUDA library lazily
    if name in ("ag_gemm", "gemm_rs", "gemm", "gemm_allreduce", "AllGatherGemm", "GemmReduceScatter"):
        from . import kernels
        return getattr(kernels, name)
    if name in ("ag_moe_group_gemm", "ExpertParallelMoE", "moe_route"):
        from . import moe
        return getattr(moe, name)
    if name in ("ag_kv_scores",):
        from . import attention
        return getattr(attention, name)
    if name in ("SymmetricHeap", "Team", "Token", "consume_token"):
        from . import shmem
        return getattr(shmem, name)
    raise AttributeError(name)
