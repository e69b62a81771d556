"""paper_2504_19442_b200: B200-native fused AllGather+GEMM / GEMM+ReduceScatter.

A drop-in for the ``ag_gemm`` / ``gemm_rs`` path of the reference package
``minishmem`` (arXiv 2504.19442's programming model): the same World /
WorldSpec / Pe / SymHandle / SignalSet surface, the same swizzle schedules
and ProblemShape, the same exception taxonomy -- with a GPU symmetric heap
over NVLink and hand-written sm_100a (tcgen05 / TMEM / TMA) kernels behind a
C ABI (include/shmem_b200.h).
"""

import os as _os

# Ranks that share one GPU (single-process worlds on a 1-GPU box) drive 2
# streams each; with the default 8 hardware queues, work of different
# streams can be serialised behind a spinning kernel.  Must be set before
# the CUDA context exists; World() checks it.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .core import (
    Pe,
    RankCtx,
    SignalSet,
    SymHandle,
    World,
    WorldSpec,
    exchange_ipc_handles,
    init_world,
    init_world_dist,
)
from .errors import (
    AllocationError,
    ArgumentError,
    CapacityError,
    CollectiveFault,
    ConfigurationError,
    OverlapInfeasibleError,
    RangeError,
    ShmemError,
    SynchronizationFault,
    UsageError,
)
from .pipelines import (
    SYNC_TOKEN,
    SYNC_WAIT,
    AgGemmBuffers,
    GemmRsBuffers,
    ProblemShape,
    ag_gemm,
    gemm,
    gemm_rs,
    make_ag_gemm_buffers,
    make_gemm_rs_buffers,
)
from .collectives import (
    ChunkLayout,
    allgather_pull_intra,
    allgather_push_intra,
    reducescatter_push_intra,
)
from .primitives import SignalOp, Token, WaitCond, consume_token
from .swizzle import TileSchedule, TileStep, ag_order_fullmesh, ag_order_switch, rs_inter_order

__all__ = [
    "AgGemmBuffers", "AllocationError", "ArgumentError", "CapacityError", "CollectiveFault",
    "ConfigurationError", "GemmRsBuffers", "OverlapInfeasibleError", "Pe", "ProblemShape",
    "RangeError", "RankCtx", "SYNC_TOKEN", "SYNC_WAIT", "ShmemError", "SignalSet", "SymHandle",
    "SynchronizationFault", "TileSchedule", "TileStep", "UsageError", "World", "WorldSpec",
    "ag_gemm", "ag_order_fullmesh", "ag_order_switch", "exchange_ipc_handles", "gemm",
    "gemm_rs", "init_world", "init_world_dist", "make_ag_gemm_buffers", "make_gemm_rs_buffers",
    "rs_inter_order", "ChunkLayout", "allgather_pull_intra", "allgather_push_intra",
    "reducescatter_push_intra", "SignalOp", "Token", "WaitCond", "consume_token",
]

__version__ = "0.1.0"
