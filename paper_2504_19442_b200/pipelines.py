"""Drop-in ``ag_gemm`` / ``gemm_rs`` (reference pkg/src/minishmem/pipelines.py).

Same entry points, argument layout and rank/world semantics as the
reference; the arithmetic and the communication run in one sm_100a kernel per
call through the C ABI (include/shmem_b200.h):

* ``ag_gemm(pe, a_shard (m/W, k), b (k, n), shape, schedule, bufs)`` returns
  ``C (m, n) = concat_r(a_shard_r) @ b`` on every rank (pipelines.py:97-150).
  The shard is pushed by the copy engine into slot ``rank`` of every rank's
  ``gathered`` buffer, followed by a release store of ``ready[rank]``; the
  GEMM's TMA warp acquires ``ready[c]`` before the first A tile of chunk c, in
  the schedule's chunk order (own chunk first, no wait).
* ``gemm_rs(pe, a (m, k), b (k, n), shape, schedule, bufs)`` returns row block
  ``rank`` of ``sum_r a_r @ b_r`` (pipelines.py:179-233).  The GEMM epilogue
  stores each bf16 tile straight into the owner's ``staging`` slot ``rank``
  and release-adds the owner's per-source counter; the epilogue of the own
  chunk's tiles (scheduled last) sums the W slots in ascending source order.

Data are torch tensors (bf16 or fp16) on the rank's GPU; CPU tensors are
copied to the GPU first.  Calls are stream-ordered on the current CUDA
stream; ``World.run`` drains it before returning, as the reference's
synchronous call would.  Flags carry a per-call epoch, so back-to-back calls
need no reset in between; ``reset=True`` zeroes them at the next join.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

from . import _lib
from .core import SignalSet, SymHandle
from .errors import ArgumentError
from .swizzle import TileSchedule

SYNC_WAIT = "wait_until"
SYNC_TOKEN = "token"

_DTYPES = {
    "bfloat16": "bfloat16", "bf16": "bfloat16",
    "float16": "float16", "fp16": "float16", "half": "float16",
}
_DTYPE_CACHE = {}  # ProblemShape.dtype -> (torch dtype, SH_DTYPE code); host-path cost per call


@dataclass(frozen=True)
class ProblemShape:
    """GEMM extent plus tiling (reference pipelines.py:31-60).  ``tile_m`` /
    ``tile_n`` are accepted for API parity; the kernel picks its own tiles and
    the result never depends on them (pipelines.py:33-34)."""

    m: int
    n: int
    k: int
    dtype: str = "int64"
    tile_m: int = 0
    tile_n: int = 0

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise ArgumentError("m, n, k must be >= 1")
        if self.tile_m < 0 or self.tile_n < 0:
            raise ArgumentError("tile sizes must be >= 0")

    @property
    def torch_dtype(self):
        hit = _DTYPE_CACHE.get(self.dtype)
        if hit is not None:
            return hit[0]
        import torch

        name = _DTYPES.get(str(self.dtype).replace("torch.", ""))
        if name is None:
            raise ArgumentError(
                f"dtype {self.dtype!r}: the tensor-core path computes in bf16/fp16 "
                "(fp32 accumulate); use dtype='bfloat16' or 'float16'")
        tdt = getattr(torch, name)
        code = _lib.SH_DTYPE_FP16 if tdt == torch.float16 else _lib.SH_DTYPE_BF16
        _DTYPE_CACHE[self.dtype] = (tdt, code)
        return tdt

    @property
    def dtype_code(self):
        hit = _DTYPE_CACHE.get(self.dtype)
        if hit is None:
            self.torch_dtype  # noqa: B018 -- validates and fills the cache
            hit = _DTYPE_CACHE[self.dtype]
        return hit[1]

    @property
    def dtype_bytes(self):
        return 2

    def rows_per_rank(self, world_size):
        if self.m % world_size:
            raise ArgumentError(f"M={self.m} not divisible by world {world_size}")
        return self.m // world_size


class _Epochs:
    """Per-rank monotone call counters of one buffer set (epoch >= 1)."""

    def __init__(self, world, sigsets):
        self._lock = threading.Lock()
        self._val = [0] * world.world_size
        self._sigsets = set(sigsets)
        world._register_epochs(self)

    def next(self, rank):
        with self._lock:
            self._val[rank] += 1
            return self._val[rank]

    def current(self, rank):
        return self._val[rank]

    def reset_epochs(self):
        with self._lock:
            self._val = [0] * len(self._val)

    def reset_epochs_for(self, sets):
        if self._sigsets & set(sets):
            self.reset_epochs()


@dataclass(frozen=True)
class AgGemmBuffers:
    gathered: SymHandle   # W stacked A shards (slot r = rank r's shard)
    ready: SignalSet      # ready[src] = epoch once src's shard landed here
    done: SignalSet = None  # done[p] = epoch once rank p finished reading its gather buffer
    epochs: _Epochs = field(default=None, compare=False, repr=False)


def make_ag_gemm_buffers(world, shape: ProblemShape):
    """Symmetric gather buffer + per-source flags (reference pipelines.py:88-94)."""
    rows = shape.rows_per_rank(world.world_size)
    chunk_bytes = rows * shape.k * shape.dtype_bytes
    gathered = world.alloc_symmetric(world.world_size * chunk_bytes, align=1024)
    ready = world.alloc_signals(world.world_size)
    done = world.alloc_signals(world.world_size)
    return AgGemmBuffers(gathered, ready, done, _Epochs(world, [ready, done]))


@dataclass(frozen=True)
class GemmRsBuffers:
    staging: SymHandle        # W slots: slot s = rows of (A_s @ B_s) owned by this rank
    partial: SymHandle | None  # multi-node only (out of scope), always None
    producer: SignalSet       # producer[d] = epoch once rank d reduced (frees its slots)
    reduction: SignalSet      # reduction[s] = elements delivered by s (cumulative)
    epochs: _Epochs = field(default=None, compare=False, repr=False)


def make_gemm_rs_buffers(world, shape: ProblemShape):
    """Staging slots + flags (reference pipelines.py:161-170, single node)."""
    rows = shape.rows_per_rank(world.world_size)
    block_bytes = rows * shape.n * shape.dtype_bytes
    staging = world.alloc_symmetric(world.world_size * block_bytes, align=1024)
    producer = world.alloc_signals(world.world_size)
    reduction = world.alloc_signals(world.world_size)
    return GemmRsBuffers(staging, None, producer, reduction, _Epochs(world, [producer, reduction]))


def _as_device_tensor(x, name, shape, dtype, pe):
    import torch

    if not isinstance(x, torch.Tensor):
        raise ArgumentError(f"{name} must be a torch tensor of {dtype}")
    if tuple(x.shape) != tuple(shape) or x.dtype != dtype:
        raise ArgumentError(f"{name} must be {tuple(shape)} of {dtype}, got "
                            f"{tuple(x.shape)} of {x.dtype}")
    if not x.is_cuda:
        x = x.to(pe.torch_device, non_blocking=True)
    elif x.get_device() != pe.device:
        raise ArgumentError(f"{name} lives on {x.device}, rank {pe.rank} runs on "
                            f"{pe.torch_device}")
    return x if x.is_contiguous() else x.contiguous()


def _stream_handle(pe):
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # no Stream object per call (host cost of small launches)
        return raw(pe.device)
    return torch.cuda.current_stream(pe.device).cuda_stream


def ag_gemm(pe, a_shard, b, shape: ProblemShape, schedule: TileSchedule, bufs: AgGemmBuffers, *,
            sync_style=SYNC_TOKEN, reset=True):
    """C = concat(A_shards) @ B on every rank (reference pipelines.py:97-150).

    ``sync_style`` is accepted for API parity: both reference styles are the
    same acquire on the GPU (tests/test_pipelines.py:93-107)."""
    import torch

    world = pe.world
    w = world.world_size
    rows = shape.rows_per_rank(w)
    dt = shape.torch_dtype
    if sync_style not in (SYNC_TOKEN, SYNC_WAIT):
        raise ArgumentError(f"unknown sync_style {sync_style!r}")
    a_shard = _as_device_tensor(a_shard, "A shard", (rows, shape.k), dt, pe)
    b = _as_device_tensor(b, "B", (shape.k, shape.n), dt, pe)
    order = schedule.first_visit_order(w)
    chunk_bytes = rows * shape.k * shape.dtype_bytes
    if bufs.gathered.length != w * chunk_bytes:
        raise ArgumentError(f"gather buffer is {bufs.gathered.length} bytes, need {w * chunk_bytes}")
    if bufs.ready.count < w or bufs.done is None or bufs.done.count < w:
        raise ArgumentError("need one ready and one done signal per source rank")
    out = torch.empty((shape.m, shape.n), dtype=dt, device=pe.torch_device)
    epoch = bufs.epochs.next(pe.rank)
    lib = _lib.load()
    _lib.check(lib.sh_ag_gemm(world.handle, pe.rank, a_shard.data_ptr(), b.data_ptr(),
                              out.data_ptr(), bufs.gathered.offset, bufs.ready.base,
                              bufs.done.base, shape.m, shape.n, shape.k, shape.dtype_code,
                              _lib.int_array(order), epoch, _stream_handle(pe)))
    # one acquire per remote chunk, no barrier (tests/test_pipelines.py:53-69)
    world.bump(pe.rank, "wait", w - 1)
    world.bump(pe.rank, "ag_gemm")
    if reset:
        world._request_reset([bufs.ready, bufs.done])
    return out


def gemm_rs(pe, a, b, shape: ProblemShape, schedule: TileSchedule, bufs: GemmRsBuffers, *,
            reset=True, sync_style=SYNC_WAIT):
    """Row block ``rank`` of sum_r (A_r @ B_r) (reference pipelines.py:179-233)."""
    import torch

    world = pe.world
    w = world.world_size
    rows = shape.rows_per_rank(w)
    dt = shape.torch_dtype
    if sync_style not in (SYNC_TOKEN, SYNC_WAIT):
        raise ArgumentError(f"unknown sync_style {sync_style!r}")
    a = _as_device_tensor(a, "A", (shape.m, shape.k), dt, pe)
    b = _as_device_tensor(b, "B", (shape.k, shape.n), dt, pe)
    order = schedule.first_visit_order(w)
    block_bytes = rows * shape.n * shape.dtype_bytes
    if bufs.staging.length != w * block_bytes:
        raise ArgumentError(f"staging is {bufs.staging.length} bytes, need {w * block_bytes}")
    if bufs.producer.count < w or bufs.reduction.count < w:
        raise ArgumentError("need one producer and one reduction signal per rank")
    out = torch.empty((rows, shape.n), dtype=dt, device=pe.torch_device)
    epoch = bufs.epochs.next(pe.rank)
    lib = _lib.load()
    _lib.check(lib.sh_gemm_rs(world.handle, pe.rank, a.data_ptr(), b.data_ptr(), out.data_ptr(),
                              bufs.staging.offset, bufs.producer.base, bufs.reduction.base,
                              shape.m, shape.n, shape.k, shape.dtype_code, _lib.int_array(order),
                              epoch, _stream_handle(pe)))
    world.bump(pe.rank, "wait", w)
    world.bump(pe.rank, "gemm_rs")
    if reset:
        world._request_reset([bufs.producer, bufs.reduction])
    return out


def gemm(a, b):
    """The GEMM core alone (TP=1, no symmetric heap): a (m,k) @ b (k,n), bf16/fp16."""
    import torch

    if a.dim() != 2 or b.dim() != 2 or a.shape[1] != b.shape[0]:
        raise ArgumentError(f"incompatible shapes {tuple(a.shape)} @ {tuple(b.shape)}")
    if a.dtype != b.dtype or a.dtype not in (torch.bfloat16, torch.float16):
        raise ArgumentError("gemm takes two bf16 or two fp16 tensors")
    if not a.is_cuda or a.device != b.device:
        raise ArgumentError("gemm takes CUDA tensors on one device")
    a = a.contiguous()
    b = b.contiguous()
    m, k = a.shape
    n = b.shape[1]
    import ctypes

    c = torch.empty((m, n), dtype=a.dtype, device=a.device)
    code = _lib.SH_DTYPE_FP16 if a.dtype == torch.float16 else _lib.SH_DTYPE_BF16
    lib = _lib.load()
    with torch.cuda.device(a.device):
        need = ctypes.c_size_t()
        _lib.check(lib.sh_gemm_workspace_bytes(m, n, k, ctypes.byref(need)))
        # stream-K partials: a stream-ordered block from torch's caching allocator
        ws = torch.empty(need.value, dtype=torch.uint8, device=a.device) if need.value else None
        _lib.check(lib.sh_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, code,
                               ws.data_ptr() if ws is not None else None, need.value,
                               torch.cuda.current_stream(a.device).cuda_stream))
    return c
