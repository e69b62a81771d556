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

Data are torch tensors (bf16 or fp16) on the rank's GPU -- the hot path --, or
numpy arrays / CPU tensors of the ProblemShape's dtype (the reference's
int64 default included, when exact in bf16), which are staged on the device
and answered in kind.  Calls are stream-ordered on the current CUDA
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

# compute types of the tensor-core path
_COMPUTE = {
    "bfloat16": "bfloat16", "bf16": "bfloat16",
    "float16": "float16", "fp16": "float16", "half": "float16",
}
# caller-side element types the drop-in also accepts (the reference's default
# is int64): operands are staged in bf16 when that is exact, results are
# handed back in the caller's type (see _HostIO)
_WIDENED = ("int64", "int32", "int16", "int8", "uint8", "float32", "float64")
_DTYPE_CACHE = {}  # ProblemShape.dtype -> (torch compute dtype, SH_DTYPE code); host cost per call


def _dtype_name(dtype):
    name = str(dtype).replace("torch.", "")
    if name in _COMPUTE or name in _WIDENED:
        return name
    try:
        import numpy as np

        return np.dtype(dtype).name
    except Exception:  # noqa: BLE001
        return name


@dataclass(frozen=True)
class ProblemShape:
    """GEMM extent plus tiling (reference pipelines.py:31-60).  ``tile_m`` /
    ``tile_n`` are accepted for API parity; the kernel picks its own tiles and
    the result never depends on them (pipelines.py:33-34).

    ``dtype`` is the caller's element type.  bf16 / fp16 are computed as is;
    the reference's int64 default and the other integer / float types are
    accepted when every operand value is exactly representable in bf16 (the
    tensor cores' input type) and come back in the caller's type."""

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
    def io_dtype(self):
        """Element type name the caller passes and gets back."""
        hit = _DTYPE_CACHE.get(self.dtype)
        if hit is not None:
            return hit[2]
        name = _dtype_name(self.dtype)
        if name not in _COMPUTE and name not in _WIDENED:
            raise ArgumentError(
                f"dtype {self.dtype!r}: the tensor-core path computes in bf16/fp16 "
                f"(fp32 accumulate) and accepts {', '.join(_WIDENED)} when exact in bf16")
        return _COMPUTE.get(name, name)

    @property
    def widened(self):
        """True when the caller's type is not the compute type (int64 etc.)."""
        hit = _DTYPE_CACHE.get(self.dtype)
        if hit is not None:
            return hit[3]
        return self.io_dtype in _WIDENED

    @property
    def torch_dtype(self):
        """The compute dtype (bf16 unless the caller asked for fp16)."""
        hit = _DTYPE_CACHE.get(self.dtype)
        if hit is not None:
            return hit[0]
        import torch

        name = self.io_dtype
        tdt = torch.float16 if name == "float16" else torch.bfloat16
        code = _lib.SH_DTYPE_FP16 if tdt == torch.float16 else _lib.SH_DTYPE_BF16
        _DTYPE_CACHE[self.dtype] = (tdt, code, name, name in _WIDENED)
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
        """Bytes per element in the symmetric buffers (the compute type)."""
        return 2

    @property
    def k_padded(self):
        """K as laid out in device memory: TMA rows are 16-byte multiples, so
        a ragged K is zero-padded to a multiple of 8 (exact: zeros add 0)."""
        return -(-self.k // 8) * 8

    @property
    def n_padded(self):
        return -(-self.n // 8) * 8

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
    chunk_bytes = rows * shape.k_padded * shape.dtype_bytes
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
    block_bytes = rows * shape.n_padded * shape.dtype_bytes
    staging = world.alloc_symmetric(world.world_size * block_bytes, align=1024)
    producer = world.alloc_signals(world.world_size)
    reduction = world.alloc_signals(world.world_size)
    return GemmRsBuffers(staging, None, producer, reduction, _Epochs(world, [producer, reduction]))


class _HostIO:
    """Operand staging of one call.

    * torch bf16/fp16 CUDA tensors of the compute type pass through (the hot
      path: no copy, no host work beyond the checks);
    * numpy arrays and CPU tensors are uploaded from pinned memory on the
      rank's stream, and the call's result goes back to the host in the same
      container (the reference returns a fresh numpy array, pipelines.py:116);
    * a widened ProblemShape dtype (int64 -- the reference default --,
      float32, ...) is staged in bf16; every value must be exactly
      representable there, else ArgumentError.  Integer results come back
      exact or not at all: the partial sums of fp32 accumulation stay below
      2**24 (checked on the operands) and every bf16-rounded value the result
      passes through is
      certified to lie within bf16's contiguous integer range |x| <= 256
      (gemm_rs: the staging slots through k*max|A|*max|B| <= 256, the output
      after the call).
    * a ragged n or k (not a multiple of 8) is zero-padded on the device."""

    def __init__(self, pe, shape: ProblemShape):
        self.pe = pe
        self.shape = shape
        self.host = False      # hand the result back in host memory
        self.numpy = False     # ... as a numpy array (else a CPU tensor)
        self.widened = shape.widened
        self.amax = {}         # operand name -> max |value| (integer certificates)

    def operand(self, x, name, rows, cols, pad_rows=False):
        import numpy as np
        import torch

        shape = self.shape
        dt = shape.torch_dtype
        if (type(x) is torch.Tensor and x.dtype == dt and x.is_cuda and not self.widened
                and rows % 8 == 0 and cols % 8 == 0):
            # hot path: the compute dtype already on the GPU
            if x.shape[0] != rows or x.shape[1] != cols or x.dim() != 2:
                raise ArgumentError(f"{name} must be {(rows, cols)} of {shape.io_dtype}, got "
                                    f"{tuple(x.shape)} of {str(x.dtype).replace('torch.', '')}")
            if x.get_device() != self.pe.device:
                raise ArgumentError(f"{name} lives on {x.device}, rank {self.pe.rank} runs on "
                                    f"{self.pe.torch_device}")
            return x if x.is_contiguous() else x.contiguous()
        want_rows = rows
        if isinstance(x, np.ndarray):
            self.host = True
            self.numpy = True
            if x.shape != (rows, cols) or np.dtype(x.dtype).name != shape.io_dtype:
                raise ArgumentError(f"{name} must be {(rows, cols)} of {shape.io_dtype}, got "
                                    f"{x.shape} of {x.dtype}")
            x = torch.from_numpy(np.ascontiguousarray(x))
        elif isinstance(x, torch.Tensor):
            tname = str(x.dtype).replace("torch.", "")
            if tuple(x.shape) != (rows, cols) or tname != shape.io_dtype:
                raise ArgumentError(f"{name} must be {(rows, cols)} of {shape.io_dtype}, got "
                                    f"{tuple(x.shape)} of {tname}")
            if x.is_cuda and x.get_device() != self.pe.device:
                raise ArgumentError(f"{name} lives on {x.device}, rank {self.pe.rank} runs on "
                                    f"{self.pe.torch_device}")
            if not x.is_cuda:
                self.host = True
        else:
            raise ArgumentError(f"{name} must be a numpy array or torch tensor of "
                                f"{shape.io_dtype}")
        if self.widened:
            x = self._narrow(x, name)
        if not x.is_cuda:
            x = x.contiguous().pin_memory().to(self.pe.torch_device, non_blocking=True)
        elif x.dtype != dt:
            x = x.to(dt)
        if pad_rows and want_rows % 8:
            x = torch.nn.functional.pad(x, (0, 0, 0, -(-want_rows // 8) * 8 - want_rows))
        if cols % 8:
            x = torch.nn.functional.pad(x, (0, -(-cols // 8) * 8 - cols))
        return x if x.is_contiguous() else x.contiguous()

    def _narrow(self, x, name):
        """bf16 copy of a widened operand, refusing values bf16 cannot hold."""
        import torch

        if x.is_cuda:
            t = x.to(torch.bfloat16)
            bad = (t.to(x.dtype) != x).any() if x.numel() else torch.zeros((), dtype=torch.bool,
                                                                            device=x.device)
            amax = x.abs().max().double() if x.numel() else torch.zeros((), dtype=torch.float64,
                                                                        device=x.device)
            flags = torch.stack([bad.double(), amax]).to("cpu", non_blocking=True)
            torch.cuda.current_stream(self.pe.device).synchronize()
            bad_v, amax_v = bool(flags[0]), float(flags[1])
        else:
            t = x.to(torch.bfloat16)
            bad_v = bool((t.to(x.dtype) != x).any()) if x.numel() else False
            amax_v = float(x.abs().max()) if x.numel() else 0.0
        if bad_v:
            raise ArgumentError(
                f"{name}: {self.shape.io_dtype} values not exactly representable in bf16 (the "
                "tensor cores' input type); pass bf16 data with dtype='bfloat16'")
        if not self.shape.io_dtype.startswith("float"):
            self.amax[name] = amax_v
            # fp32 accumulation is exact while every partial sum < 2**24 (the
            # other operand is bounded by 256, enforced by its owner's check)
            if self.shape.k * amax_v * 256.0 >= 2.0 ** 24:
                raise ArgumentError(
                    f"{name}: k={self.shape.k} x max|value| {amax_v:g} could leave fp32's exact "
                    "integer range in the accumulator")
            if amax_v > 256:
                raise ArgumentError(f"{name}: integer operands must lie in [-256, 256] "
                                    "(exact products in bf16)")
        return t

    def prepare(self, out):
        """Everything that may block the host thread or allocate pinned
        memory happens before the collective is issued (see World.run: a
        page-locked allocation or a pageable copy on one rank thread can wait
        for a sibling rank's kernel that spins on a flag this thread has not
        yet released).  Then, with several ranks in this process, a host
        rendezvous: no rank issues the collective before every rank staged."""
        import torch

        if self.host:
            self.pinned = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        elif self.widened and not self.shape.io_dtype.startswith("float"):
            self.chk = torch.empty((1,), dtype=torch.float32, pin_memory=True)
        world = self.pe.world
        if (self.host or self.widened) and len(world.local_ranks) > 1:
            world._host_join(self.pe)

    def output(self, out):
        """The call's result for the caller: without the padding, in the
        caller's type and container."""
        import numpy as np
        import torch

        shape = self.shape
        integer = self.widened and not shape.io_dtype.startswith("float")
        if self.host:
            self.pinned.copy_(out, non_blocking=True)
            torch.cuda.current_stream(self.pe.device).synchronize()
            arr = self.pinned[:, :shape.n].float().numpy()
            if integer and arr.size and float(np.abs(arr).max()) > 256:
                self._not_exact(float(np.abs(arr).max()))
            if self.numpy:
                return arr.astype(shape.io_dtype if self.widened else np.float32)
            if self.widened:
                return torch.from_numpy(arr.astype(shape.io_dtype))
            return self.pinned[:, :shape.n].clone()
        res = out[:, :shape.n] if out.shape[1] != shape.n else out
        if not self.widened:
            return res
        if integer:
            # integer certificate: the output's bf16 rounding was exact
            self.chk.copy_(res.abs().max().float().reshape(1), non_blocking=True)
            torch.cuda.current_stream(self.pe.device).synchronize()
            if float(self.chk[0]) > 256:
                self._not_exact(float(self.chk[0]))
        return res.to(getattr(torch, shape.io_dtype))

    @staticmethod
    def _not_exact(peak):
        raise ArgumentError(
            f"integer result reaches {peak:g}: beyond bf16's exact integer range (|x| <= 256) "
            "the product is rounded; use dtype='bfloat16'")


def _check_out(out, rows, cols, dt, pe, io):
    import torch

    if io.host or io.widened:
        raise ArgumentError("out= takes CUDA operands of the compute dtype (bf16/fp16); "
                            "host / widened calls return a fresh result")
    if not isinstance(out, torch.Tensor) or not out.is_cuda:
        raise ArgumentError("out must be a CUDA tensor")
    if tuple(out.shape) != (rows, cols) or out.dtype != dt or not out.is_contiguous():
        raise ArgumentError(f"out must be a contiguous {(rows, cols)} tensor of {dt}, got "
                            f"{tuple(out.shape)} of {out.dtype}")
    if out.get_device() != pe.device:
        raise ArgumentError(f"out lives on {out.device}, rank {pe.rank} runs on {pe.torch_device}")
    return out


def _stream_handle(pe):
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:  # no Stream object per call (host cost of small launches)
        return raw(pe.device)
    return torch.cuda.current_stream(pe.device).cuda_stream


def ag_gemm(pe, a_shard, b, shape: ProblemShape, schedule: TileSchedule, bufs: AgGemmBuffers, *,
            sync_style=SYNC_TOKEN, reset=True, out=None):
    """C = concat(A_shards) @ B on every rank (reference pipelines.py:97-150).

    ``sync_style`` is accepted for API parity: both reference styles are the
    same acquire on the GPU (tests/test_pipelines.py:93-107).  ``out`` (B200
    extension): a preallocated contiguous (m, n) CUDA tensor of the compute
    dtype to write C into, so a steady loop allocates nothing."""
    import torch

    world = pe.world
    w = world.world_size
    rows = shape.rows_per_rank(w)
    dt = shape.torch_dtype
    if sync_style not in (SYNC_TOKEN, SYNC_WAIT):
        raise ArgumentError(f"unknown sync_style {sync_style!r}")
    io = _HostIO(pe, shape)
    a_shard = io.operand(a_shard, "A shard", rows, shape.k)
    b = io.operand(b, "B", shape.k, shape.n, pad_rows=True)
    kp, np_ = shape.k_padded, shape.n_padded
    order = schedule.first_visit_order(w)
    chunk_bytes = rows * kp * shape.dtype_bytes
    if bufs.gathered.length != w * chunk_bytes:
        raise ArgumentError(f"gather buffer is {bufs.gathered.length} bytes, need {w * chunk_bytes}")
    if bufs.ready.count < w or bufs.done is None or bufs.done.count < w:
        raise ArgumentError("need one ready and one done signal per source rank")
    if out is not None:
        _check_out(out, shape.m, shape.n, dt, pe, io)
    c = out if out is not None and np_ == shape.n else torch.empty((shape.m, np_), dtype=dt,
                                                                   device=pe.torch_device)
    io.prepare(c)
    epoch = bufs.epochs.next(pe.rank)
    lib = _lib.load()
    args = (world.handle, pe.rank, a_shard.data_ptr(), b.data_ptr(), c.data_ptr(),
            bufs.gathered.offset, bufs.ready.base, bufs.done.base, shape.m, np_, kp,
            shape.dtype_code, _lib.int_array(order), epoch, 0)
    if world.phased:
        # kernel-serialising tool attached: pushes, join, then the GEMM
        _lib.check(lib.sh_ag_gemm_ex(*args, _lib.SH_PHASE_COMM, _stream_handle(pe)))
        world._phase_join(pe)
        _lib.check(lib.sh_ag_gemm_ex(*args, _lib.SH_PHASE_COMPUTE, _stream_handle(pe)))
    else:
        _lib.check(lib.sh_ag_gemm_ex(*args, _lib.SH_PHASE_ALL, _stream_handle(pe)))
    # one acquire per remote chunk, no barrier (tests/test_pipelines.py:53-69)
    world.bump(pe.rank, "wait", w - 1)
    world.bump(pe.rank, "ag_gemm")
    if reset:
        world._request_reset([bufs.ready, bufs.done])
    if out is not None:
        if c is not out:
            out.copy_(c[:, :shape.n])
        return out
    return io.output(c)


def gemm_rs(pe, a, b, shape: ProblemShape, schedule: TileSchedule, bufs: GemmRsBuffers, *,
            reset=True, sync_style=SYNC_WAIT, out=None):
    """Row block ``rank`` of sum_r (A_r @ B_r) (reference pipelines.py:179-233).

    ``out`` (B200 extension): a preallocated contiguous (m/W, n) CUDA tensor
    of the compute dtype for the reduced rows."""
    import torch

    world = pe.world
    w = world.world_size
    rows = shape.rows_per_rank(w)
    dt = shape.torch_dtype
    if sync_style not in (SYNC_TOKEN, SYNC_WAIT):
        raise ArgumentError(f"unknown sync_style {sync_style!r}")
    io = _HostIO(pe, shape)
    a = io.operand(a, "A", shape.m, shape.k)
    b = io.operand(b, "B", shape.k, shape.n, pad_rows=True)
    kp, np_ = shape.k_padded, shape.n_padded
    order = schedule.first_visit_order(w)
    block_bytes = rows * np_ * shape.dtype_bytes
    if bufs.staging.length != w * block_bytes:
        raise ArgumentError(f"staging is {bufs.staging.length} bytes, need {w * block_bytes}")
    if bufs.producer.count < w or bufs.reduction.count < w:
        raise ArgumentError("need one producer and one reduction signal per rank")
    if io.widened and not shape.io_dtype.startswith("float"):
        # every contribution is rounded to bf16 in its staging slot before the
        # reduction: certify the slots from the local operands
        slot_bound = shape.k * io.amax["A"] * io.amax["B"]
        if slot_bound > 256:
            raise ArgumentError(
                f"integer contributions up to k*max|A|*max|B| = {slot_bound:g} exceed bf16's "
                "exact integer range (|x| <= 256) in the staging slots; use dtype='bfloat16'")
    if out is not None:
        _check_out(out, rows, shape.n, dt, pe, io)
    y = out if out is not None and np_ == shape.n else torch.empty((rows, np_), dtype=dt,
                                                                   device=pe.torch_device)
    io.prepare(y)
    epoch = bufs.epochs.next(pe.rank)
    lib = _lib.load()
    args = (world.handle, pe.rank, a.data_ptr(), b.data_ptr(), y.data_ptr(),
            bufs.staging.offset, bufs.producer.base, bufs.reduction.base, shape.m, np_, kp,
            shape.dtype_code, _lib.int_array(order), epoch)
    if world.phased:
        # kernel-serialising tool attached: scatter, join, then the reduction
        _lib.check(lib.sh_gemm_rs_ex(*args, _lib.SH_PHASE_COMM, _stream_handle(pe)))
        world._phase_join(pe)
        _lib.check(lib.sh_gemm_rs_ex(*args, _lib.SH_PHASE_COMPUTE, _stream_handle(pe)))
    else:
        _lib.check(lib.sh_gemm_rs_ex(*args, _lib.SH_PHASE_ALL, _stream_handle(pe)))
    world.bump(pe.rank, "wait", w)
    world.bump(pe.rank, "gemm_rs")
    if reset:
        world._request_reset([bufs.producer, bufs.reduction])
    if out is not None:
        if y is not out:
            out.copy_(y[:, :shape.n])
        return out
    return io.output(y)


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
