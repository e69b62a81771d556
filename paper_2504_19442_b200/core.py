"""World construction and the GPU symmetric heap (hot-path subsystem 1).

Same geometry and addressing as the reference (pkg/src/minishmem/core.py):
every rank owns a slab of ``heap_bytes + 8*signal_count`` bytes, a symmetric
handle is an (offset, length) valid in every slab, and signal ``sig`` is the
u64 at ``slab + heap_bytes + 8*sig`` (core.py:159-160, 242-261).  The slabs
are device memory: in one process every rank's slab is peer-mapped into every
other rank's GPU (NVLink / NVSwitch); across processes (torchrun, one rank per
GPU) the slabs are exchanged with CUDA IPC handles.  All of it lives in the C
ABI (``_lib``); this module is the Python mirror of the reference's World.

Two ways to build a world:

* ``init_world(WorldSpec(world_size=W))`` -- the reference's model: all ranks
  are threads of this process, ``world.run(fn)`` calls ``fn(pe)`` once per rank
  concurrently and returns the per-rank results (core.py:449-487).  Rank r uses
  GPU ``devices[r]`` (default ``r % torch.cuda.device_count()``), so W ranks may
  share one GPU (each rank gets its own CUDA stream).
* ``init_world_dist(...)`` -- one process per GPU under torch.distributed;
  ``run(fn)`` executes this process's rank only.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading
from collections import deque
from dataclasses import dataclass

from . import _lib
from .errors import (
    ArgumentError,
    CollectiveFault,
    ConfigurationError,
    RangeError,
    ShmemError,
    SynchronizationFault,
    UsageError,
)

SIG_BYTES = 8


@dataclass(frozen=True)
class WorldSpec:
    """Rank geometry plus per-rank slab sizing (reference core.py:35-66).

    ``devices`` (B200 extension) pins rank r to GPU ``devices[r]``."""

    world_size: int
    n_nodes: int = 1
    local_world_size: int | None = None
    heap_bytes: int = 1 << 20
    signal_count: int | None = None
    timeout_s: float = 5.0
    devices: tuple | None = None

    def __post_init__(self):
        lws = self.local_world_size
        if lws is None:
            if self.n_nodes < 1 or self.world_size % self.n_nodes:
                raise ConfigurationError(
                    f"world_size {self.world_size} not divisible by n_nodes {self.n_nodes}")
            lws = self.world_size // self.n_nodes
            object.__setattr__(self, "local_world_size", lws)
        if self.world_size < 1 or self.n_nodes < 1 or lws < 1:
            raise ConfigurationError("world_size, n_nodes, local_world_size must be >= 1")
        if self.world_size != self.n_nodes * lws:
            raise ConfigurationError(
                f"world_size {self.world_size} != n_nodes {self.n_nodes} x local {lws}")
        if self.heap_bytes <= 0:
            raise ConfigurationError("heap_bytes must be > 0")
        if self.signal_count is None:
            object.__setattr__(self, "signal_count", max(4 * self.world_size, 64))
        if self.signal_count < self.world_size:
            raise ConfigurationError("signal_count must be >= world_size")
        if self.timeout_s <= 0:
            raise ConfigurationError("timeout_s must be > 0")
        if self.devices is not None:
            devs = tuple(int(d) for d in self.devices)
            if len(devs) != self.world_size:
                raise ConfigurationError("devices must name one GPU per rank")
            object.__setattr__(self, "devices", devs)


@dataclass(frozen=True)
class RankCtx:
    rank: int
    node_id: int
    local_rank: int


@dataclass(frozen=True)
class SymHandle:
    """Rank-independent (offset, length) into every rank's slab."""

    offset: int
    length: int

    def check(self, off, nbytes):
        if off < 0 or nbytes < 0 or off + nbytes > self.length:
            raise RangeError(f"access [{off}, {off + nbytes}) outside handle of {self.length} bytes")


@dataclass(frozen=True)
class SignalSet:
    """Contiguous signal words in the symmetric pad."""

    base: int
    count: int

    def at(self, i):
        if i < 0 or i >= self.count:
            raise ArgumentError(f"signal index {i} out of {self.count}")
        return self.base + i


class Pe:
    """A rank bound to its world, GPU and stream (reference primitives.py:76-96)."""

    def __init__(self, world, ctx: RankCtx, device: int):
        self.world = world
        self.ctx = ctx
        self.rank = ctx.rank
        self.device = device
        self._stream = None

    @property
    def torch_device(self):
        dev = self.__dict__.get("_tdev")
        if dev is None:
            import torch

            dev = self._tdev = torch.device("cuda", self.device)
        return dev

    def stream(self):
        """This rank's CUDA stream (one per rank, so ranks sharing a GPU run
        concurrently)."""
        import torch

        if self._stream is None:
            self._stream = torch.cuda.Stream(device=self.device)
        return self._stream

    def barrier_all(self):
        """Host-side rendezvous of every rank (plus device drain)."""
        self.world.bump(self.rank, "barrier_all")
        self.world._barrier(self)

    def sync_all(self):
        """Barrier without the completion reading of the reference (core.py:
        sync_all); on the GPU the drain makes both the same."""
        self.world.bump(self.rank, "sync_all")
        self.world._barrier(self)

    def quiet(self):
        """Complete this rank's outstanding transfers (reference primitives.py
        quiet): every put/get is stream-ordered, so drain the current stream."""
        import torch

        self.world.bump(self.rank, "quiet")
        torch.cuda.current_stream(self.device).synchronize()

    def my_pe(self):
        return self.rank

    def n_pes(self):
        return self.world.world_size

    def remote_ptr(self, handle: SymHandle, peer, off=0, nbytes=None):
        """Zero-copy CUDA uint8 view of ``peer``'s replica of ``handle``, mapped
        into this rank's GPU (NVLink loads/stores; reference remote_ptr)."""
        import torch

        self._check_peer(peer)
        n = handle.length - off if nbytes is None else nbytes
        return self.world.heap_view(self.rank, handle, torch.uint8, (n,), off=off, peer=peer)

    # ------------------------------------------------------------------
    # one-sided primitives (reference primitives.py:126-257), stream-ordered

    def _stream_handle(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def _payload(self, src, src_off=0, nbytes=None):
        """Device bytes of ``src`` (bytes / numpy / torch tensor)."""
        import numpy as np
        import torch

        if isinstance(src, torch.Tensor):
            t = src.contiguous().view(-1).view(torch.uint8)
        else:
            buf = src.tobytes() if isinstance(src, np.ndarray) else bytes(src)
            t = torch.frombuffer(bytearray(buf), dtype=torch.uint8) if buf else \
                torch.empty(0, dtype=torch.uint8)
        n = t.numel() - src_off if nbytes is None else nbytes
        if src_off < 0 or n < 0 or src_off + n > t.numel():
            raise RangeError(f"source range [{src_off}, {src_off + n}) outside {t.numel()} bytes")
        t = t[src_off:src_off + n]
        if t.device.type != "cuda":
            t = t.to(self.torch_device)
        return t

    def _check_peer(self, peer):
        if peer < 0 or peer >= self.world.world_size:
            raise ArgumentError(f"peer {peer} out of range (world {self.world.world_size})")

    def _check_sig(self, sig):
        if sig < 0 or sig >= self.world.spec.signal_count:
            raise ArgumentError(f"signal {sig} out of pad of {self.world.spec.signal_count}")

    def putmem(self, dst: SymHandle, src, peer, *, nbytes=None, dst_off=0, src_off=0):
        """Copy ``src`` into ``peer``'s replica of ``dst`` (copy engine, NVLink)."""
        self._check_peer(peer)
        payload = self._payload(src, src_off, nbytes)
        dst.check(dst_off, payload.numel())
        self.world.bump(self.rank, "putmem")
        _lib.check(self.world._lib.sh_putmem(self.world.handle, self.rank, peer,
                                             dst.offset + dst_off, payload.data_ptr(),
                                             payload.numel(), self._stream_handle()))
        return payload  # keep alive until the caller's stream passes the copy

    def putmem_signal(self, dst: SymHandle, src, sig, value, peer, *, op=None, nbytes=None,
                      dst_off=0, src_off=0):
        """putmem followed by a signal on ``peer`` that is ordered after the data
        (same stream; the stream write carries a memory barrier)."""
        from .primitives import SignalOp

        keep = self.putmem(dst, src, peer, nbytes=nbytes, dst_off=dst_off, src_off=src_off)
        self.signal_op(peer, sig, op or SignalOp.SET, value)
        return keep

    def putmem_nbi(self, dst: SymHandle, src, peer, **kw):
        """Non-blocking put: every put is already stream-ordered and asynchronous."""
        return self.putmem(dst, src, peer, **kw)

    def getmem_nbi(self, dst, src: SymHandle, peer, **kw):
        return self.getmem(dst, src, peer, **kw)

    def getmem(self, dst, src: SymHandle, peer, *, nbytes=None, dst_off=0, src_off=0):
        """Copy ``peer``'s replica of ``src`` into ``dst`` (a CUDA tensor or the
        rank's own replica of a SymHandle)."""
        import torch

        self._check_peer(peer)
        if isinstance(dst, SymHandle):
            n = (dst.length - dst_off) if nbytes is None else nbytes
            dst.check(dst_off, n)
            src.check(src_off, n)
            out_ptr = self.world.heap_ptr(self.rank, dst, dst_off)
        else:
            if not isinstance(dst, torch.Tensor) or not dst.is_cuda:
                raise ArgumentError("getmem destination must be a CUDA tensor or SymHandle")
            flat = dst.view(-1).view(torch.uint8)
            n = (flat.numel() - dst_off) if nbytes is None else nbytes
            if dst_off + n > flat.numel():
                raise RangeError("getmem destination too small")
            src.check(src_off, n)
            out_ptr = flat.data_ptr() + dst_off
        self.world.bump(self.rank, "getmem")
        _lib.check(self.world._lib.sh_getmem(self.world.handle, self.rank, out_ptr, peer,
                                             src.offset + src_off, n, self._stream_handle()))

    def signal_op(self, peer, sig, op, value):
        from .primitives import SignalOp

        self._check_peer(peer)
        self._check_sig(sig)
        self.world.bump(self.rank, "signal_op")
        code = _lib.SH_SIG_SET if op == SignalOp.SET else _lib.SH_SIG_ADD
        _lib.check(self.world._lib.sh_signal_op(self.world.handle, self.rank, peer, sig, code,
                                                int(value), self._stream_handle()))

    def notify(self, peer, sig, value):
        from .primitives import SignalOp

        self.signal_op(peer, sig, SignalOp.SET, value)

    def signal_wait_until(self, sig, cond, value, timeout=None):
        """The rank's stream waits until its own signal satisfies ``cond``."""
        self._check_sig(sig)
        self.world.bump(self.rank, "signal_wait_until")
        _lib.check(self.world._lib.sh_signal_wait(self.world.handle, self.rank, sig, cond.code,
                                                  int(value), self._stream_handle()))
        return value

    def wait(self, sig, value, timeout=None):
        from .primitives import Token, WaitCond

        self.world.bump(self.rank, "wait")
        self.signal_wait_until(sig, WaitCond.EQ, value, timeout=timeout)
        return Token(sig, value)

    def signal_read(self, sig):
        """Current value of the rank's own signal (synchronises the stream)."""
        import torch

        torch.cuda.current_stream(self.device).synchronize()
        return self.world.sig_read(self.rank, sig)

    # ------------------------------------------------------------------
    # node-scope multimem (reference primitives.py:291-315)

    def _node_range(self):
        lws = self.world.local_world_size
        return self.ctx.node_id * lws, lws

    def multimem_st(self, handle: SymHandle, off=0, nbytes=None):
        """Replicate the caller's bytes at ``handle`` into every same-node
        rank's replica (SM-driven NVLink stores, one read of the source)."""
        n = handle.length - off if nbytes is None else nbytes
        handle.check(off, n)
        self.world.bump(self.rank, "multimem_st")
        first, count = self._node_range()
        _lib.check(self.world._lib.sh_multimem_st(self.world.handle, self.rank, first, count,
                                                  handle.offset + off, n, self._stream_handle()))

    def multimem_ld_reduce(self, handle: SymHandle, dtype, off=0, nbytes=None):
        """Element-wise sum of all same-node replicas (ascending rank order,
        numpy ``out += replica`` arithmetic), as a new CUDA tensor."""
        import torch

        tdt, code = _multimem_dtype(dtype)
        esize = torch.empty((), dtype=tdt).element_size()
        n = handle.length - off if nbytes is None else nbytes
        handle.check(off, n)
        if n % esize:
            raise ArgumentError(f"{n} bytes not a multiple of {esize}-byte elements")
        self.world.bump(self.rank, "multimem_ld_reduce")
        out = torch.empty(n // esize, dtype=tdt, device=self.torch_device)
        first, count = self._node_range()
        _lib.check(self.world._lib.sh_multimem_ld_reduce(
            self.world.handle, self.rank, first, count, handle.offset + off, n, code,
            out.data_ptr(), self._stream_handle()))
        return out

    def local_view(self, handle: SymHandle, dtype=None, shape=None):
        """Zero-copy CUDA view of this rank's replica of ``handle``."""
        import torch

        dtype = dtype or torch.uint8
        if shape is None:
            shape = (handle.length // torch.empty((), dtype=dtype).element_size(),)
        return self.world.heap_view(self.rank, handle, dtype, shape)

    def __repr__(self):
        return f"Pe(rank={self.rank}, device=cuda:{self.device})"


def _multimem_dtype(dtype):
    """(torch dtype, SH_DTYPE code) for a numpy / torch / string dtype."""
    import numpy as np
    import torch

    table = {torch.bfloat16: (torch.bfloat16, 0), torch.float16: (torch.float16, 1),
             torch.float32: (torch.float32, 2), torch.int32: (torch.int32, 3),
             torch.int64: (torch.int64, 4), torch.uint8: (torch.uint8, 5),
             torch.int8: (torch.int8, 6)}
    if isinstance(dtype, torch.dtype):
        key = dtype
    else:
        name = str(dtype) if isinstance(dtype, str) else np.dtype(dtype).name
        key = {"bfloat16": torch.bfloat16, "float16": torch.float16, "float32": torch.float32,
               "int32": torch.int32, "int64": torch.int64, "uint8": torch.uint8,
               "int8": torch.int8}.get(name)
    if key not in table:
        raise ArgumentError(f"multimem_ld_reduce does not support dtype {dtype}")
    return table[key]


def _typestr_table():
    import torch

    return {torch.uint8: "|u1", torch.int8: "|i1", torch.bool: "|b1", torch.int16: "<i2",
            torch.int32: "<i4", torch.int64: "<i8", torch.float16: "<f2", torch.bfloat16: "<V2",
            torch.float32: "<f4", torch.float64: "<f8"}


_TYPESTR = {}  # torch dtype -> __cuda_array_interface__ typestr (filled on first use)


def _typestr(dtype):
    if not _TYPESTR:
        _TYPESTR.update(_typestr_table())
    return _TYPESTR.get(dtype)


_TOOL_ENV = ("CUDA_INJECTION64_PATH", "NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_PORT_BASE",
             "NV_SANITIZER_INJECTION_PORT_BASE")
_TOOL_LIBS = ("libcuda-injection", "libsanitizer-collection", "libTreeLauncherTargetInjection",
              "libInterceptorInjectionTarget")


def serialising_tool():
    """True when kernels are serialised by a tool: Nsight Compute and
    compute-sanitizer attach through LD_PRELOAD + an injection library
    (their launch variables, or the library mapped into this process);
    CUDA_LAUNCH_BLOCKING=1 serialises every launch.  SHB_PHASED=0/1
    overrides the detection."""
    import os

    forced = os.environ.get("SHB_PHASED")
    if forced is not None and forced != "":
        return forced not in ("0", "false", "no")
    if os.environ.get("CUDA_LAUNCH_BLOCKING", "0") not in ("0", ""):
        return True
    if any(os.environ.get(v) for v in _TOOL_ENV):
        return True
    pre = os.environ.get("LD_PRELOAD", "")
    if any(lib in pre for lib in _TOOL_LIBS + ("TreeLauncher",)):
        return True
    try:
        with open("/proc/self/maps") as f:
            maps = f.read()
    except OSError:
        return False
    return any(lib in maps for lib in _TOOL_LIBS)


class _HostBarrier:
    def __init__(self, parties):
        self.parties = parties
        self.cond = threading.Condition()
        self.count = 0
        self.phase = 0

    def wait(self, timeout):
        with self.cond:
            phase = self.phase
            self.count += 1
            if self.count == self.parties:
                self.count = 0
                self.phase += 1
                self.cond.notify_all()
                return
            if not self.cond.wait_for(lambda: self.phase != phase, timeout=timeout):
                raise SynchronizationFault("barrier_all timed out")


def _check_stream_queues(devs):
    """Ranks sharing a GPU each use a compute and a copy stream; every one of
    them needs its own hardware queue, or a spinning kernel can block the
    copy it waits for (false dependency).  CUDA_DEVICE_MAX_CONNECTIONS is read
    at context creation, so refuse loudly instead of deadlocking."""
    import os
    from collections import Counter

    per_dev = max(Counter(devs).values())
    if per_dev <= 1:
        return
    need = 2 * per_dev + 2
    have = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
    if have < need:
        raise ConfigurationError(
            f"{per_dev} ranks share one GPU: set CUDA_DEVICE_MAX_CONNECTIONS>={need} before "
            "CUDA initialises (import paper_2504_19442_b200 before torch does it)")


class World:
    """Symmetric heap + signal pads on GPUs, per-rank execution contexts."""

    def __init__(self, spec: WorldSpec, scheduler="free", seed=0, *, _member=None):
        import torch

        if spec.n_nodes != 1:
            raise ConfigurationError("multi-node worlds are out of scope for the GPU path "
                                     "(one NVSwitch node); use n_nodes=1")
        if scheduler not in ("free", None):
            # the reference's cooperative schedulers fuzz CPU thread
            # interleavings; GPU concurrency is real hardware
            raise ConfigurationError(f"scheduler {scheduler!r} is CPU-only; the GPU world is 'free'")
        if not torch.cuda.is_available():
            raise ConfigurationError("no CUDA device: the symmetric heap lives in GPU memory")
        self.spec = spec
        self._lib = _lib.load()
        self._handle = ctypes.c_void_p()
        self._closed = False
        self._counters = [dict() for _ in range(spec.world_size)]
        self._stats_lock = threading.Lock()
        self._reset_sets = set()
        self._reset_lock = threading.Lock()
        self._epoch_holders = []
        lws = spec.local_world_size
        self.ranks = [RankCtx(r, r // lws, r % lws) for r in range(spec.world_size)]
        ndev = torch.cuda.device_count()
        if _member is None:
            devs = spec.devices or tuple(r % ndev for r in range(spec.world_size))
            _check_stream_queues(devs)
            arr = _lib.int_array(devs)
            _lib.check(self._lib.sh_world_create(spec.world_size, arr, spec.heap_bytes,
                                                 spec.signal_count, float(spec.timeout_s),
                                                 ctypes.byref(self._handle)))
            self.local_ranks = list(range(spec.world_size))
            self.devices = list(devs)
        else:
            rank, device = _member
            _lib.check(self._lib.sh_world_create_member(
                spec.world_size, rank, device, spec.heap_bytes, spec.signal_count,
                float(spec.timeout_s), ctypes.byref(self._handle)))
            self.local_ranks = [rank]
            self.devices = [device if r == rank else -1 for r in range(spec.world_size)]
        self.pes = [Pe(self, ctx, self.devices[ctx.rank]) if ctx.rank in self.local_ranks else None
                    for ctx in self.ranks]
        self._barrier_obj = _HostBarrier(len(self.local_ranks))
        self._phase_obj = _HostBarrier(len(self.local_ranks))
        self._host_obj = _HostBarrier(len(self.local_ranks))
        self._host_obj = _HostBarrier(len(self.local_ranks))
        self._workers = None
        self._dist = _member is not None
        self._broken = None   # reason a rank's device work never drained (see recover)
        self._seq = 0         # run() job sequence (stale results of a timed-out job are dropped)
        # Ranks of this process that wait on each other's kernels assume those
        # kernels run concurrently.  Under a kernel-serialising tool they do
        # not, so the fused ops split into phases joined on the host.
        self.phased = len(self.local_ranks) > 1 and serialising_tool()

    # ------------------------------------------------------------------
    # geometry

    @property
    def world_size(self):
        return self.spec.world_size

    @property
    def n_nodes(self):
        return self.spec.n_nodes

    @property
    def local_world_size(self):
        return self.spec.local_world_size

    @property
    def handle(self):
        return self._handle

    def pe(self, rank):
        p = self.pes[rank]
        if p is None:
            raise ArgumentError(f"rank {rank} is not hosted by this process")
        return p

    # ------------------------------------------------------------------
    # symmetric allocation (reference core.py:211-237)

    def alloc_symmetric(self, nbytes, align=8):
        if nbytes < 0:
            raise ArgumentError("negative allocation")
        off = ctypes.c_size_t()
        _lib.check(self._lib.sh_alloc(self._handle, nbytes, align, ctypes.byref(off)))
        return SymHandle(off.value, nbytes)

    def alloc_signals(self, count):
        if count < 0:
            raise ArgumentError("negative signal allocation")
        base = ctypes.c_int()
        _lib.check(self._lib.sh_alloc_signals(self._handle, count, ctypes.byref(base)))
        return SignalSet(base.value, count)

    # ------------------------------------------------------------------
    # addresses and raw access

    def heap_ptr(self, rank, handle: SymHandle, off=0, peer=None):
        """Device address of ``peer``'s replica of ``handle`` as seen from
        ``rank``'s GPU (peer defaults to rank)."""
        handle.check(off, 0)
        ptr = ctypes.c_void_p()
        _lib.check(self._lib.sh_heap_ptr(self._handle, rank, rank if peer is None else peer,
                                         handle.offset + off, ctypes.byref(ptr)))
        return ptr.value

    def _local_rank_for(self, rank):
        if rank in self.local_ranks:
            return rank
        return self.local_ranks[0]

    def heap_view(self, rank, handle: SymHandle, dtype, shape, off=0, peer=None):
        """Zero-copy CUDA tensor view of ``peer``'s replica of ``handle`` as
        mapped on ``rank``'s GPU (reference core.py:245-252)."""
        import math

        import torch

        typestr = _typestr(dtype)
        if typestr is None:
            raise ArgumentError(f"heap views support {sorted(str(t) for t in _TYPESTR)}, "
                                f"not {dtype}")
        nbytes = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
        handle.check(off, nbytes)
        ptr = self.heap_ptr(rank, handle, off, peer=peer)

        class _Arr:
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                        "data": (ptr, False), "version": 2}

        if dtype == torch.bfloat16:
            # no bf16 typestr in the interface: view as int16 and reinterpret
            _Arr.__cuda_array_interface__["typestr"] = "<i2"
            return torch.as_tensor(_Arr(), device=torch.device("cuda", self.devices[rank])).view(
                torch.bfloat16)
        return torch.as_tensor(_Arr(), device=torch.device("cuda", self.devices[rank]))

    def read_tensor(self, rank, handle: SymHandle, dtype, shape, off=0):
        """Device-side copy of rank's replica of ``handle`` (for layout checks
        of the gathered / staging buffers)."""
        import torch

        viewer = self._local_rank_for(rank)
        torch.cuda.synchronize(self.devices[viewer])
        view = self.heap_view(viewer, handle, dtype, shape, off, peer=rank)
        out = view.clone()
        torch.cuda.synchronize(self.devices[viewer])
        return out

    def copy_into(self, rank, handle: SymHandle, off, payload, chunked=None):
        """Write ``payload`` into ``rank``'s replica of ``handle``, synchronously
        (reference core.py:306-324; ``chunked`` is the CPU scheduler's knob and
        has no meaning here)."""
        import torch

        viewer = self._local_rank_for(rank)
        pe = self.pes[viewer]
        with torch.cuda.device(pe.device):
            data = pe._payload(payload)
            handle.check(off, data.numel())
            stream = torch.cuda.current_stream(pe.device)
            _lib.check(self._lib.sh_putmem(self._handle, viewer, rank, handle.offset + off,
                                           data.data_ptr(), data.numel(), stream.cuda_stream))
            stream.synchronize()

    def read_from(self, rank, handle: SymHandle, off, nbytes):
        """Bytes of rank's replica (reference core.py:326-328)."""
        import torch

        handle.check(off, nbytes)
        t = self.read_tensor(rank, handle, torch.uint8, (nbytes,), off)
        return bytes(t.cpu().numpy().tobytes())

    def _dev_of(self, rank):
        d = self.devices[rank]
        return d if d >= 0 else self.devices[self.local_ranks[0]]

    def sig_read(self, rank, sig):
        out = (ctypes.c_uint64 * 1)()
        _lib.check(self._lib.sh_read_signals(self._handle, rank, sig, 1, out))
        return int(out[0])

    def read_signals(self, rank, sigs: SignalSet):
        out = (ctypes.c_uint64 * max(1, sigs.count))()
        _lib.check(self._lib.sh_read_signals(self._handle, rank, sigs.base, sigs.count, out))
        return [int(out[i]) for i in range(sigs.count)]

    def zero_signals(self, rank, base, count, stream=None):
        _lib.check(self._lib.sh_reset_signals(self._handle, rank, base, count,
                                              ctypes.c_void_p(stream or 0)))

    def zero_all_signals(self):
        with self._quiescent():
            for r in self.local_ranks:
                self.zero_signals(r, 0, self.spec.signal_count)
        for holder in self._epoch_holders:
            holder.reset_epochs()

    @contextlib.contextmanager
    def _quiescent(self):
        """Zeroing window for signal words.  Peers write this rank's flags
        from their own streams (done / producer releases after their GEMMs),
        so every local device is drained and -- one process per GPU -- every
        process has drained (barrier) before the words are cleared, and no
        process starts a new call, whose first act is writing peers' flags,
        before every process has cleared its own (second barrier)."""
        import torch

        for r in self.local_ranks:
            torch.cuda.synchronize(self._dev_of(r))
        if self._dist:
            import torch.distributed as dist

            dist.barrier()
        yield
        for r in self.local_ranks:
            torch.cuda.synchronize(self._dev_of(r))
        if self._dist:
            import torch.distributed as dist

            dist.barrier()

    def sweep_signals(self):
        """{(rank, sig): value} for every nonzero signal word of local ranks."""
        hot = {}
        for r in self.local_ranks:
            vals = self.read_signals(r, SignalSet(0, self.spec.signal_count))
            for s, v in enumerate(vals):
                if v:
                    hot[(r, s)] = v
        return hot

    # ------------------------------------------------------------------
    # instrumentation (reference core.py:420-432)

    def bump(self, rank, name, n=1):
        with self._stats_lock:
            c = self._counters[rank]
            c[name] = c.get(name, 0) + n

    def counters(self, rank):
        with self._stats_lock:
            return dict(self._counters[rank])

    def reset_counters(self):
        with self._stats_lock:
            for c in self._counters:
                c.clear()

    # ------------------------------------------------------------------
    # timeline (reference core.py:434-444; device stamps, see timeline.py)

    def start_trace(self, records_per_cta=512, launches=16):
        from .timeline import start_trace

        start_trace(self, records_per_cta, launches)

    def stop_trace(self):
        from .timeline import stop_trace

        return stop_trace(self)

    # ------------------------------------------------------------------
    # device error words

    def poll_error(self, rank):
        code = ctypes.c_int()
        _lib.check(self._lib.sh_poll_error(self._handle, rank, ctypes.byref(code)))
        return code.value

    def check_errors(self, rank):
        code = self.poll_error(rank)
        if code:
            what = {1: "AllGather chunk flag", 2: "ReduceScatter slot release",
                    3: "ReduceScatter arrival counter", 4: "stream flag wait",
                    5: "stream-K partial", 6: "own-chunk staging stores"}.get(code, "flag")
            raise SynchronizationFault(
                f"rank {rank}: device wait on {what} exceeded {self.spec.timeout_s} s")

    def recover(self):
        """Clear device error words and host rendezvous state (core.py:489-493).

        A world left broken by a stream that never drained (a stream-side
        wait on a flag nobody released -- a peer that died) is first
        unblocked: every local signal word is saturated from a side stream,
        which satisfies any pending >= wait.  Every wait on the way is
        bounded; if a stream still does not drain the world stays broken and
        ShmemError says so (only a new process clears a wedged GPU queue)."""
        import time

        import torch

        if self._broken:
            deadline = time.monotonic() + 10.0
            for r in self.local_ranks:
                dev = self._dev_of(r)
                with torch.cuda.device(dev):
                    side = torch.cuda.Stream(device=dev)
                    # the library's own preloaded kernel: a first launch of a
                    # lazily loaded (torch) kernel would synchronise the
                    # context against the blocked stream
                    _lib.check(self._lib.sh_fill_signals(self._handle, r, 0,
                                                         self.spec.signal_count, 1 << 62,
                                                         ctypes.c_void_p(side.cuda_stream)))
                    while not side.query() and time.monotonic() < deadline:
                        time.sleep(1e-3)
            for r in self.local_ranks:
                pe = self.pes[r]
                if pe is not None and pe._stream is not None:
                    while not pe._stream.query() and time.monotonic() < deadline:
                        time.sleep(1e-3)
                    if not pe._stream.query():
                        raise ShmemError(f"{self._broken}; the stream is still blocked after "
                                         "releasing every signal -- restart the process")
        for r in self.local_ranks:
            torch.cuda.synchronize(self._dev_of(r))
            _lib.check(self._lib.sh_clear_error(self._handle, r))
        if self._broken:
            for r in self.local_ranks:
                self.zero_signals(r, 0, self.spec.signal_count)
                torch.cuda.synchronize(self._dev_of(r))
            for holder in self._epoch_holders:
                holder.reset_epochs()
            self._broken = None
        self._barrier_obj = _HostBarrier(len(self.local_ranks))
        self._phase_obj = _HostBarrier(len(self.local_ranks))
        self._host_obj = _HostBarrier(len(self.local_ranks))

    # ------------------------------------------------------------------
    # epochs / reset

    def _register_epochs(self, holder):
        self._epoch_holders.append(holder)

    def _request_reset(self, sigsets):
        with self._reset_lock:
            for s in sigsets:
                self._reset_sets.add(s)

    def _apply_resets(self):
        """After a join every rank is past every flag of the finished calls,
        so zeroing is race-free (the epoch protocol needs no reset in between;
        this restores the reference's flag hygiene, collectives.py:67-69).
        With one process per GPU the join is the barrier pair of
        ``_quiescent``: a call is rank-collective, so every process requests
        the same resets and reaches this point (reference collectives.py:1-10)."""

        with self._reset_lock:
            sets, self._reset_sets = self._reset_sets, set()
        if not sets:
            return
        with self._quiescent():
            for r in self.local_ranks:
                for s in sets:
                    self.zero_signals(r, s.base, s.count)
        for holder in self._epoch_holders:
            holder.reset_epochs_for(sets)

    # ------------------------------------------------------------------
    # running rank functions (reference core.py:449-547)

    def _barrier(self, pe):
        import torch

        torch.cuda.synchronize(pe.device)
        if self._dist:
            import torch.distributed as dist

            dist.barrier()
        else:
            self._barrier_obj.wait(self.spec.timeout_s * 4 + 30)

    def _phase_join(self, pe):
        """Host join between the phases of a phased fused call: this rank's
        stream has drained (its pushes / scatters have landed) and so have
        every other local rank's."""
        import torch

        torch.cuda.current_stream(pe.device).synchronize()
        self._phase_obj.wait(self.spec.timeout_s * 4 + 30)

    def _host_join(self, pe):
        """Rendezvous of the local rank threads before a collective with host
        operands is issued (no device synchronisation)."""
        self._host_obj.wait(self.spec.timeout_s * 4 + 30)

    def _drain(self, pe, stream):
        """Wait for the rank's stream with a host deadline.  Device spins are
        bounded and report through the error word; a stream-side wait on a
        flag nobody writes (a peer that died) is not, so the host gives up
        after the reference's deadline (core.py:467-468) and the world needs
        recover()."""
        import time

        deadline = time.monotonic() + self.spec.timeout_s * 4 + 30
        nap = 5e-5
        while not stream.query():
            self.check_errors(pe.rank)
            if time.monotonic() > deadline:
                self._broken = (f"rank {pe.rank}: device work did not drain within "
                                f"{self.spec.timeout_s * 4 + 30:.0f} s")
                raise SynchronizationFault(self._broken + " (a flag was never released)")
            time.sleep(nap)
            nap = min(nap * 2, 2e-3)

    def _run_rank(self, fn, rank):
        import torch

        pe = self.pes[rank]
        torch.cuda.set_device(pe.device)
        s = pe.stream()
        s.wait_stream(torch.cuda.current_stream(pe.device))
        with torch.cuda.stream(s):
            val = fn(pe)
        self._drain(pe, s)
        self.check_errors(rank)
        return val

    def run(self, fn, timeout=None):
        """Run ``fn(pe)`` on every local rank concurrently; per-rank results in
        rank order.  Device work of each rank is drained before returning, and
        any failure is aggregated into ``CollectiveFault``.

        Ranks that share a process must not block on the GPU inside ``fn``
        once they have issued a collective (``.cpu()``, ``.item()``, pageable
        ``.to('cuda')``): the CUDA driver serialises pageable copies, so a rank
        waiting on its stream there can hold back a sibling's launch that its
        stream is waiting for.  Stage inputs first, return device tensors.
        For the same reason every CUDA kernel a body launches between
        collectives (a torch op, say) should have run once before: under lazy
        module loading its first launch synchronises the context, i.e. waits
        for a sibling's spinning wait that waits for this rank (the library
        preloads its own kernels)."""
        if self._closed:
            raise ConfigurationError("world is closed")
        if self._broken:
            raise UsageError(f"world needs recover(): {self._broken}")
        ranks = self.local_ranks
        if len(ranks) == 1:
            try:
                res = [self._run_rank(fn, ranks[0])]
            except BaseException as exc:  # noqa: BLE001 - aggregate like the reference
                raise CollectiveFault(f"collective failed on ranks {ranks[0]}: "
                                      f"{type(exc).__name__}: {exc}", {ranks[0]: exc}) from exc
            self._apply_resets()
            return res
        self._ensure_workers()
        self._seq += 1
        seq = self._seq
        for r in ranks:
            self._jobs[r].append((seq, fn))
            self._job_ev[r].set()
        wait_s = (timeout or self.spec.timeout_s) * 4.0 + 60.0
        results, failures = {}, {}
        import time

        deadline = time.monotonic() + wait_s
        for r in ranks:
            got = None
            while got is None:
                left = deadline - time.monotonic()
                if left <= 0 or not self._done_ev[r].wait(left):
                    break
                with self._result_lock:
                    self._done_ev[r].clear()
                    tagged = self._results.pop(r, None)
                    # a result of an earlier job that timed out is dropped
                    if tagged is not None and tagged[0] == seq:
                        got = tagged[1:]
            if got is None:
                failures[r] = TimeoutError(f"rank {r} did not finish")
                self._broken = f"rank {r} did not finish job {seq}"
                continue
            ok, val = got
            if ok:
                results[r] = val
            else:
                failures[r] = val
        if failures:
            raise CollectiveFault(
                "collective failed on ranks "
                + ", ".join(f"{r}: {type(e).__name__}: {e}" for r, e in sorted(failures.items())),
                failures)
        self._apply_resets()
        return [results[r] for r in ranks]

    def _ensure_workers(self):
        if self._workers is not None:
            return
        self._jobs = {r: deque() for r in self.local_ranks}
        self._job_ev = {r: threading.Event() for r in self.local_ranks}
        self._done_ev = {r: threading.Event() for r in self.local_ranks}
        self._results = {}
        self._result_lock = threading.Lock()
        self._workers = []
        for r in self.local_ranks:
            t = threading.Thread(target=self._worker_loop, args=(r,), daemon=True, name=f"rank{r}")
            t.start()
            self._workers.append(t)

    def _worker_loop(self, rank):
        while True:
            self._job_ev[rank].wait()
            self._job_ev[rank].clear()
            if self._closed:
                return
            while self._jobs[rank]:
                seq, fn = self._jobs[rank].popleft()
                try:
                    res = (seq, True, self._run_rank(fn, rank))
                except BaseException as exc:  # noqa: BLE001
                    res = (seq, False, exc)
                with self._result_lock:
                    self._results[rank] = res
                    self._done_ev[rank].set()

    def close(self):
        if self._closed:
            return
        self._closed = True
        if self._workers:
            for ev in self._job_ev.values():
                ev.set()
        if self._handle:
            try:
                import torch

                if self._broken:
                    self.recover()
                for r in self.local_ranks:
                    torch.cuda.synchronize(self._dev_of(r))
            except Exception:  # noqa: BLE001
                pass
            if self._broken:
                # a wedged stream would hang the destroy's device drain: leak
                # the slabs instead (the process is expected to exit)
                self._handle = ctypes.c_void_p()
                return
            self._lib.sh_world_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def init_world(spec: WorldSpec, scheduler="free", seed=0) -> World:
    """Single-process world: every rank a thread (reference core.py:565-567)."""
    return World(spec, scheduler=scheduler, seed=seed)


def exchange_ipc_handles(world: World, all_gather):
    """Attach every peer slab: ``all_gather(bytes) -> list[bytes]`` is the
    out-of-band exchange (torch.distributed.all_gather_object in practice,
    any transport in tests).  One rank per process."""
    lib = world._lib
    size = lib.sh_ipc_handle_size()
    buf = (ctypes.c_char * size)()
    _lib.check(lib.sh_export_ipc_handle(world.handle, buf))
    handles = all_gather(bytes(buf))
    if len(handles) != world.world_size or any(len(h) != size for h in handles):
        raise ConfigurationError("IPC handle exchange returned a malformed list")
    blob = b"".join(handles)
    arr = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
    _lib.check(lib.sh_import_ipc_handles(world.handle, arr))


def init_world_dist(heap_bytes=1 << 30, signal_count=None, timeout_s=5.0, device=None) -> World:
    """One process per GPU under torch.distributed (already initialised):
    this process hosts rank ``dist.get_rank()`` on ``device`` (default
    LOCAL_RANK).  Peers' slabs are mapped with CUDA IPC."""
    import os

    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        raise ConfigurationError("torch.distributed is not initialised")
    ws, rank = dist.get_world_size(), dist.get_rank()
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank % max(1, torch.cuda.device_count())))
    spec = WorldSpec(world_size=ws, heap_bytes=heap_bytes, signal_count=signal_count,
                     timeout_s=timeout_s)
    world = World(spec, _member=(rank, device))

    from .dist import all_gather_bytes

    if ws > 1:
        exchange_ipc_handles(world, all_gather_bytes)
    dist.barrier()
    return world
