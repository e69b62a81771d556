"""Standalone one-sided collectives on the GPU symmetric heap (§8 row f3).

The comm halves of the fused kernels, usable on their own, with the
reference's signatures and semantics (pkg/src/minishmem/collectives.py):

* ``allgather_push_intra`` (collectives.py:83-102): the owner copies its
  chunk into slot ``rank`` of every rank's buffer (copy engine over NVLink)
  and raises that rank's per-source signal; no barrier anywhere.
* ``allgather_pull_intra`` (collectives.py:105-125): publish the own chunk,
  one barrier, then fetch remote chunks in the caller's order.
* ``reducescatter_push_intra`` (collectives.py:178-194 + rs_intra_streams
  131-175): chunk ``dest`` of the input goes to slot ``rank`` of ``dest``'s
  staging once ``producer[dest]`` is set; the owner sums its slots in
  ascending source order (fp32 accumulate for bf16/fp16; element type for
  fp32/int32/int64, matching numpy's ``acc +=`` bit for bit).

All operations are stream-ordered on each rank's current CUDA stream;
``World.run`` drains them.  As in the reference, rounds on the same buffers
must be separated by a join (``World.run``) when ``reset=True``.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .core import SignalSet, SymHandle
from .errors import ArgumentError
from .primitives import SignalOp, WaitCond, consume_token
from .swizzle import ag_push_order

SYNC_WAIT = "wait_until"
SYNC_TOKEN = "token"


@dataclass(frozen=True)
class ChunkLayout:
    """Per-rank slot arithmetic of a symmetric buffer split into equal chunks
    (reference collectives.py:28-56)."""

    world_size: int
    total_elems: int
    elem_bytes: int

    def __post_init__(self):
        if self.total_elems % self.world_size:
            raise ArgumentError(
                f"{self.total_elems} elements do not split into {self.world_size} chunks")

    @property
    def chunk_elems(self):
        return self.total_elems // self.world_size

    @property
    def chunk_bytes(self):
        return self.chunk_elems * self.elem_bytes

    @property
    def total_bytes(self):
        return self.total_elems * self.elem_bytes

    def span(self, chunk):
        if not 0 <= chunk < self.world_size:
            raise ArgumentError(f"chunk {chunk} out of {self.world_size}")
        return chunk * self.chunk_bytes, self.chunk_bytes


def _await(pe, sig, value, style):
    if style == SYNC_TOKEN:
        consume_token(pe.wait(sig, value), None)
    elif style == SYNC_WAIT:
        pe.signal_wait_until(sig, WaitCond.EQ, value)
    else:
        raise ArgumentError(f"unknown sync_style {style!r}")


def _reset_own_signals(pe, sigs: SignalSet, count):
    """Zero the rank's own signal words, stream-ordered (collectives.py:67-69)."""
    import torch

    pe.world.zero_signals(pe.rank, sigs.base, count,
                          stream=torch.cuda.current_stream(pe.device).cuda_stream)


def allgather_push_intra(pe, dst: SymHandle, sigs: SignalSet, local, *, wait_all=True,
                         reset=True, sync_style=SYNC_WAIT):
    """Push-mode AllGather: slot ``r`` of every replica of ``dst`` receives rank
    r's bytes; consumers proceed per slot, no barrier."""
    payload = pe._payload(local)
    n = payload.numel()
    world = pe.world.world_size
    if dst.length != world * n:
        raise ArgumentError(f"gather buffer is {dst.length} bytes, need {world * n}")
    if sigs.count < world:
        raise ArgumentError("need one signal per source rank")
    # own slot first, then the peers in the order the ring schedule consumes
    for peer in [pe.rank] + ag_push_order(pe.rank, world):
        pe.putmem(dst, payload, peer, dst_off=pe.rank * n)
        pe.signal_op(peer, sigs.at(pe.rank), SignalOp.SET, 1)
    if wait_all:
        for src in range(world):
            _await(pe, sigs.at(src), 1, sync_style)
        if reset:
            _reset_own_signals(pe, sigs, world)


def allgather_pull_intra(pe, dst: SymHandle, sigs: SignalSet, local, *, order=None, reset=True):
    """Pull-mode AllGather: publish the own chunk, make it visible with one
    barrier, then fetch the remote chunks in ``order``."""
    payload = pe._payload(local)
    n = payload.numel()
    world = pe.world.world_size
    if dst.length != world * n:
        raise ArgumentError(f"gather buffer is {dst.length} bytes, need {world * n}")
    if sigs.count < world:
        raise ArgumentError("need one signal per source rank")
    pe.putmem(dst, payload, pe.rank, dst_off=pe.rank * n)
    pe.signal_op(pe.rank, sigs.at(pe.rank), SignalOp.SET, 1)
    pe.barrier_all()  # every rank's own chunk is in place
    for src in order if order is not None else range(world):
        if src == pe.rank:
            continue
        pe.getmem(dst, dst, src, nbytes=n, dst_off=src * n, src_off=src * n)
        pe.signal_op(pe.rank, sigs.at(src), SignalOp.SET, 1)
    if reset:
        _reset_own_signals(pe, sigs, world)


_RS_DTYPES = None


def _rs_dtype_code(dtype):
    import torch

    global _RS_DTYPES
    if _RS_DTYPES is None:
        _RS_DTYPES = {torch.bfloat16: _lib.SH_DTYPE_BF16, torch.float16: _lib.SH_DTYPE_FP16,
                      torch.float32: _lib.SH_DTYPE_FP32, torch.int32: _lib.SH_DTYPE_I32,
                      torch.int64: _lib.SH_DTYPE_I64}
    code = _RS_DTYPES.get(dtype)
    if code is None:
        raise ArgumentError(f"dtype {dtype} not supported (bf16/fp16/fp32/int32/int64)")
    return code


def reducescatter_push_intra(pe, staging: SymHandle, producer_sigs: SignalSet,
                             reduce_sigs: SignalSet, local_vals, out, *, order=None, reset=True,
                             sync_style=SYNC_WAIT):
    """Push-mode ReduceScatter: chunk ``dest`` of ``local_vals`` is scattered to
    slot ``rank`` of ``dest``'s staging once ``producer_sigs[dest]`` is 1; each
    rank reduces its W slots in ascending source order into ``out``.

    ``local_vals`` / ``out`` are CUDA tensors of one dtype (``out`` is written
    in place, like the reference's ``out[:] = acc``)."""
    import torch

    world = pe.world.world_size
    if not isinstance(local_vals, torch.Tensor) or not isinstance(out, torch.Tensor):
        raise ArgumentError("local_vals and out must be torch tensors")
    if out.dtype != local_vals.dtype:
        raise ArgumentError(f"dtype mismatch: {local_vals.dtype} vs {out.dtype}")
    code = _rs_dtype_code(out.dtype)
    chunk = out.numel()
    if local_vals.numel() != world * chunk:
        raise ArgumentError(f"input holds {local_vals.numel()} elements, need {world}x{chunk}")
    if not local_vals.is_contiguous():
        raise ArgumentError("input must be C-contiguous (the scatter reads it in place)")
    if not out.is_cuda or not out.is_contiguous():
        raise ArgumentError("out must be a contiguous CUDA tensor")
    chunk_bytes = chunk * out.element_size()
    if staging.length != world * chunk_bytes:
        raise ArgumentError(f"staging is {staging.length} bytes, need {world * chunk_bytes}")
    if producer_sigs.count < world or reduce_sigs.count < world:
        raise ArgumentError("need one producer and one reduction signal per rank")
    flat = local_vals.to(pe.torch_device).view(world, chunk)
    # scatter (copy-engine role, collectives.py:156-161)
    for dest in order if order is not None else range(world):
        _await(pe, producer_sigs.at(dest), 1, sync_style)
        pe.putmem(staging, flat[dest], dest, dst_off=pe.rank * chunk_bytes)
        pe.signal_op(dest, reduce_sigs.at(pe.rank), SignalOp.SET, 1)
    # reduce (collectives.py:163-171): every source landed, then ascending sum
    for src in range(world):
        _await(pe, reduce_sigs.at(src), 1, sync_style)
    _lib.check(pe.world._lib.sh_reduce_slots(pe.world.handle, pe.rank, staging.offset, world,
                                             chunk, code, out.data_ptr(), pe._stream_handle()))
    if reset:
        _reset_own_signals(pe, reduce_sigs, world)
        _reset_own_signals(pe, producer_sigs, world)
    return out
