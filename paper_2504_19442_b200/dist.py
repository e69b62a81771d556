"""Host-side plumbing of the one-process-per-GPU world (torch.distributed).

Only control data crosses this layer -- IPC handles of the symmetric slabs,
argument-agreement checks, timings.  Tensor data never does: it moves over
NVLink through the symmetric heap (C ABI).  Works with any backend, so the
multi-rank host logic is testable on CPU with gloo.
"""

from __future__ import annotations

from .errors import ConfigurationError


def _dist():
    import torch.distributed as dist

    if not dist.is_initialized():
        raise ConfigurationError("torch.distributed is not initialised")
    return dist


def all_gather_bytes(blob: bytes) -> list:
    """Every rank's ``blob`` in rank order (used for the 64-byte CUDA IPC
    handles of the symmetric slabs)."""
    dist = _dist()
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, bytes(blob))
    return out


def check_collective_args(**kwargs):
    """A call is rank-collective: every rank must pass consistent arguments
    (reference collectives.py:1-10).  Raises ConfigurationError
    naming the first disagreeing key.  Debug aid; costs one all-gather."""
    dist = _dist()
    mine = sorted(kwargs.items())
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, mine)
    for r, theirs in enumerate(allv):
        if theirs != mine:
            diff = [k for (k, v), (_, w) in zip(mine, theirs) if v != w]
            raise ConfigurationError(f"rank {dist.get_rank()} and rank {r} disagree on {diff}")


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over ranks (bench timing rule: slowest rank)."""
    import torch

    dist = _dist()
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
