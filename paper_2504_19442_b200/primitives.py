"""One-sided primitive vocabulary (reference pkg/src/minishmem/primitives.py:26-73).

The operations themselves are methods of ``Pe`` (core.py) and run on the GPU:
``putmem`` / ``getmem`` are copy-engine transfers into / out of a peer's slab,
``signal_op`` is a release store (or device red.add) on a peer's signal word,
``signal_wait_until`` / ``wait`` make the rank's stream wait on its own pad
(GPU front end for EQ/GE, bounded one-thread spin otherwise).  Everything is
stream-ordered on the rank's current CUDA stream, so a wait orders every later
read of the stream after the signalled data, which is the data-before-signal
contract of the reference."""

from __future__ import annotations

import enum
from dataclasses import dataclass

from .errors import UsageError


class SignalOp(enum.Enum):
    SET = "set"
    ADD = "add"


class WaitCond(enum.Enum):
    EQ = "eq"
    NE = "ne"
    GE = "ge"
    GT = "gt"
    LE = "le"
    LT = "lt"

    @property
    def code(self):
        return {"eq": 0, "ne": 1, "ge": 2, "gt": 3, "le": 4, "lt": 5}[self.value]

    def holds(self, observed, value):
        return {
            "eq": observed == value, "ne": observed != value, "ge": observed >= value,
            "gt": observed > value, "le": observed <= value, "lt": observed < value,
        }[self.value]


@dataclass
class Token:
    """Witness that a wait was enqueued; single use."""

    sig: int
    value: int
    _consumed: bool = False


def consume_token(token: Token, payload):
    """Tie ``payload`` reads to the wait that produced ``token`` (single use)."""
    if not isinstance(token, Token):
        raise UsageError("consume_token needs a Token produced by wait()")
    if token._consumed:
        raise UsageError(f"token for signal {token.sig} consumed twice")
    token._consumed = True
    return payload
