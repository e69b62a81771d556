"""Timeline evidence emitter (§8 row f2).

Device ``%globaltimer`` stamps recorded by the fused kernels while tracing is
enabled (``sh_trace_enable``), turned into events and into the Chrome-trace
document of the reference's ``Timeline.to_chrome_trace``
(pkg/src/minishmem/costmodel.py:185-190: ``{name, ph: "X", ts, dur, pid =
rank, tid = resource}``), plus the per-launch exposed-communication summary:
how long CTAs sat waiting for a remote chunk (AG) or for peers' partial rows
(fused RS) instead of computing.

    world.start_trace()            # or timeline.start_trace(world)
    ... ag_gemm / gemm_rs calls ...
    events = world.stop_trace()
    json.dump(timeline.to_chrome_trace(events), open("trace.json", "w"))
"""

from __future__ import annotations

import ctypes
from collections import defaultdict

from . import _lib

_KINDS = {1: "chunk_wait", 2: "tile_epilogue", 3: "peer_wait", 4: "cta", 5: "mma_item",
          6: "own_reduce"}
_MODES = {0: "ag_gemm", 1: "gemm_rs", 2: "rs_reduce"}


def start_trace(world, records_per_cta=512, launches=16):
    """Enable device tracing on every local rank (ring of ``launches`` launches)."""
    for r in world.local_ranks:
        _lib.check(world._lib.sh_trace_enable(world.handle, r, records_per_cta, launches))
    world._trace_cfg = (records_per_cta, launches)


def stop_trace(world):
    """Collect the recorded events of every local rank and disable tracing."""
    events = []
    recs, launches = getattr(world, "_trace_cfg", (0, 0))
    if not recs:
        return events
    for r in world.local_ranks:
        events += read_trace(world, r, recs, launches)
        _lib.check(world._lib.sh_trace_enable(world.handle, r, 0, 0))
    world._trace_cfg = (0, 0)
    return events


def read_trace(world, rank, records_per_cta, launches):
    import numpy as np

    grid = 256  # upper bound; the library reports the real grid in info[2]
    info = (ctypes.c_int * (4 + launches))()
    words = launches * grid * records_per_cta * 4
    buf = np.zeros(words, dtype=np.uint64)
    _lib.check(world._lib.sh_trace_read(world.handle, rank,
                                        buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                        words, info))
    count, slots, grid, cap = info[0], info[1], info[2], info[3]
    modes = [info[4 + i] for i in range(slots)]
    rec = buf[: slots * grid * cap * 4].reshape(slots, grid, cap, 4)
    used = min(count, slots)
    first = count - used  # oldest launch still in the ring
    events = []
    for n in range(first, count):
        slot = n % slots
        for cta in range(grid):
            for j in range(cap):
                kind_aux, t0, t1, tile = (int(x) for x in rec[slot, cta, j])
                kind = kind_aux >> 56
                if kind == 0 or t1 < t0:
                    continue
                events.append({
                    "rank": rank, "launch": n, "kernel": _MODES.get(modes[slot], "?"),
                    "op": _KINDS.get(kind, str(kind)), "cta": cta,
                    "chunk": kind_aux & 0xFFFFFFFF if kind in (1, 2, 3) else None,
                    "item_kind": (kind_aux >> 32) & 0xFF if kind == 2 else None,
                    "ranges": (kind_aux >> 32) & 0xFF if kind == 1 else None,
                    "stage_wait_ns": kind_aux & 0xFFFFFFFF if kind == 5 else None,
                    "drain_ns": kind_aux & 0xFFFFFFFF if kind == 6 else None,
                    "tile": tile, "t0_ns": t0, "t1_ns": t1,
                })
    return events


def to_chrome_trace(events):
    """Chrome trace event list (chrome://tracing / Perfetto), the reference's
    shape (costmodel.py:185-190, schemas.TRACE): pid = rank, tid = the CTA
    as a resource name, times in us from the earliest record."""
    if not events:
        return []
    base = min(e["t0_ns"] for e in events)
    out = []
    for e in events:
        name = e["op"] if e["chunk"] is None else f"{e['op']}[c{e['chunk']}]"
        out.append({"name": f"{e['kernel']}#{e['launch']} {name}", "ph": "X",
                    "ts": (e["t0_ns"] - base) / 1e3, "dur": (e["t1_ns"] - e["t0_ns"]) / 1e3,
                    "pid": e["rank"], "tid": f"cta{e['cta']}"})
    return out


def exposed_comm(events):
    """Per (rank, launch): kernel span and time CTAs spent waiting on remote
    data -- max and mean over CTAs of the summed chunk / peer waits."""
    by = defaultdict(lambda: {"span": [None, None], "wait": defaultdict(int)})
    for e in events:
        key = (e["rank"], e["launch"], e["kernel"])
        d = by[key]
        if e["op"] == "cta":
            lo, hi = d["span"]
            d["span"] = [e["t0_ns"] if lo is None else min(lo, e["t0_ns"]),
                         e["t1_ns"] if hi is None else max(hi, e["t1_ns"])]
        elif e["op"] in ("chunk_wait", "peer_wait"):
            d["wait"][e["cta"]] += e["t1_ns"] - e["t0_ns"]
    out = []
    for (rank, launch, kernel), d in sorted(by.items()):
        waits = list(d["wait"].values()) or [0]
        lo, hi = d["span"]
        out.append({"rank": rank, "launch": launch, "kernel": kernel,
                    "span_us": None if lo is None else (hi - lo) / 1e3,
                    "wait_max_us": max(waits) / 1e3,
                    "wait_mean_us": sum(waits) / len(waits) / 1e3})
    return out
