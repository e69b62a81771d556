"""CPU oracle for the ag_gemm / gemm_rs hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the timed CPU
baseline; the product path (paper_2504_19442_b200) never calls it.

It restates, in numpy, what the reference package computes on this path
(/root/reference/pkg/src/minishmem, read-only; the algorithm itself lives in
numpy's ``@`` / ``+=``, numpy>=1.24 unpinned per pkg/pyproject.toml:10-13):

* ``ag_gemm``  (pipelines.py:97-150): every rank returns
  ``vstack(shards) @ b_rank``; the symmetric ``gathered`` buffer of every rank
  holds slot r = bytes of rank r's shard (allgather_push_intra,
  collectives.py:83-102, pushes to every peer including self).
* ``gemm_rs``  (pipelines.py:179-216 + rs_intra_streams, collectives.py:131-175):
  rank d's staging slot s = rows d of ``a_s @ b_s`` (scatter, :156-161);
  rank d's output = sum over s ascending of those slots (reduce, :163-171).

Parity is pinned: tests/test_oracle_golden.py checks these functions against
fixtures produced by running the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------
# dense semantics (the equality the reference's own tests assert,
# tests/test_pipelines.py:37-50, :150-163)

def ag_gemm_reference(shards, b):
    """C = concat(A_shards) @ B  (pipelines.py:100, 142-144)."""
    return np.vstack(shards) @ b


def gathered_layout(shards):
    """Rank-independent content of ``gathered`` after the push (collectives.py:95-97)."""
    return np.vstack(shards)


def gemm_rs_reference(amats, bmats):
    """Per-rank outputs: row block r of sum_s a_s @ b_s, summed in ascending s
    (collectives.py:165: fixed ascending order keeps floats reproducible)."""
    w = len(amats)
    m = amats[0].shape[0]
    rows = m // w
    acc = None
    for a, b in zip(amats, bmats):
        prod = a @ b
        acc = prod if acc is None else acc + prod
    return [acc[r * rows:(r + 1) * rows] for r in range(w)]


def staging_layout(amats, bmats, dest):
    """Rank ``dest``'s staging buffer: slot s = rows ``dest`` of a_s @ b_s
    (collectives.py:160, dst_off = rank * chunk_bytes)."""
    w = len(amats)
    rows = amats[0].shape[0] // w
    return np.stack([(a @ b)[dest * rows:(dest + 1) * rows] for a, b in zip(amats, bmats)])


# ----------------------------------------------------------------------------
# schedules (swizzle.py:65-117), restated for cross-checking the product's

def ag_order_switch(rank, world):
    """swizzle.py:65-78: step s -> chunk (rank+s) mod world."""
    return [(rank + s) % world for s in range(world)]


def rs_inter_order(rank, node_id, local_rank, n_nodes, local_world):
    """swizzle.py:99-117: peer-node blocks first, own node last; each block
    starts at local_rank+1."""
    out = []
    for dn in range(1, n_nodes + 1):
        node = (node_id + dn) % n_nodes
        for dl in range(1, local_world + 1):
            out.append(node * local_world + (local_rank + dl) % local_world)
    return out


def first_visit_order(chunks, world):
    """pipelines.py:71-79."""
    seen = []
    for c in chunks:
        if c not in seen:
            seen.append(c)
    if sorted(seen) != list(range(world)):
        raise ValueError(f"schedule covers chunks {sorted(seen)}, need 0..{world - 1}")
    return seen


# ----------------------------------------------------------------------------
# algorithmic port (the CPU baseline): the reference's per-rank structure --
# push every shard into every gathered replica, then consume chunks in
# schedule order tile by tile; produce partial chunks in schedule order,
# scatter into owners' staging slots, reduce ascending.  One process, ranks
# simulated in sequence; BLAS threads do the arithmetic like the reference.

def port_ag_gemm(shards, b_per_rank, orders, tile_m=0, tile_n=0):
    w = len(shards)
    rows, k = shards[0].shape
    gathered = [np.empty((w * rows, k), dtype=shards[0].dtype) for _ in range(w)]
    for src in range(w):                      # allgather_push_intra, every peer incl. self
        for peer in range(w):
            gathered[peer][src * rows:(src + 1) * rows] = shards[src]
    outs = []
    for rank in range(w):
        b = b_per_rank[rank]
        n = b.shape[1]
        out = np.zeros((w * rows, n), dtype=shards[0].dtype)
        tm, tn = tile_m or rows, tile_n or n
        for chunk in orders[rank]:
            a_chunk = shards[rank] if chunk == rank else gathered[rank][chunk * rows:(chunk + 1) * rows]
            base = chunk * rows
            for r0 in range(0, rows, tm):
                for c0 in range(0, n, tn):
                    out[base + r0:base + min(r0 + tm, rows), c0:c0 + tn] = (
                        a_chunk[r0:r0 + tm] @ b[:, c0:c0 + tn])
        outs.append(out)
    return outs, gathered


def port_gemm_rs(amats, b_per_rank, orders):
    w = len(amats)
    m = amats[0].shape[0]
    rows = m // w
    n = b_per_rank[0].shape[1]
    staging = [np.empty((w, rows, n), dtype=amats[0].dtype) for _ in range(w)]
    for src in range(w):
        for dest in orders[src]:              # producer chunk order, then scatter
            part = amats[src][dest * rows:(dest + 1) * rows] @ b_per_rank[src]
            staging[dest][src] = part
    outs = []
    for dest in range(w):
        acc = np.zeros((rows, n), dtype=amats[0].dtype)
        for src in range(w):                  # ascending source order
            acc += staging[dest][src]
        outs.append(acc)
    return outs, staging
