"""The N>1 host path with two CPU processes over gloo: handle exchange,
argument agreement, max-over-ranks timing."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_19442_b200 import ConfigurationError
        from paper_2504_19442_b200.dist import (all_gather_bytes, check_collective_args,
                                                max_over_ranks)

        handles = all_gather_bytes(bytes([rank]) * 64)
        ok_gather = handles == [bytes([r]) * 64 for r in range(world)]
        check_collective_args(m=8192, n=3584, epoch=3)
        try:
            check_collective_args(m=8192, epoch=3 + rank)
            mismatch = False
        except ConfigurationError as e:
            mismatch = "epoch" in str(e)
        mx = max_over_ranks(1.5 + rank)
        q.put((rank, ok_gather, mismatch, mx))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_plumbing_over_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_gather, mismatch, mx in res:
        assert ok_gather and mismatch and mx == pytest.approx(2.5)
