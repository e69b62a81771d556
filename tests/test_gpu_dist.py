"""The one-process-per-rank path (init_world_dist: CUDA IPC handles exchanged
over torch.distributed) with two processes.  On a one-GPU box both processes
share cuda:0 -- their kernels are time-sliced by the driver, so the flag
protocol is exercised across real process/context boundaries (slowly)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_19442_b200 as sb
        from oracle import minishmem_oracle as oracle

        dev = torch.cuda.device_count() and rank % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        world_obj = sb.init_world_dist(heap_bytes=1 << 24, timeout_s=60.0, device=dev)
        pe = world_obj.pe(rank)
        g = np.random.default_rng(7)
        shards = [g.integers(-2, 3, (256, 128)) for _ in range(world)]
        b = g.integers(-1, 2, (128, 128))
        amats = [g.integers(-2, 3, (256 * world, 128)) for _ in range(world)]
        ag_shape = sb.ProblemShape(m=256 * world, n=128, k=128, dtype="bfloat16")
        rs_shape = sb.ProblemShape(m=256 * world, n=128, k=128, dtype="bfloat16")
        agb = sb.make_ag_gemm_buffers(world_obj, ag_shape)
        rsb = sb.make_gemm_rs_buffers(world_obj, rs_shape)
        t = lambda a: torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).cuda(dev)  # noqa: E731
        x, bb, a = t(shards[rank]), t(b), t(amats[rank])

        def body(pe):
            outs = []
            for _ in range(2):  # back to back: epochs, no reset
                h = sb.ag_gemm(pe, x, bb, ag_shape, sb.ag_order_switch(pe.rank, world), agb,
                               reset=False)
                y = sb.gemm_rs(pe, a, bb, rs_shape, sb.rs_inter_order(pe.ctx, 1, world), rsb,
                               reset=False)
                outs.append((h, y))
            return outs

        outs = world_obj.run(body)[0]
        ok_ag = all(np.array_equal(h.float().cpu().numpy(), oracle.ag_gemm_reference(shards, b))
                    for h, _ in outs)
        ref = oracle.gemm_rs_reference(amats, [b] * world)[rank]
        ok_rs = all(np.array_equal(y.float().cpu().numpy(), ref) for _, y in outs)

        # the default reset=True path, back to back: every join zeroes the
        # flags only after both processes drained (World._quiescent), so no
        # late peer store survives the reset and every call is exact
        why = [] if ok_rs else ["back-to-back rs mismatch"]
        for it in range(4):
            h, y = world_obj.run(lambda pe: (
                sb.ag_gemm(pe, x, bb, ag_shape, sb.ag_order_switch(pe.rank, world), agb),
                sb.gemm_rs(pe, a, bb, rs_shape, sb.rs_inter_order(pe.ctx, 1, world), rsb)))[0]
            ok_ag = ok_ag and np.array_equal(h.float().cpu().numpy(),
                                             oracle.ag_gemm_reference(shards, b))
            yv = y.float().cpu().numpy()
            if not np.array_equal(yv, ref):
                why.append(f"it{it}: rs max|diff| {np.abs(yv - ref).max()} at "
                           f"{np.unravel_index(np.abs(yv - ref).argmax(), ref.shape)}")
                ok_rs = False
            hot = world_obj.sweep_signals()
            if hot:
                why.append(f"it{it}: hot signals {hot}")
                ok_rs = False
            # the sweep reads this rank's pad: a faster peer must not start
            # its next call (whose first act writes this rank's ready flag)
            # before the sweep is done
            dist.barrier()
        gathered = world_obj.read_tensor(rank, agb.gathered, torch.bfloat16, (256 * world, 128))
        ok_layout = np.array_equal(gathered.float().cpu().numpy(), oracle.gathered_layout(shards))
        dist.barrier()
        world_obj.close()
        q.put((rank, ok_ag, ok_rs, ok_layout, "; ".join(why) if not ok_rs else ""))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, False, False, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_ipc_world():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=540) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for rank, ok_ag, ok_rs, ok_layout, err in res:
        assert not err, f"rank {rank}: {err}"
        assert ok_ag and ok_rs and ok_layout, (rank, ok_ag, ok_rs, ok_layout)
