import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import torch
import paper_2504_19442_b200 as sb
from paper_2504_19442_b200.primitives import SignalOp, WaitCond
W, N = 2, 4096
EP = int(sys.argv[1]) if len(sys.argv) > 1 else 50
with sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 20, timeout_s=5.0, devices=(0,) * W)) as w:
    recv = w.alloc_symmetric(N * 8)
    data_sig, ack_sig = w.alloc_signals(1).base, w.alloc_signals(1).base
    dev = torch.device("cuda", 0)
    src = torch.empty(N, dtype=torch.int64, device=dev)
    seen = torch.zeros((), dtype=torch.int64, device=dev)
    def body(pe):
        if pe.rank == 0:
            for e in range(1, EP + 1):
                if e > 1:
                    pe.signal_wait_until(ack_sig, WaitCond.GE, e - 1)
                src.fill_(e)
                pe.putmem_signal(recv, src, data_sig, e, 1)
        else:
            view = w.heap_view(1, recv, torch.int64, (N,))
            for e in range(1, EP + 1):
                pe.signal_wait_until(data_sig, WaitCond.GE, e)
                seen.add_(1)
                pe.signal_op(0, ack_sig, SignalOp.SET, e)
    t0 = time.time()
    try:
        w.run(body, timeout=20)
        print("ok", EP, time.time() - t0)
    except Exception as e:
        print("FAIL", type(e).__name__, str(e)[:200])
        print("seen", int(seen), "data(rank1)", w.read_signals(1, sb.SignalSet(data_sig, 1)),
              "ack(rank0)", w.read_signals(0, sb.SignalSet(ack_sig, 1)))
