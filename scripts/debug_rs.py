import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2504_19442_b200 as sb
import torch

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "rs"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
stage = sys.argv[4] if len(sys.argv) > 4 else "device"
shape = sb.ProblemShape(m=256 * W, n=192, k=320, dtype="bfloat16")
w = sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=1 << 24, timeout_s=3.0))
rsb = sb.make_gemm_rs_buffers(w, shape)
agb = sb.make_ag_gemm_buffers(w, shape)
An = [np.random.default_rng(r).integers(-2, 3, (shape.m, shape.k)) for r in range(W)]
Sn = [np.random.default_rng(r).integers(-2, 3, (shape.m // W, shape.k)) for r in range(W)]
Bn = np.random.default_rng(99).integers(-1, 2, (shape.k, shape.n))
A = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in An]
S = [torch.from_numpy(x).to(torch.bfloat16).cuda() for x in Sn]
B = torch.from_numpy(Bn).to(torch.bfloat16).cuda()
Sp = [torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in Sn]
Bp = torch.from_numpy(Bn).to(torch.bfloat16).pin_memory()

def inputs(pe, i):
    if stage == "device":
        return (A if mode == "rs" else S)[pe.rank], B
    if stage == "pinned":
        return Sp[pe.rank].to(pe.torch_device, non_blocking=True), Bp.to(pe.torch_device, non_blocking=True)
    x = (An if mode == "rs" else Sn)[pe.rank]
    return (torch.from_numpy(x).to(torch.bfloat16).to(pe.torch_device),
            torch.from_numpy(Bn).to(torch.bfloat16).to(pe.torch_device))

fails = 0
for it in range(iters):
    t0 = time.time()
    try:
        if mode == "rs":
            def body(pe):
                a, b = inputs(pe, it)
                return sb.gemm_rs(pe, a, b, shape, sb.rs_inter_order(pe.ctx, 1, W), rsb)
        else:
            def body(pe):
                a, b = inputs(pe, it)
                return sb.ag_gemm(pe, a, b, shape, sb.ag_order_switch(pe.rank, W), agb)
        outs = w.run(body)
    except Exception as e:
        fails += 1
        print(it, "FAIL", round(time.time() - t0, 3), str(e)[:200], flush=True)
        torch.cuda.synchronize()
        for r in range(W):
            print(" rank", r, "err", w.poll_error(r), "prod", w.read_signals(r, rsb.producer),
                  "red", w.read_signals(r, rsb.reduction), "ready", w.read_signals(r, agb.ready),
                  "done", w.read_signals(r, agb.done), flush=True)
        w.recover()
        w.zero_all_signals()
print(f"W={W} mode={mode} stage={stage}: {fails}/{iters} failed", flush=True)
