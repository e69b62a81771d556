"""Single-GPU proxy of one tensor-parallel rank (bench.py ``tp8_proxy``).

The gpurun pool grants one B200 per call, so the TP=8 per-rank
configuration of the north star (BASELINE C3 / C4: reference
pipelines.py:126-144 and :201-216 at W=8) cannot run on NVLink here.  This
proxy runs rank 0's REAL kernels at that configuration -- W=8 chunking, 7
flag-gated remote chunks, 7 peer destinations, the 8-slot fused reduction --
with the full persistent grid (``sh_set_rank_solo``), and emulates the 7 peers
with a feeder stream on the same GPU:

* AG (``ag_gemm``, compute half): the feeder copies each peer's shard into
  rank 0's ``gathered`` slot with the copy engine and releases ``ready[src]``
  (per sub-chunk, the library's epoch encoding), paced so that the chunk
  consumed at step i lands when it would over one NVLink ingress at
  ``bw`` bytes/s: the owners push in ring order (``ag_push_order``), so rank 0
  receives one chunk at a time and step i's last byte lands at
  ``i * chunk_bytes / bw``.  Rank 0's own outgoing pushes are not issued: on
  hardware they read the shard from HBM and cross NVLink; the emulated
  incoming copies put the same read + write bytes on this HBM instead.
* RS (``gemm_rs``, fused): rank 0 scatters its partial rows into the 7 peers'
  staging slots (same-GPU memory) and adds to their arrival counters as on
  hardware; the feeder delivers peer s's contribution to rank 0's own chunk
  into staging slot s and sets ``reduction[s]`` at the time peer s finishes
  that chunk under ``rs_inter_order`` -- position 7 - s of 8, i.e. at
  ``(8 - s) / 8`` of a call (calibrated from the same call with everything
  delivered up front).
* Back-pressure words (``done`` / ``producer``) are saturated once: no peer
  ever holds rank 0 back.

Modes: ``preset`` = all remote data and flags in place before the call (the
kernel alone, safe under ncu); ``paced`` = NVLink-paced arrival (what the
exposed-communication figure is taken from).  Not a SCALE substitute: NVLink
contention, peer skew and the copy engines of 7 other GPUs are not modelled.
"""

from __future__ import annotations

import ctypes
import statistics

import torch

import paper_2504_19442_b200 as sb
from paper_2504_19442_b200 import _lib

NVLINK_BW = 770e9  # measured per-direction NVLink 5 rate used across DESIGN.md


def _sub_ranges(rows, S):
    """The library's sub-chunk row ranges (sh_ag_gemm_ex: multiples of 256)."""
    if S <= 1:
        return [(0, rows)]
    sub = ((rows + S - 1) // S + 255) // 256 * 256
    return [(r0, min(sub, rows - r0)) for r0 in range(0, rows, sub)]


class TpProxy:
    """Rank 0 of a W-rank world on one GPU, peers emulated by a feeder."""

    def __init__(self, W, m, n_ag, k_ag, n_rs, k_rs, *, bw=NVLINK_BW, seed=0, timeout_s=20.0):
        self.W = W
        self.bw = bw
        self.ag = sb.ProblemShape(m, n_ag, k_ag, dtype="bfloat16")
        self.rs = sb.ProblemShape(m, n_rs, k_rs, dtype="bfloat16")
        rows = m // W
        self.rows = rows
        ag_bytes = W * rows * k_ag * 2
        rs_bytes = W * rows * n_rs * 2
        heap = ag_bytes + rs_bytes + (8 << 20)
        self.world = sb.init_world(sb.WorldSpec(world_size=W, heap_bytes=heap, timeout_s=timeout_s,
                                                devices=(0,) * W))
        w = self.world
        self.lib = _lib.load()
        _lib.check(self.lib.sh_set_rank_solo(w.handle, 0, 1))
        self.agb = sb.make_ag_gemm_buffers(w, self.ag)
        self.rsb = sb.make_gemm_rs_buffers(w, self.rs)
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev).manual_seed(seed)
        bf = torch.bfloat16
        # rank 0's operands, and every emulated peer's AG shard / RS contribution
        self.x = torch.randn(W, rows, k_ag, device=dev, dtype=bf, generator=g)
        self.b_ag = torch.randn(k_ag, n_ag, device=dev, dtype=bf, generator=g) / k_ag ** 0.5
        self.a_rs = torch.randn(m, k_rs, device=dev, dtype=bf, generator=g)
        self.b_rs = torch.randn(k_rs, n_rs, device=dev, dtype=bf, generator=g) / k_rs ** 0.5
        self.peer_rows = torch.randn(W, rows, n_rs, device=dev, dtype=bf, generator=g)
        self.c = torch.empty(m, n_ag, device=dev, dtype=bf)
        self.y = torch.empty(rows, n_rs, device=dev, dtype=bf)
        self.origin = torch.zeros(1, dtype=torch.int64, device=dev)
        self.main = torch.cuda.Stream(device=dev)
        self.feed = torch.cuda.Stream(device=dev)
        self.ag_order = sb.ag_order_switch(0, W).first_visit_order(W)
        self.rs_order = sb.rs_inter_order(sb.RankCtx(0, 0, 0), 1, W).first_visit_order(W)
        sat = 1 << 62
        h = w.handle
        for base in (self.agb.done.base, self.rsb.producer.base):
            _lib.check(self.lib.sh_fill_signals(h, 0, base, W, sat, ctypes.c_void_p(self.feed.cuda_stream)))
        self.feed.synchronize()
        self.ag_epoch = 0
        self.rs_epoch = 0
        self.t_rs_est_ns = None

    def close(self):
        self.world.close()

    # ------------------------------------------------------------------ AG
    def _ag_call(self, mode, subchunks):
        W, lib, w = self.W, self.lib, self.world
        sh = self.ag
        rows, k = self.rows, sh.k
        chunk = rows * k * 2
        self.ag_epoch += 1
        e = self.ag_epoch
        S = subchunks if subchunks else self._auto_sub()
        ranges = _sub_ranges(rows, S)
        S_eff = len(ranges)
        fs = ctypes.c_void_p(self.feed.cuda_stream)
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        gate = torch.cuda.Event()
        if mode == "paced":
            self.main.wait_stream(self.feed)  # previous call's feeder is done
            gate.record(self.main)
            self.feed.wait_event(gate)
            _lib.check(lib.sh_pace_mark(ctypes.c_void_p(self.origin.data_ptr()), fs))
        else:
            self.feed.wait_stream(self.main)
        landed = 0
        for step in range(1, W):
            c = self.ag_order[step]
            for j, (r0, nr) in enumerate(ranges):
                nbytes = nr * k * 2
                landed += nbytes
                if mode == "paced":
                    _lib.check(lib.sh_pace_wait(ctypes.c_void_p(self.origin.data_ptr()),
                                                int(landed / self.bw * 1e9), fs))
                src = self.x[c].data_ptr() + r0 * k * 2
                _lib.check(lib.sh_putmem(w.handle, c, 0, self.agb.gathered.offset + c * chunk + r0 * k * 2,
                                         ctypes.c_void_p(src), nbytes, fs))
                _lib.check(lib.sh_signal_op(w.handle, c, 0, self.agb.ready.base + c, _lib.SH_SIG_SET,
                                            (e - 1) * S_eff + j + 1, fs))
        if mode != "paced":
            self.main.wait_stream(self.feed)
        ms = ctypes.c_void_p(self.main.cuda_stream)
        start.record(self.main)
        order = _lib.int_array(self.ag_order)
        _lib.check(lib.sh_ag_gemm_ex(w.handle, 0, self.x[0].data_ptr(), self.b_ag.data_ptr(),
                                     self.c.data_ptr(), self.agb.gathered.offset, self.agb.ready.base,
                                     self.agb.done.base, sh.m, sh.n, sh.k, sh.dtype_code, order, e,
                                     S, _lib.SH_PHASE_COMPUTE, ms))
        end.record(self.main)
        return start, end

    def _auto_sub(self):
        out = ctypes.c_int()
        _lib.check(self.lib.sh_ag_subchunks(self.ag.m, self.ag.k, self.W, ctypes.byref(out)))
        return out.value

    # ------------------------------------------------------------------ RS
    def _rs_call(self, mode):
        W, lib, w = self.W, self.lib, self.world
        sh = self.rs
        rows, n = self.rows, sh.n
        slot = rows * n * 2
        self.rs_epoch += 1
        e = self.rs_epoch
        fs = ctypes.c_void_p(self.feed.cuda_stream)
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        gate = torch.cuda.Event()
        if mode == "paced":
            self.main.wait_stream(self.feed)
            gate.record(self.main)
            self.feed.wait_event(gate)
            _lib.check(lib.sh_pace_mark(ctypes.c_void_p(self.origin.data_ptr()), fs))
        else:
            self.feed.wait_stream(self.main)
        # peer s handles chunk 0 at position (0 - s - 1) mod W of rs_inter_order
        arrivals = sorted(((-s - 1) % W, s) for s in range(1, W))
        for pos, s in arrivals:
            if mode == "paced":
                _lib.check(lib.sh_pace_wait(ctypes.c_void_p(self.origin.data_ptr()),
                                            int((pos + 1) / W * self.t_rs_est_ns), fs))
            _lib.check(lib.sh_putmem(w.handle, s, 0, self.rsb.staging.offset + s * slot,
                                     ctypes.c_void_p(self.peer_rows[s].data_ptr()), slot, fs))
            _lib.check(lib.sh_signal_op(w.handle, s, 0, self.rsb.reduction.base + s, _lib.SH_SIG_SET,
                                        e * rows * n, fs))
        if mode != "paced":
            self.main.wait_stream(self.feed)
        ms = ctypes.c_void_p(self.main.cuda_stream)
        start.record(self.main)
        _lib.check(lib.sh_gemm_rs_ex(w.handle, 0, self.a_rs.data_ptr(), self.b_rs.data_ptr(),
                                     self.y.data_ptr(), self.rsb.staging.offset,
                                     self.rsb.producer.base, self.rsb.reduction.base, sh.m, sh.n,
                                     sh.k, sh.dtype_code, _lib.int_array(self.rs_order), e,
                                     _lib.SH_PHASE_ALL, ms))
        end.record(self.main)
        return start, end

    # ------------------------------------------------------------------ driver
    def time_op(self, op, mode, iters, warmup=3, subchunks=0):
        call = (lambda: self._ag_call(mode, subchunks)) if op == "ag" else (lambda: self._rs_call(mode))
        if op == "rs" and mode == "paced" and self.t_rs_est_ns is None:
            self.t_rs_est_ns = statistics.median(self.time_op("rs", "preset", iters, warmup)) * 1e3
        evs = []
        for i in range(warmup + iters):
            ev = call()
            if i >= warmup:
                evs.append(ev)
        self.main.synchronize()
        self.feed.synchronize()
        self.world.check_errors(0)
        return [a.elapsed_time(b) * 1e3 for a, b in evs]  # us

    def check(self):
        """Rank 0's results against torch fp32 (rel-Frobenius, north-star 1e-2)."""
        self.time_op("ag", "preset", 1, warmup=0)
        ref = (self.x.reshape(-1, self.ag.k).float() @ self.b_ag.float())
        err_ag = ((self.c.float() - ref).norm() / ref.norm()).item()
        self.time_op("rs", "preset", 1, warmup=0)
        part = self.a_rs[: self.rows].float() @ self.b_rs.float()
        ref = part.to(torch.bfloat16).float() + self.peer_rows[1:].float().sum(0)
        err_rs = ((self.y.float() - ref).norm() / ref.norm()).item()
        g = self.world.read_tensor(0, self.agb.gathered, torch.bfloat16,
                                   (self.W * self.rows, self.ag.k))
        layout_ok = bool(torch.equal(g.to(self.x.device), self.x.reshape(-1, self.ag.k)))
        return {"ag_rel_fro": err_ag, "rs_rel_fro": err_rs, "gathered_bit_exact": layout_ok}

    def trace_waits(self, op, subchunks=0):
        """One traced paced call: per-CTA exposed waits from the device timeline."""
        from paper_2504_19442_b200 import timeline

        self.world.start_trace()
        try:
            self.time_op(op, "paced", 1, warmup=0, subchunks=subchunks)
        finally:
            ev = self.world.stop_trace()
        summ = [s for s in timeline.exposed_comm(ev) if s["rank"] == 0]
        return summ[-1] if summ else None


def cublas_us(m, n, k, iters=30, warmup=5):
    """torch.matmul (cuBLASLt) of one rank's GEMM, CUDA events, median."""
    dev = torch.device("cuda", 0)
    a = torch.randn(m, k, device=dev, dtype=torch.bfloat16)
    b = torch.randn(k, n, device=dev, dtype=torch.bfloat16)
    out = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    ts = []
    for i in range(warmup + iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=out)
        e.record()
        if i >= warmup:
            ts.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) * 1e3 for x, y in ts)


def run(W=8, m=8192, iters=30, peak_tflops=None, log=print):
    """The tp8_proxy block of bench.py: C3 AG and C4 RS at TP=W, rank 0."""
    import os

    k_full, n_full = 8192, 28672  # Llama-3-70B MLP (BASELINE C3/C4)
    px = TpProxy(W, m, n_full // W, k_full, k_full, n_full // W)
    try:
        out = {"what": f"single-GPU proxy of rank 0 at TP={W} (tp_proxy.py): real kernels, "
                       f"peers emulated by a copy-engine feeder paced at {NVLINK_BW / 1e9:.0f} GB/s",
               "W": W, "ag_shape": {"m": m, "n": n_full // W, "k": k_full},
               "rs_shape": {"m": m, "n": k_full, "k": n_full // W}}
        out["parity"] = px.check()
        flops = 2.0 * m * (n_full // W) * k_full
        nvl_bytes = (W - 1) / W * m * k_full * 2
        res = {}
        for op in ("ag", "rs"):
            pre = statistics.median(px.time_op(op, "preset", iters))
            paced = statistics.median(px.time_op(op, "paced", iters))
            r = {"preset_us": pre, "paced_us": paced, "exposed_us": paced - pre,
                 "tflops_paced": flops / paced / 1e6}
            if peak_tflops:
                t_gemm = flops / (peak_tflops * 1e12) * 1e6
                t_nvl = nvl_bytes / 900e9 * 1e6
                r["roofline_us"] = max(t_gemm, t_nvl)
                r["roofline_frac"] = r["roofline_us"] / paced
            res[op] = r
        # sub-chunk flags and the weighted stream-K partition, A/B on the paced AG
        ab = {}
        for label, env, sub in (("sub1", None, 1), ("sub4", None, 4), ("sub4_nolate", "0,0", 4)):
            if env is None:
                os.environ.pop("SHB_SK_LATE", None)
            else:
                os.environ["SHB_SK_LATE"] = env
            ab[label] = statistics.median([t for t in px.time_op("ag", "paced", iters, subchunks=sub)])
        os.environ.pop("SHB_SK_LATE", None)
        res["ag"]["ab_paced_us"] = ab
        for op in ("ag", "rs"):
            res[op]["trace"] = px.trace_waits(op)
        # unfused: cuBLAS of the same per-rank GEMM + the collective's bytes at
        # the same NVLink rate (modelled: no NCCL peers on a one-GPU box)
        t_comm = nvl_bytes / NVLINK_BW * 1e6
        res["ag"]["unfused_modelled_us"] = cublas_us(m, n_full // W, k_full) + t_comm
        res["rs"]["unfused_modelled_us"] = cublas_us(m, k_full, n_full // W) + t_comm
        for op in ("ag", "rs"):
            res[op]["speedup_vs_unfused_modelled"] = res[op]["unfused_modelled_us"] / res[op]["paced_us"]
        res["unfused_how"] = (f"torch.matmul of the per-rank GEMM (measured) + {nvl_bytes / 1e6:.1f} MB "
                              f"at {NVLINK_BW / 1e9:.0f} GB/s (modelled NCCL transfer, not overlapped)")
        out.update(res)
        return out
    finally:
        px.close()


if __name__ == "__main__":
    import json
    import sys

    sys.stdout.write(json.dumps(run(iters=int(sys.argv[1]) if len(sys.argv) > 1 else 30,
                                    peak_tflops=1700.9)) + "\n")
