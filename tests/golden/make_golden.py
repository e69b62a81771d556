"""Generate golden fixtures by running the REFERENCE implementation.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports the reference package `minishmem` in place from
/root/reference/pkg/src (read-only; only in the build container -- the GPU box
never reads /root/reference) and records, for small seeded problems:

* ag_gemm outputs and the bit-exact `gathered` layout (pipelines.py:97-150),
* gemm_rs outputs and the bit-exact `staging` layout (pipelines.py:179-233),
* schedule orders from swizzle.py (ag_order_switch / ag_order_fullmesh /
  rs_inter_order) for several world sizes,

into tests/golden/*.npz / schedules.json.  Integer (int64) payloads with small
magnitudes make every value exact in bf16 too, so the same fixtures pin the
GPU path bit-exactly; one fp32 case pins the float path within tolerance.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from minishmem import RankCtx, WorldSpec, init_world
    from minishmem.pipelines import (ProblemShape, ag_gemm, gemm_rs, make_ag_gemm_buffers,
                                     make_gemm_rs_buffers)
    from minishmem.swizzle import ag_order_fullmesh, ag_order_switch, rs_inter_order

    # ---------------------------------------------------------------- schedules
    sched = {"ag_order_switch": {}, "rs_inter_order_1node": {}, "ag_order_fullmesh": {},
             "rs_inter_order_2node": {}}
    for w in (1, 2, 3, 4, 8, 16):
        sched["ag_order_switch"][w] = [ag_order_switch(r, w).chunk_order() for r in range(w)]
        sched["rs_inter_order_1node"][w] = [
            rs_inter_order(RankCtx(r, 0, r), 1, w).chunk_order() for r in range(w)]
        sched["ag_order_fullmesh"][w] = [
            [[s.chunk, s.subchunk] for s in ag_order_fullmesh(r, w, 3).steps] for r in range(w)]
    for lws in (2, 4):
        w = 2 * lws
        sched["rs_inter_order_2node"][w] = [
            rs_inter_order(RankCtx(r, r // lws, r % lws), 2, lws).chunk_order() for r in range(w)]
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(sched, f, indent=1, sort_keys=True)

    # ---------------------------------------------------------------- pipelines
    def run_ag(w, m, n, k, dtype, seed, lo=-2, hi=3):
        rng = np.random.default_rng(seed)
        rows = m // w
        if dtype == "int64":
            shards = [rng.integers(lo, hi, (rows, k)).astype(np.int64) for _ in range(w)]
            bs = [rng.integers(-1, 2, (k, n)).astype(np.int64) for _ in range(w)]
        else:
            shards = [rng.standard_normal((rows, k)).astype(np.float32) for _ in range(w)]
            bs = [rng.standard_normal((k, n)).astype(np.float32) for _ in range(w)]
        shape = ProblemShape(m=m, n=n, k=k, dtype=dtype)
        spec = WorldSpec(world_size=w, heap_bytes=w * rows * k * 8 + (1 << 16))
        with init_world(spec) as world:
            bufs = make_ag_gemm_buffers(world, shape)
            outs = world.run(lambda pe: ag_gemm(pe, shards[pe.rank], bs[pe.rank], shape,
                                                ag_order_switch(pe.rank, w), bufs))
            gathered = [np.frombuffer(world.read_from(r, bufs.gathered, 0, bufs.gathered.length),
                                      dtype=dtype).reshape(m, k) for r in range(w)]
        return dict(shards=np.stack(shards), b=np.stack(bs), out=np.stack(outs),
                    gathered=np.stack(gathered))

    def run_rs(w, m, n, k, dtype, seed):
        rng = np.random.default_rng(seed)
        rows = m // w
        if dtype == "int64":
            amats = [rng.integers(-2, 3, (m, k)).astype(np.int64) for _ in range(w)]
            bs = [rng.integers(-1, 2, (k, n)).astype(np.int64) for _ in range(w)]
        else:
            amats = [rng.standard_normal((m, k)).astype(np.float32) for _ in range(w)]
            bs = [rng.standard_normal((k, n)).astype(np.float32) for _ in range(w)]
        shape = ProblemShape(m=m, n=n, k=k, dtype=dtype)
        spec = WorldSpec(world_size=w, heap_bytes=w * rows * n * 8 + (1 << 16))
        with init_world(spec) as world:
            bufs = make_gemm_rs_buffers(world, shape)
            outs = world.run(lambda pe: gemm_rs(pe, amats[pe.rank], bs[pe.rank], shape,
                                                rs_inter_order(pe.ctx, 1, w), bufs))
            staging = [np.frombuffer(world.read_from(r, bufs.staging, 0, bufs.staging.length),
                                     dtype=dtype).reshape(w, rows, n) for r in range(w)]
        return dict(a=np.stack(amats), b=np.stack(bs), out=np.stack(outs),
                    staging=np.stack(staging))

    cases = {
        "ag_w2_int": run_ag(2, 256, 64, 128, "int64", 1),
        "ag_w4_int": run_ag(4, 512, 128, 64, "int64", 2),
        "ag_w8_int": run_ag(8, 2048, 64, 64, "int64", 3),
        "ag_w2_f32": run_ag(2, 256, 64, 128, "float32", 4),
        "rs_w2_int": run_rs(2, 512, 64, 64, "int64", 5),
        "rs_w4_int": run_rs(4, 1024, 64, 64, "int64", 6),
        "rs_w8_int": run_rs(8, 2048, 64, 64, "int64", 7),
        "rs_w4_f32": run_rs(4, 1024, 64, 64, "float32", 8),
    }
    for name, arrays in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
        print(name, {k: v.shape for k, v in arrays.items()})


if __name__ == "__main__":
    main()
