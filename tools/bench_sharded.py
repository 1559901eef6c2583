#!/usr/bin/env python
"""Row-sharded tableau (paper_2507_03092_b200/sharded.py) timed on ONE GPU with 1..8 shards resident on it
(the in-process exchange), next to the unsharded engine on the same circuit; records must be identical.
Under torchrun the same script runs one shard per rank over NCCL (--local-shards 1).

    python tools/bench_sharded.py [--d 25 71] [--shards 1 2 4 8] [--out gpurun_out/sharded.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SEED = 20250703


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, nargs="+", default=[25, 71])
    ap.add_argument("--shards", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    import paper_2507_03092_b200 as sk
    from paper_2507_03092_b200 import dist as skdist
    from paper_2507_03092_b200.sharded import ShardedTableau
    rank, local_rank, world = skdist.init()
    rows = []
    for d in args.d:
        circ = sk.surface_code_circuit(d, d, True)
        ctx = sk.Context(local_rank)
        t1, out1, det1, _ = ctx.sim(circ, SEED); t1.close()
        t0 = time.perf_counter(); t1, out1, det1, _ = ctx.sim(circ, SEED); ctx.sync(); single_s = time.perf_counter() - t0
        t1.close(); ctx.close()
        for L in args.shards:
            t = ShardedTableau.create_cuda(circ.n, local_shards=L, device_index=local_rank)
            skdist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(t.stream)
            t0 = time.perf_counter()
            out, det = t.sim(circ, SEED)
            e1.record(t.stream); t.stream.synchronize()
            wall = time.perf_counter() - t0
            dev_s = skdist.max_over_ranks(e0.elapsed_time(e1) * 1e-3)
            ok = bool((out == out1).all() and (det == det1).all())
            k = [s.counters() for s in t.shards]
            row = {"d": d, "n": circ.n, "ranks": world, "local_shards": L, "global_shards": world * L, "sharded_s": dev_s, "wall_s": wall,
                   "unsharded_sk_sim_s": single_s, "record_identical": ok, "n_rand": t.stats["n_rand"], "n_det": t.stats["n_det"],
                   "pivot_searches": t.stats["searches"], "collectives": dict(t.ex.calls), "exchange_bytes": t.ex.bytes,
                   "k_rand_per_shard": [a for a, _ in k], "k_det_per_shard": [b for _, b in k]}
            t.close()
            if rank == 0:
                print(json.dumps(row), flush=True)
            rows.append(row)
            assert ok, "sharded record differs from the unsharded engine"
    if args.out and rank == 0:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)
    skdist.finalize()


if __name__ == "__main__":
    main()
