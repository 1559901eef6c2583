"""Grouping (config C4) at a given N and mode, for profiling: python tools/group_time.py N mode(0 GC|1 QWC)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_03092_b200 as sk
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rng = np.random.default_rng(20250703)
x = rng.integers(0, 2**64, (N, 2), dtype=np.uint64); z = rng.integers(0, 2**64, (N, 2), dtype=np.uint64); r = np.zeros(N, np.uint8)
ctx = sk.Context(0)
rows = sk.Rows(ctx, 128, x, z, r)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    ctx.sync(); t0 = time.perf_counter()
    g, ng = rows.group_first_fit(mode)
    ctx.sync(); dt = time.perf_counter() - t0
    print(f"N={N} mode={mode}: {dt:.3f} s, {ng} groups, {N*(N-1)/2/dt:.3e} pairs/s")
