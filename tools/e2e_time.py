"""End-to-end time of `sk_sim` with host buffers at d=71 (argv[1] = repetitions, default 3): per-call wall clock and the median.
SK_DEBUG_E2E=1 prints the host-side stage times of every call on stderr."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_03092_b200 as sk
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = sk.Context(0)
circ = sk.surface_code_circuit(71, 71, True)
ts = []
for i in range(reps):
    t0 = time.perf_counter(); tt, o, d, _ = ctx.sim(circ, 1); ctx.sync(); t1 = time.perf_counter(); tt.close(); t2 = time.perf_counter()
    ts.append(1e3 * (t1 - t0))
    if reps <= 5: print(f"sim {1e3*(t1-t0):.1f} ms  close {1e3*(t2-t1):.1f} ms")
w = sorted(ts[2:]) if reps > 4 else sorted(ts)
print(f"median of {len(w)} calls (first two dropped when reps > 4): {w[len(w)//2]:.2f} ms  min {w[0]:.2f}  max {w[-1]:.2f}  checksum {int(o.sum())} {int(d.sum())}")
