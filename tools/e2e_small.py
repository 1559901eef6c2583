"""sk_sim end to end (host buffers) at several distances: python tools/e2e_small.py [d ...]"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03092_b200 as sk
ctx = sk.Context(0)
for d in [int(x) for x in sys.argv[1:]] or [5, 11, 25, 41, 71]:
    circ = sk.surface_code_circuit(d, d, True); circ.num_measurements
    ts = []
    for i in range(8):
        t0 = time.perf_counter(); tt, o, dd, _ = ctx.sim(circ, 1); ctx.sync(); ts.append(time.perf_counter() - t0); tt.close()
    print(f"d={d}: sk_sim e2e min {1e3*min(ts[3:]):.2f} ms  median {1e3*sorted(ts[3:])[2]:.2f} ms")
