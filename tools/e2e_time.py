import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_03092_b200 as sk
ctx = sk.Context(0)
circ = sk.surface_code_circuit(71, 71, True)
for i in range(3):
    t0 = time.perf_counter(); tt, o, d, _ = ctx.sim(circ, 1); ctx.sync(); t1 = time.perf_counter(); tt.close(); t2 = time.perf_counter()
    print(f"sim {1e3*(t1-t0):.1f} ms  close {1e3*(t2-t1):.1f} ms")
