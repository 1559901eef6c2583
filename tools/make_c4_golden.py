"""Golden group checksums of config C4 at full size (N = 10^6 random 128-qubit Paulis, GC and QWC first fit) from the CPU
oracle -- about 10-20 minutes per mode on one core, so it is run once here and the result committed as
tests/golden/c4_groups_1e6.json; tests/test_gpu_rows_parity.py compares the device's groups with it.
Usage: python tools/make_c4_golden.py [N]"""
import hashlib, importlib.util, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from oracle import oracle_py as orc
spec = importlib.util.spec_from_file_location("workloads", os.path.join(ROOT, "paper_2507_03092_b200", "workloads.py"))   # no CUDA library needed
wl = importlib.util.module_from_spec(spec); spec.loader.exec_module(wl)

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
x, z, coeff = wl.c4_terms(N)
out = {"N": N, "n": 128, "seed": 20250703, "generator": "paper_2507_03092_b200/workloads.py c4_terms", "modes": {}}
for mode, name in ((0, "GC"), (1, "QWC")):
    o = orc.Rows(128, x, z, np.zeros(N, np.uint8))
    t0 = time.perf_counter(); g, ng, calls = o.group_first_fit(mode); dt = time.perf_counter() - t0
    g = np.ascontiguousarray(g, np.uint32)
    out["modes"][name] = {"groups": int(ng), "sha256": hashlib.sha256(g.tobytes()).hexdigest(), "predicate_calls": int(calls), "oracle_seconds": round(dt, 1),
                          "first16": g[:16].tolist(), "last4": g[-4:].tolist()}
    print(name, out["modes"][name], flush=True)
path = os.path.join(ROOT, "tests", "golden", f"c4_groups_{N}.json")
json.dump(out, open(path, "w"), indent=1)
print("wrote", path)
