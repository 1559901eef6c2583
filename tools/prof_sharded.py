import sys, os, cProfile, pstats
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2507_03092_b200 as sk
from paper_2507_03092_b200.sharded import ShardedTableau
circ = sk.surface_code_circuit(71, 71, True)
for rep in range(2):
    t = ShardedTableau.create_cuda(circ.n, local_shards=1, device_index=0)
    if rep == 1:
        pr = cProfile.Profile(); pr.enable()
    out, det = t.sim(circ, 20250703)
    t.stream.synchronize()
    if rep == 1:
        pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
    t.close()
