"""Per kernel-class device time of a surface-code program (CUDA events around every op)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_03092_b200 as sk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 71
ctx = sk.Context(0)
circ = sk.surface_code_circuit(d, d, True)
prog = sk.Program(ctx, circ); tab = sk.Tableau(ctx, circ.n)
for rep in range(3):
    tab.reset(); ctx.sync()
    print(prog.run_profiled(tab, 20250703))
