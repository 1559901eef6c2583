"""quick_time.py without the final data-qubit measurement block (scratch tool: isolates the cost of that block)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_03092_b200 as sk
d = int(sys.argv[1]); rounds = int(sys.argv[2]); final = int(sys.argv[3])
ctx = sk.Context(0)
circ = sk.surface_code_circuit(d, rounds, bool(final))
prog = sk.Program(ctx, circ); tab = sk.Tableau(ctx, circ.n)
stream = torch.cuda.ExternalStream(ctx.stream)
for rep in range(3):
    tab.reset(); ctx.reset_counters(); ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); prog.run(tab, 20250703); e1.record(stream); ctx.sync()
    c = ctx.counters()
    print(f"final={final} rounds={rounds}: device {e0.elapsed_time(e1):.3f} ms n_rand={c['n_rand']} k_rand={c['k_rand']} phases", [round(v/1e3) for v in c["meas_phase_ns"][:8]])
