"""Quick device timing of a surface-code program (scratch tool, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2507_03092_b200 as sk

d = int(sys.argv[1]) if len(sys.argv) > 1 else 25
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else d
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = sk.Context(0)
circ = sk.surface_code_circuit(d, rounds, True)
t0 = time.time(); prog = sk.Program(ctx, circ); t1 = time.time()
print(f"d={d} n={circ.n} gates={len(circ.gates)} meas={circ.num_measurements} program_create={t1-t0:.3f}s")
tab = sk.Tableau(ctx, circ.n)
stream = torch.cuda.ExternalStream(ctx.stream)
for rep in range(reps):
    tab.reset(); ctx.reset_counters(); ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream); prog.run(tab, 20250703); e1.record(stream)
    w1 = time.time(); ctx.sync(); w2 = time.time()
    out, det = prog.read_record()
    c = ctx.counters()
    print(f"rep{rep}: device {e0.elapsed_time(e1):.3f} ms  enqueue {1e3*(w1-w0):.2f} ms  wall {1e3*(w2-w0):.2f} ms  "
          f"n_rand={c['n_rand']} n_det={c['n_det']} k_rand={c['k_rand']} k_det={c['k_det']} waves={c['waves']} layers={c['layers']} "
          f"transposes={c['transposes']} launches={c['kernel_launches']}")
    print("   meas phases us [P1,P2,gather,factorise,values+detA,apply+detB,bar(wave),bar(panel)]:", [round(v/1e3) for v in c["meas_phase_ns"][:8]])
print("outcome checksum", int(out.sum()), int(det.sum()))
