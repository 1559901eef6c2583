"""-m gpu: the row-sharded tableau (sk_shard_* C ABI + paper_2507_03092_b200/sharded.py) against the CPU oracle.
Several shards live on the one GPU of the test box (`local_shards`), so the whole protocol -- pivot candidates
min-reduced over shards, pivot row handed from its owner to every shard, partial products multiplied in shard
order -- runs through the CUDA kernels; with torch.distributed the same calls go over NCCL."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

H, S, SDG, X, Y, Z, CX, CZ, SWAP, M, T, TDG = range(12)
SEED = 20250703


def run_both(sk, orc, circ, seed, local_shards):
    """Both ways a random measurement block can run: on the tableau assembled from all shards (the default: one allgather of
    the rows per block) and with an exchange per measurement (replicate_random_blocks = False)."""
    run_one(sk, orc, circ, seed, local_shards, False)
    return run_one(sk, orc, circ, seed, local_shards, True)


def run_one(sk, orc, circ, seed, local_shards, replicate):
    from paper_2507_03092_b200.sharded import ShardedTableau
    t = ShardedTableau.create_cuda(circ.n, local_shards=local_shards, device_index=0)
    t.replicate_random_blocks = replicate
    try:
        out, det = t.sim(circ, seed)
        x, z, r = t.gather_tableau()
        stats = dict(t.stats)
        k = [s.counters() for s in t.shards]
    finally:
        t.close()
    o = orc.Tableau(circ.n)
    oo, od, rc = o.sim(circ.gates, seed)
    assert rc == 0
    ox, oz, orr = o.get()
    assert (det == od).all(), "deterministic flags differ"
    assert (out == oo).all(), "outcomes differ"
    assert (x == ox).all() and (z == oz).all(), "tableau bits differ"
    assert (r == orr).all(), "signs differ"
    assert stats["n_rand"] == int((od == 0).sum()) and stats["n_det"] == int((od == 1).sum())
    if (od == 0).any(): assert (stats["replicated_blocks"] >= 1) == replicate
    return stats, k


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
@pytest.mark.parametrize("d", [3, 5, 7])
def test_surface_code_sharded_matches_oracle(sk, orc, d, shards):
    run_both(sk, orc, sk.surface_code_circuit(d, d, True), SEED, shards)


@pytest.mark.parametrize("shards", [2, 4])
@pytest.mark.parametrize("n", [64, 200])
def test_random_layered_sharded_matches_oracle(sk, orc, n, shards):
    run_both(sk, orc, sk.random_layered_circuit(n, 11 + n), 7, shards)


@pytest.mark.parametrize("n,shards", [(1, 1), (5, 2), (65, 2), (130, 3), (257, 4), (300, 8)])
def test_random_circuits_with_measurements_sharded(sk, orc, n, shards):
    rng = np.random.default_rng(1000 + n)
    gates = []
    for _ in range(300 + 4 * n):
        if rng.random() < 0.2:
            gates.append((M, int(rng.integers(0, n)), 0)); continue
        k = int(rng.choice([H, S, SDG, X, Y, Z, CX, CZ, SWAP]))
        a = int(rng.integers(0, n)); b = 0
        if k in (CX, CZ, SWAP):
            if n == 1: k = H
            else: b = int(rng.integers(0, n - 1)); b += b >= a
        gates.append((k, a, b))
    run_both(sk, orc, sk.Circuit(n, gates), 99, shards)


def test_sharded_equals_unsharded_engine_d25_first_round(sk, ctx, orc):
    """config C2's circuit cut to 2 rounds: sharded record == single-GPU sk_sim record (and the oracle's)."""
    circ = sk.surface_code_circuit(25, 2, True)
    t1, out1, det1, _ = ctx.sim(circ, SEED)
    t1.close()
    from paper_2507_03092_b200.sharded import ShardedTableau
    t = ShardedTableau.create_cuda(circ.n, local_shards=4, device_index=0)
    try:
        out, det = t.sim(circ, SEED)
    finally:
        t.close()
    assert (out == out1).all() and (det == det1).all()


def test_shard_argument_errors(sk, ctx):
    import ctypes as C
    L = sk.lib()
    h = C.c_void_p()
    assert L.sk_shard_create(ctx._h, 0, 0, 0, C.byref(h)) == sk.SK_EDIM
    assert L.sk_shard_create(ctx._h, 10, 4, 11, C.byref(h)) == sk.SK_EDIM
    assert L.sk_shard_create(ctx._h, 100, 64, 100, C.byref(h)) == sk.SK_OK
    buf = (C.c_uint64 * 64)()
    assert L.sk_shard_pivot_row(h, 3, buf) == sk.SK_EDIM          # stabilizer 3 lives in another shard
    g = sk.gates_array([(T, 0, 0)])
    assert L.sk_shard_apply_gates(h, g.ctypes.data_as(C.c_void_p), 1) == sk.SK_EUNSUPPORTED
    L.sk_shard_destroy(h)


def test_two_processes_one_shard_each_over_a_process_group(sk, orc):
    """Two OS processes, one CudaShard each (both on GPU 0), exchanging through torch.distributed.  NCCL refuses two
    ranks on one device, so the group is gloo with the device buffers staged through the host; the driver code and
    every kernel are the ones an NCCL job runs."""
    import os, socket, subprocess, sys, textwrap
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = textwrap.dedent("""
        import sys
        sys.path.insert(0, %r)
        import numpy as np
        import paper_2507_03092_b200 as sk
        from paper_2507_03092_b200 import dist
        from paper_2507_03092_b200.sharded import ShardedTableau
        from oracle import oracle_py as orc
        rank, local_rank, world = dist.init("gloo")
        for circ, seed in ((sk.surface_code_circuit(7, 7, True), 20250703), (sk.random_layered_circuit(128, 3), 5)):
          for replicate in (True, False):
            t = ShardedTableau.create_cuda(circ.n, local_shards=1, device_index=0)
            t.replicate_random_blocks = replicate
            out, det = t.sim(circ, seed)
            x, z, r = t.gather_tableau()
            calls = dict(t.ex.calls); nrep = t.stats["replicated_blocks"]
            t.close()
            o = orc.Tableau(circ.n)
            oo, od, rc = o.sim(circ.gates, seed)
            ox, oz, orr = o.get()
            assert rc == 0 and (out == oo).all() and (det == od).all(), "record differs from the oracle"
            assert (x == ox).all() and (z == oz).all() and (r == orr).all(), "tableau differs from the oracle"
            assert calls["allgather"] >= 1 and calls["allreduce_min"] >= 1
            if replicate: assert calls["broadcast"] == 0 and nrep >= 1
            else: assert calls["broadcast"] == int((od == 0).sum())
        dist.finalize()
        print("rank", rank, "ok")
    """ % root)
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK="0", WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", script], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=280)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    assert "rank 0 ok" in outs[0] and "rank 1 ok" in outs[1], outs


@pytest.mark.parametrize("local", [1, 2, 3, 4])
def test_grouping_sharded_by_row_blocks(sk, ctx, orc, local):
    """SURVEY 8e, second row: first fit with the pair matrix sharded by row blocks (sk_group_shard_*; shard s evaluates the
    groups of the bitmap words w % S == s); S local shards on one device, bitmaps OR-ed in process.  Groups identical to the
    oracle and to the unsharded sk_group_first_fit, GC and QWC."""
    from paper_2507_03092_b200.group_sharded import group_first_fit_cuda
    rng = np.random.default_rng(17 + local)
    for n, m, dens in ((128, 6000, 0.5), (128, 3000, 0.03), (40, 2500, 0.3)):
        W = (n + 63) // 64
        bits = rng.random((2, m, n)) < dens
        x = np.zeros((m, W), np.uint64); z = np.zeros((m, W), np.uint64)
        for q in range(n):
            x[:, q >> 6] |= bits[0, :, q].astype(np.uint64) << np.uint64(q & 63); z[:, q >> 6] |= bits[1, :, q].astype(np.uint64) << np.uint64(q & 63)
        rows = sk.Rows(ctx, n, x, z); o = orc.Rows(n, x, z, np.zeros(m, np.uint8))
        for mode in (0, 1):
            (g, ng), ex = group_first_fit_cuda(rows, mode, local_shards=local, device_index=0)
            og, ong, _ = o.group_first_fit(mode)
            assert ng == ong and (g == og).all(), (n, m, mode)
            g1, ng1 = rows.group_first_fit(mode)
            assert ng1 == ng and (g1 == g).all()
        rows.close()
    wide = sk.Rows(ctx, 200, np.ones((4, 4), np.uint64), np.zeros((4, 4), np.uint64))
    with pytest.raises(sk.UnsupportedError): group_first_fit_cuda(wide, 0, local_shards=2, device_index=0)
