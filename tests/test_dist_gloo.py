"""N > 1 host logic of bench.py on CPU: world_size 2, gloo, 127.0.0.1."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p


def test_slot_ranges_partition_the_rows():
    sys.path.insert(0, ROOT)
    from paper_2507_03092_b200 import dist
    for n in (1, 17, 64, 65, 1249, 10081):
        for world in (1, 2, 4, 8):
            rs = [dist.slot_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a <= b and (b % 64 == 0 or b == n)
    assert dist.shot_seed(20250703, 0) == 20250703 and dist.shot_seed(20250703, 3) == 20250703 ^ 3


def test_world_size_2_gloo_replicas():
    script = textwrap.dedent("""
        import os, sys
        sys.path.insert(0, %r)
        from paper_2507_03092_b200 import dist
        rank, local_rank, world = dist.init("gloo")
        assert world == 2
        seed = dist.shot_seed(20250703, rank)
        dist.barrier()
        t = dist.max_over_ranks(10.0 + rank)            # rank 1 is the slow one
        assert t == 11.0, t
        sums = dist.gather_records(1000 + seed)
        assert sums == [1000 + 20250703, 1000 + (20250703 ^ 1)], sums
        lo, hi = dist.slot_range(10081, rank, world)
        assert (lo, hi) == ((0, 5056), (5056, 10081))[rank]
        dist.finalize()
        print("rank", rank, "ok")
    """ % ROOT)
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", script], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=180)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    assert "rank 0 ok" in outs[0] and "rank 1 ok" in outs[1]


def _run_two_ranks(script):
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, "-c", script], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs
    assert "rank 0 ok" in outs[0] and "rank 1 ok" in outs[1], outs


def test_world_size_2_gloo_row_sharded_protocol():
    """The row-sharded driver (paper_2507_03092_b200/sharded.py) over a real 2-rank process group: allreduce-min of
    the pivot candidates, broadcast of the pivot row, allgather of the partial products.  The per-shard arithmetic
    is tests/shard_stub.py here (no GPU in this container); on the GPU box the same driver runs on CudaShard
    (tests/test_gpu_sharded.py).  2 ranks x 2 local shards = 4 global shards; record and tableau == oracle."""
    script = textwrap.dedent("""
        import os, sys
        sys.path.insert(0, %r)
        import numpy as np
        import paper_2507_03092_b200 as sk
        from paper_2507_03092_b200 import dist
        from paper_2507_03092_b200.sharded import ShardedTableau, Exchange, counter_bit
        from tests.shard_stub import StubShard
        from oracle import oracle_py as orc
        rank, local_rank, world = dist.init("gloo")
        assert world == 2
        rng = np.random.default_rng(5)
        n = 70
        gates = []
        for _ in range(500):
            u = rng.random()
            if u < 0.2: gates.append((9, int(rng.integers(0, n)), 0)); continue
            k = int(rng.choice([0, 1, 2, 3, 4, 5, 6, 7, 8])); a = int(rng.integers(0, n)); b = 0
            if k >= 6: b = int(rng.integers(0, n - 1)); b += b >= a
            gates.append((k, a, b))
        for circ, seed in ((sk.surface_code_circuit(3, 3, True), 20250703), (sk.surface_code_circuit(5, 2, True), 1), (sk.Circuit(n, gates), 99)):
          for replicate in (True, False):       # random blocks on the assembled tableau (default) / exchange per measurement
            ex = Exchange(2)
            assert ex.nshards == 4
            shards = [StubShard(circ.n, *dist.slot_range(circ.n, rank * 2 + l, 4)) for l in range(2)]
            t = ShardedTableau(circ.n, shards, ex)
            t.replicate_random_blocks = replicate
            out, det = t.sim(circ, seed)
            x, z, r = t.gather_tableau()
            o = orc.Tableau(circ.n)
            oo, od, rc = o.sim(circ.gates, seed)
            ox, oz, orr = o.get()
            assert rc == 0 and (out == oo).all() and (det == od).all(), "record differs from the oracle"
            assert (x == ox).all() and (z == oz).all() and (r == orr).all(), "tableau differs from the oracle"
            assert ex.calls["allreduce_min"] >= 1 and ex.calls["allgather"] >= 1
            assert t.stats["n_rand"] == int((od == 0).sum()) and t.stats["n_det"] == int((od != 0).sum())
            if (od == 0).any():
                if replicate: assert ex.calls["broadcast"] == 0 and t.stats["replicated_blocks"] >= 1
                else: assert ex.calls["broadcast"] == int((od == 0).sum()) and t.stats["replicated_blocks"] == 0
        # CounterRng bits (ref: rng.hpp:33-39; SURVEY 8c probe values)
        assert "".join(str(counter_bit(0, i)) for i in range(32)) == "01111010000000100000010000111101"
        assert "".join(str(counter_bit(7, i)) for i in range(32)) == "01010011011101100101001001101001"
        dist.finalize()
        print("rank", rank, "ok")
    """ % ROOT)
    _run_two_ranks(script)


def test_world_size_2_gloo_grouping_sharded_by_row_blocks():
    """SURVEY 8e, second row: the grouping driver (paper_2507_03092_b200/group_sharded.py) over a real 2-rank process group --
    2 ranks x 2 local shards = 4 global shards, each evaluating the predicates of its own bitmap words; the block bitmaps are
    OR-combined by an allreduce-SUM; every shard resolves the block itself.  Per-shard arithmetic is tests/group_shard_stub.py
    here (no GPU in this container; the CUDA shards run the same driver in tests/test_gpu_sharded.py).  Groups == oracle."""
    script = textwrap.dedent("""
        import os, sys
        sys.path.insert(0, %r)
        import numpy as np
        from paper_2507_03092_b200 import dist
        from paper_2507_03092_b200.group_sharded import GroupExchange, group_first_fit_sharded
        from tests.group_shard_stub import StubGroupShard
        from oracle import oracle_py as orc
        rank, local_rank, world = dist.init("gloo")
        rng = np.random.default_rng(3)                   # same input on every rank (the term list is replicated)
        for n, m, mode in ((128, 2600, 0), (128, 2100, 1), (20, 1500, 0)):
            W = (n + 63) // 64
            x = rng.integers(0, 1 << 62, (m, W), dtype=np.uint64); z = rng.integers(0, 1 << 62, (m, W), dtype=np.uint64)
            if n < 64: x &= np.uint64((1 << n) - 1); z &= np.uint64((1 << n) - 1)
            ex = GroupExchange(2)
            assert ex.nshards == 4
            shards = [StubGroupShard(x, z, mode, ex.rank * 2 + l, ex.nshards) for l in range(2)]
            g, ng = group_first_fit_sharded(shards, ex)
            og, ong, _ = orc.Rows(n, x, z, np.zeros(m, np.uint8)).group_first_fit(mode)
            assert ng == ong and (g == og).all(), (n, m, mode, ng, ong)
            assert ex.calls == shards[0].blocks
        dist.finalize()
        print("rank", rank, "ok")
    """ % ROOT)
    _run_two_ranks(script)
