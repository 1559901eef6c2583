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
