"""Row-sharded CHP tableau across GPUs (north_star "Multi-GPU sharding").

One process per GPU (torch.distributed, NCCL); every process owns one or more ROW SHARDS of the
same tableau: shard g holds the slots `dist.slot_range(n, g, G)` = stabilizer i and destabilizer i
for i in the range.  All arithmetic is in the CUDA kernels behind the `sk_shard_*` C ABI
(csrc/kernels_shard.cuh); this module is the host driver that strings them together with the three
exchanges a measurement needs:

  Clifford gates        no communication (rows are independent)
  pivot search          allreduce-MIN of one int32 per pending measurement
  random measurement    broadcast of the pivot row from its owner (16*Wp + 16 bytes), every shard
                        rowsums its own rows, the owner rewrites the pair
  deterministic ones    batched: ONE allgather of the shards' partial products for a whole run of
                        deterministic measurements, multiplied in shard order (valid
                        because Pauli multiplication is associative)

`local_shards > 1` puts several shards on one GPU: the same code path with the exchange done in
process, which is how the protocol is verified on a single B200 (tests/test_gpu_sharded.py).
The tableau, signs and measurement record are bit-identical to the unsharded engine.
There is no CPU implementation of a shard in this package: `CudaShard` needs the CUDA library.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import dist as skdist

NONE = 0x7F7F7F7F          # kShardNone in csrc/kernels_shard.cuh
_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """ref: proj/include/stabkit/rng.hpp:23-28"""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def counter_bit(seed: int, ordinal: int) -> int:
    """CounterRng{seed}.bit(ordinal), ref: proj/include/stabkit/rng.hpp:33-39"""
    return splitmix64((seed & _M64) ^ splitmix64((ordinal ^ 0xD1B54A32D192ED03) & _M64)) & 1


class CudaShard:
    """One sk_shard.  Exchange buffers are torch CUDA tensors whose pointers go through the C ABI."""

    def __init__(self, ctx, n: int, lo: int, hi: int, device):
        import torch
        from . import lib
        self._torch, self._lib = torch, lib()
        self.ctx, self.n, self.lo, self.hi, self.device = ctx, int(n), int(lo), int(hi), device
        self.W = (self.n + 63) // 64
        self._h = C.c_void_p()
        ctx.check(self._lib.sk_shard_create(ctx._h, n, lo, hi, C.byref(self._h)))
        self.PW = int(self._lib.sk_shard_partial_words(self._h))

    def close(self):
        if self._h and self.ctx._h:
            self._lib.sk_shard_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def apply_gates(self, gates: np.ndarray):
        self.ctx.check(self._lib.sk_shard_apply_gates(self._h, gates.ctypes.data_as(C.c_void_p), len(gates)))

    def pivot_search(self, qubits: np.ndarray):
        out = self._torch.empty(len(qubits), dtype=self._torch.int32, device=self.device)
        self.ctx.check(self._lib.sk_shard_pivot_search(self._h, qubits.ctypes.data_as(C.c_void_p), len(qubits), C.c_void_p(out.data_ptr())))
        return out

    def det_partial(self, qubits: np.ndarray):
        out = self._torch.empty((len(qubits), self.PW), dtype=self._torch.int64, device=self.device)
        self.ctx.check(self._lib.sk_shard_det_partial(self._h, qubits.ctypes.data_as(C.c_void_p), len(qubits), C.c_void_p(out.data_ptr())))
        return out

    def det_combine(self, gathered) -> np.ndarray:
        g, m, pw = gathered.shape
        assert pw == self.PW and gathered.is_contiguous()
        out = np.zeros(m, np.uint8)
        self.ctx.check(self._lib.sk_shard_det_combine(self._h, C.c_void_p(gathered.data_ptr()), g, m, out.ctypes.data_as(C.c_void_p)))
        return out

    def pivot_row(self, p: int):
        out = self._torch.empty(self.PW, dtype=self._torch.int64, device=self.device)
        self.ctx.check(self._lib.sk_shard_pivot_row(self._h, p, C.c_void_p(out.data_ptr())))
        return out

    def new_row_buffer(self):
        return self._torch.empty(self.PW, dtype=self._torch.int64, device=self.device)

    def random_update(self, q: int, p: int, row, outcome: int):
        self.ctx.check(self._lib.sk_shard_random_update(self._h, q, p, C.c_void_p(row.data_ptr()), outcome))

    # -- replicated elimination of a random block: rows as one contiguous device block -----------------------
    def block_words(self, nloc: int | None = None) -> int:
        nloc = (self.hi - self.lo) if nloc is None else nloc
        Wp = (self.W + 1) & ~1
        return 4 * nloc * Wp + 2 * ((nloc + 63) // 64)

    def new_block(self, words: int):
        return self._torch.zeros(max(words, 1), dtype=self._torch.int64, device=self.device)

    def export_rows(self, buf):
        self.ctx.check(self._lib.sk_shard_export_rows(self._h, C.c_void_p(buf.data_ptr())))

    def import_rows(self, buf):
        self.ctx.check(self._lib.sk_shard_import_rows(self._h, C.c_void_p(buf.data_ptr())))

    def make_full(self):
        """The full tableau the blocks of all shards are assembled in (single-GPU engine, same context / stream)."""
        return _CudaFull(self.ctx, self.n)

    def download(self):
        nloc = self.hi - self.lo
        x = np.zeros((2 * nloc, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(2 * nloc, np.uint8)
        self.ctx.check(self._lib.sk_shard_download(self._h, x.ctypes.data_as(C.c_void_p), z.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p)))
        return x, z, r

    def counters(self):
        out = (C.c_uint64 * 2)()
        self.ctx.check(self._lib.sk_shard_counters(self._h, out))
        return int(out[0]), int(out[1])


class _CudaFull:
    """A full sk_tableau fed with shard blocks (sk_tableau_import_block / commit / export_block)."""

    def __init__(self, ctx, n):
        from . import Tableau, lib
        self._lib, self.ctx, self.t = lib(), ctx, Tableau(ctx, n)

    def import_block(self, lo, hi, buf):
        self.ctx.check(self._lib.sk_tableau_import_block(self.t._h, lo, hi, C.c_void_p(buf.data_ptr())))

    def commit(self):
        self.ctx.check(self._lib.sk_tableau_commit_blocks(self.t._h))

    def measure_batch(self, qubits, seed, ordinal0):
        return self.t.measure_batch(qubits, seed, ordinal0)

    def export_block(self, lo, hi, buf):
        self.ctx.check(self._lib.sk_tableau_export_block(self.t._h, lo, hi, C.c_void_p(buf.data_ptr())))

    def close(self):
        self.t.close()


class Exchange:
    """The three collectives of the protocol over (local shards) x (torch.distributed ranks).
    Global shard index = rank * local + l.  Works on CUDA tensors (nccl) and CPU tensors (gloo)."""

    def __init__(self, local: int):
        import torch
        import torch.distributed as td
        self.torch, self.td = torch, td
        self.on = td.is_available() and td.is_initialized()
        self.rank = td.get_rank() if self.on else 0
        self.world = td.get_world_size() if self.on else 1
        self.local = int(local)
        self.nshards = self.world * self.local
        self.calls = {"allreduce_min": 0, "allgather": 0, "broadcast": 0}
        self.bytes = 0
        # gloo has no CUDA all_gather: with that backend device buffers are staged through the host (used by the
        # 2-process test that shares one GPU, where NCCL refuses two ranks on a device)
        self.stage = self.on and td.get_backend() == "gloo"

    def _to_wire(self, t):
        return t.cpu() if (self.stage and t.is_cuda) else t

    def allreduce_min(self, tensors) -> np.ndarray:
        t = tensors[0] if len(tensors) == 1 else self.torch.stack(list(tensors)).amin(dim=0)
        if self.on and self.world > 1:
            t = self._to_wire(t.contiguous())
            self.td.all_reduce(t, op=self.td.ReduceOp.MIN)
            self.calls["allreduce_min"] += 1
            self.bytes += t.numel() * 4
        return t.cpu().numpy()

    def allgather(self, tensors):
        loc = self.torch.stack(list(tensors))                      # [local, m, PW]
        if not (self.on and self.world > 1):
            return loc.contiguous()
        wire = self._to_wire(loc.contiguous())
        outs = [self.torch.empty_like(wire) for _ in range(self.world)]
        self.td.all_gather(outs, wire)
        self.calls["allgather"] += 1
        self.bytes += loc.numel() * 8 * self.world
        return self.torch.cat(outs, dim=0).to(loc.device).contiguous()   # [world * local, m, PW], shard order

    def broadcast(self, row, owner_shard: int, empty):
        owner_rank = owner_shard // self.local
        buf = row if self.rank == owner_rank else empty()
        if self.on and self.world > 1:
            wire = self._to_wire(buf)
            self.td.broadcast(wire, src=owner_rank)
            if wire is not buf:
                buf.copy_(wire)
            self.calls["broadcast"] += 1
            self.bytes += buf.numel() * 8
        return buf


class ShardedTableau:
    """SPEC:104-224 tableau + SPEC:310-318 sim on row shards; same record as the unsharded engine."""

    def __init__(self, n: int, shards, exchange: Exchange, stream=None):
        self.n, self.shards, self.ex, self.stream = int(n), list(shards), exchange, stream
        assert len(self.shards) == exchange.local
        self.G = exchange.nshards
        self.first = exchange.rank * exchange.local              # global index of shards[0]
        self.ranges = [skdist.slot_range(self.n, g, self.G) for g in range(self.G)]
        for l, s in enumerate(self.shards):
            assert (s.lo, s.hi) == self.ranges[self.first + l], "shard does not hold the slots of its global index"
        self._win = 64
        self.stats = {"n_rand": 0, "n_det": 0, "searches": 0, "replicated_blocks": 0}
        # A measurement block is handled by the exchange-per-measurement protocol only up to its first random measurement; from
        # there every rank assembles the full tableau (ONE allgather of the shards' rows), runs the single-GPU measurement kernel on
        # it -- the same result everywhere -- and takes its rows back.  False: the per-measurement protocol throughout (the only
        # option when the full tableau does not fit one GPU).
        self.replicate_random_blocks = True
        self._full = None

    # -- construction on CUDA ------------------------------------------------------------------
    @classmethod
    def create_cuda(cls, n: int, local_shards: int = 1, device_index: int | None = None):
        import torch
        from . import Context
        rank, local_rank, world = skdist.env_world()
        dev_i = local_rank if device_index is None else device_index
        device = torch.device("cuda", dev_i)
        torch.cuda.set_device(device)
        stream = torch.cuda.Stream(device)
        ctx = Context(dev_i, stream.cuda_stream)                   # library work and torch collectives share one stream
        ex = Exchange(local_shards)
        with torch.cuda.stream(stream):
            shards = [CudaShard(ctx, n, *skdist.slot_range(n, ex.rank * local_shards + l, ex.nshards), device) for l in range(local_shards)]
        t = cls(n, shards, ex, stream)
        t.ctx = ctx
        return t

    def close(self):
        if self._full is not None:
            self._full.close(); self._full = None
        for s in self.shards:
            s.close()
        self.shards = []
        if getattr(self, "ctx", None) is not None:
            self.ctx.close()
            self.ctx = None

    def _on_stream(self):
        if self.stream is None:
            import contextlib
            return contextlib.nullcontext()
        import torch
        return torch.cuda.stream(self.stream)

    def owner_of(self, p: int) -> int:
        for g, (lo, hi) in enumerate(self.ranges):
            if lo <= p < hi:
                return g
        raise IndexError(p)

    # -- operations ----------------------------------------------------------------------------
    def apply_gates(self, gates: np.ndarray):
        for s in self.shards:
            s.apply_gates(gates)

    def measure_batch(self, qubits, seed: int, ordinal0: int):
        """m consecutive Z measurements; bit-identical to m sequential measure_z calls."""
        qubits = np.ascontiguousarray(qubits, np.uint32)
        m = len(qubits)
        out, det = np.zeros(m, np.uint8), np.zeros(m, np.uint8)
        pos = 0
        with self._on_stream():
            while pos < m:
                w = min(self._win, m - pos)
                qs = qubits[pos:pos + w]
                cand = self.ex.allreduce_min([s.pivot_search(qs) for s in self.shards])
                self.stats["searches"] += 1
                rnd = np.flatnonzero(cand != NONE)
                r0 = int(rnd[0]) if len(rnd) else w
                if r0 > 0:                                          # deterministic prefix, one allgather
                    parts = self.ex.allgather([s.det_partial(qs[:r0]) for s in self.shards])
                    out[pos:pos + r0] = self.shards[0].det_combine(parts)
                    det[pos:pos + r0] = 1
                    self.stats["n_det"] += r0
                if r0 < w and self.replicate_random_blocks:         # the rest of the block on the assembled tableau
                    o, d = self._replicated_block(qubits[pos + r0:], seed, ordinal0 + pos + r0)
                    out[pos + r0:] = o; det[pos + r0:] = d
                    self.stats["n_rand"] += int((d == 0).sum()); self.stats["n_det"] += int((d != 0).sum())
                    self._win = 64
                    return out, det
                if r0 < w:                                          # first random measurement of the window
                    p, q = int(cand[r0]), int(qs[r0])
                    owner = self.owner_of(p)
                    l = owner - self.first
                    mine = self.shards[l].pivot_row(p) if 0 <= l < len(self.shards) else None
                    row = self.ex.broadcast(mine, owner, self.shards[0].new_row_buffer)
                    bit = counter_bit(seed, ordinal0 + pos + r0)
                    for s in self.shards:
                        s.random_update(q, p, row, bit)
                    out[pos + r0] = bit
                    self.stats["n_rand"] += 1
                    pos += r0 + 1
                    self._win = max(8, min(self._win, 2 * (r0 + 1)))   # candidates after a random one are stale
                else:
                    pos += w
                    self._win = min(8192, self._win * 4)
        return out, det

    def _replicated_block(self, qubits, seed: int, ordinal0: int):
        """Measurements `qubits` (ordinals ordinal0..) on the full tableau assembled from all shards; rows back afterwards."""
        sh0 = self.shards[0]
        words = max(sh0.block_words(hi - lo) for lo, hi in self.ranges)
        loc = [s.new_block(words) for s in self.shards]
        for s, b in zip(self.shards, loc):
            s.export_rows(b)
        allb = self.ex.allgather([b.view(1, words) for b in loc])       # [G, 1, words], shard order
        if self._full is None:
            self._full = sh0.make_full()
        for g, (lo, hi) in enumerate(self.ranges):
            if hi > lo:
                self._full.import_block(lo, hi, allb[g, 0])
        self._full.commit()
        o, d = self._full.measure_batch(np.ascontiguousarray(qubits, np.uint32), seed, ordinal0)
        for s, b in zip(self.shards, loc):
            if s.hi > s.lo:
                self._full.export_block(s.lo, s.hi, b)
                s.import_rows(b)
        self.stats["replicated_blocks"] += 1
        return o, d

    def sim(self, circ, seed: int):
        """Clifford runs -> apply_gates, measurement runs -> measure_batch.  -> (outcomes, deterministic)"""
        from . import M as KIND_M
        gates = circ.gates
        is_m = gates["kind"] == KIND_M
        nm = int(is_m.sum())
        out, det = np.zeros(nm, np.uint8), np.zeros(nm, np.uint8)
        edges = np.flatnonzero(np.diff(is_m.astype(np.int8))) + 1
        bounds = [0, *edges.tolist(), len(gates)]
        ordinal = 0
        for a, b in zip(bounds[:-1], bounds[1:]):
            if a == b:
                continue
            if is_m[a]:
                o, d = self.measure_batch(gates["q0"][a:b], seed, ordinal)
                out[ordinal:ordinal + (b - a)] = o; det[ordinal:ordinal + (b - a)] = d
                ordinal += b - a
            else:
                self.apply_gates(np.ascontiguousarray(gates[a:b]))
        return out, det

    # -- read-back -----------------------------------------------------------------------------
    def download_local(self):
        with self._on_stream():
            return [(s.lo, s.hi, *s.download()) for s in self.shards]

    def gather_tableau(self):
        """Full tableau on every rank (SPEC:110 row order) -- for tests and small n."""
        W = (self.n + 63) // 64
        x = np.zeros((2 * self.n, W), np.uint64); z = np.zeros_like(x); r = np.zeros(2 * self.n, np.uint8)
        for lo, hi, sx, sz, sr in self.download_local():
            k = hi - lo
            x[lo:hi] = sx[:k]; x[self.n + lo:self.n + hi] = sx[k:]
            z[lo:hi] = sz[:k]; z[self.n + lo:self.n + hi] = sz[k:]
            r[lo:hi] = sr[:k]; r[self.n + lo:self.n + hi] = sr[k:]
        if self.ex.on and self.ex.world > 1:
            import torch
            pack = torch.from_numpy(np.concatenate([x.view(np.int64).ravel(), z.view(np.int64).ravel(), r.astype(np.int64)]))
            if self.ex.td.get_backend() == "nccl":
                pack = pack.cuda()
            self.ex.td.all_reduce(pack, op=self.ex.td.ReduceOp.SUM)     # slots are disjoint, everything else is zero: sum == or
            pack = pack.cpu().numpy()
            nw = 2 * self.n * W
            x = pack[:nw].view(np.uint64).reshape(2 * self.n, W); z = pack[nw:2 * nw].view(np.uint64).reshape(2 * self.n, W)
            r = pack[2 * nw:].astype(np.uint8)
        return x, z, r
