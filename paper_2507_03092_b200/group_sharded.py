"""First-fit commutation grouping with the pair matrix sharded by row blocks (north_star
"Commutation grouping shards the pair matrix by row blocks").

One process per GPU (torch.distributed, NCCL).  Every shard holds the replicated term list and the replicated group
assignment; the expensive part -- the conflict bitmap of each block of 1024 terms against the groups placed so far
(proj/src/pauli.cpp:117-140 predicates, `k_conflict_groups`) -- is split: global shard s of S evaluates the groups of the
bitmap words w with w % S == s.  Per block:

    conflicts   every shard fills its own words of the block's bitmap            (no communication)
    combine     OR of the shards' bitmaps = allreduce-SUM, the words are disjoint (one collective per block)
    resolve     every shard runs the sequential first-fit resolver on the combined bitmap: identical groups everywhere

`local_shards > 1` keeps several shards in one process (the combine is then an in-process OR), which is how the protocol
is verified on a single B200.  Groups are bit-identical to `sk_group_first_fit` and to the CPU oracle.
The resolver is sequential in the term index and replicated, so only the predicate evaluations scale with the shards.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import dist as skdist


class CudaGroupShard:
    """One sk_group_shard over a (replicated) sk_rows block."""

    def __init__(self, rows, mode: int, shard: int, nshards: int, device):
        import torch
        from . import lib
        self._torch, self._lib, self.rows, self.ctx, self.device = torch, lib(), rows, rows.ctx, device
        self._h = C.c_void_p()
        self.ctx.check(self._lib.sk_group_shard_create(rows._h, mode, shard, nshards, C.byref(self._h)))
        self.blocks = int(self._lib.sk_group_shard_blocks(self._h))
        self.words = int(self._lib.sk_group_shard_bitmap_words(self._h))
        self.count = rows.count

    def close(self):
        if self._h and self.ctx._h:
            self._lib.sk_group_shard_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def new_bitmap(self):
        return self._torch.zeros(self.words, dtype=self._torch.int32, device=self.device)

    def conflicts(self, block: int, bitmap):
        self.ctx.check(self._lib.sk_group_shard_conflicts(self._h, block, C.c_void_p(bitmap.data_ptr())))

    def resolve(self, block: int, bitmap):
        self.ctx.check(self._lib.sk_group_shard_resolve(self._h, block, C.c_void_p(bitmap.data_ptr())))

    def result(self):
        g = np.zeros(self.count, np.uint32); ng = C.c_uint64(0)
        self.ctx.check(self._lib.sk_group_shard_result(self._h, g.ctypes.data_as(C.c_void_p), C.byref(ng)))
        return g, int(ng.value)


class GroupExchange:
    """OR of the shards' block bitmaps over (local shards) x (torch.distributed ranks); global shard = rank * local + l."""

    def __init__(self, local: int):
        import torch
        import torch.distributed as td
        self.torch, self.td = torch, td
        self.on = td.is_available() and td.is_initialized()
        self.rank = td.get_rank() if self.on else 0
        self.world = td.get_world_size() if self.on else 1
        self.local = int(local)
        self.nshards = self.world * self.local
        self.calls, self.bytes = 0, 0
        self.stage = self.on and td.get_backend() == "gloo"          # gloo: device buffers travel through the host

    def allreduce_or(self, bitmaps):
        """-> one tensor holding the OR of all shards' bitmaps (bitmaps[0] is reused)."""
        t = bitmaps[0]
        for b in bitmaps[1:]:
            t.bitwise_or_(b)
        if self.on and self.world > 1:
            wire = t.cpu() if (self.stage and t.is_cuda) else t
            self.td.all_reduce(wire, op=self.td.ReduceOp.SUM)        # disjoint words: SUM == OR
            if wire is not t:
                t.copy_(wire)
            self.calls += 1
            self.bytes += t.numel() * 4
        return t


def group_first_fit_sharded(shards, exchange: GroupExchange):
    """shards: this process's shards (global shard index = exchange.rank * local + l).  -> (group ids u32[N], groups)."""
    assert len(shards) == exchange.local
    bms = [s.new_bitmap() for s in shards]
    for k in range(shards[0].blocks):
        for s, b in zip(shards, bms):
            s.conflicts(k, b)
        comb = exchange.allreduce_or(bms)
        for s, b in zip(shards[1:], bms[1:]):                        # every shard resolves on its own copy (the resolver adds the block-mates' bits)
            b.copy_(comb)
        for s, b in zip(shards, bms):
            s.resolve(k, b)
    return shards[0].result()


def group_first_fit_cuda(rows, mode: int, local_shards: int = 1, device_index: int | None = None):
    """Convenience: sharded first fit of an sk.Rows block on this process's GPU (x local shards), over the initialised
    process group if there is one.  Every rank passes the same rows."""
    import torch
    rank, local_rank, world = skdist.env_world()
    device = torch.device("cuda", local_rank if device_index is None else device_index)
    ex = GroupExchange(local_shards)
    stream = torch.cuda.ExternalStream(rows.ctx.stream)
    with torch.cuda.stream(stream):
        shards = [CudaGroupShard(rows, mode, ex.rank * local_shards + l, ex.nshards, device) for l in range(local_shards)]
        try:
            return group_first_fit_sharded(shards, ex), ex
        finally:
            for s in shards:
                s.close()
