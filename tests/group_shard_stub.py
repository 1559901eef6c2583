"""CPU stand-in for paper_2507_03092_b200.group_sharded.CudaGroupShard (TEST INFRASTRUCTURE: lets the multi-process driver
run over gloo on a machine without a GPU).  Same protocol: conflicts() fills the bitmap words this shard owns, resolve()
runs first fit on the combined bitmap.  Predicates in numpy (proj/src/pauli.cpp:117-140)."""
import numpy as np
import torch

B = 1024


def _conflict(x, z, px, pz, mode):
    v = (x & pz) ^ (px & z)
    if mode == 1:
        return (v != 0).any(axis=-1)
    par = np.zeros(v.shape[:-1], np.uint64)
    for w in range(v.shape[-1]):
        u = v[..., w].copy()
        for sh in (32, 16, 8, 4, 2, 1):
            u ^= u >> np.uint64(sh)
        par ^= u & np.uint64(1)
    return par == 1


class StubGroupShard:
    def __init__(self, x, z, mode, shard, nshards):
        self.x, self.z, self.mode, self.shard, self.nshards = x, z, mode, shard, nshards
        self.count = len(x); self.Bk = min(self.count, B); self.GW32 = self.count // 32 + 2
        self.blocks = (self.count + self.Bk - 1) // self.Bk
        self.words = self.Bk * self.GW32
        self.group = np.zeros(self.count, np.uint32); self.ng = 0

    def new_bitmap(self):
        return torch.zeros(self.words, dtype=torch.int32)

    def conflicts(self, k, bitmap):
        bm = np.zeros((self.Bk, self.GW32), np.uint32)
        t0 = k * self.Bk; b = min(self.Bk, self.count - t0)
        if t0 > 0:
            owned = (self.group[:t0] >> 5) % self.nshards == self.shard          # placed terms whose group word this shard owns
            idx = np.flatnonzero(owned)
            for t in range(b):
                c = _conflict(self.x[idx], self.z[idx], self.x[t0 + t], self.z[t0 + t], self.mode)
                g = self.group[idx[c]]
                np.bitwise_or.at(bm[t], g >> 5, np.uint32(1) << (g & 31))
        bitmap.copy_(torch.from_numpy(bm.view(np.int32).reshape(-1)))

    def resolve(self, k, bitmap):
        bm = bitmap.numpy().view(np.uint32).reshape(self.Bk, self.GW32).copy()
        t0 = k * self.Bk; b = min(self.Bk, self.count - t0)
        for t in range(b):
            g = 0
            while (bm[t, g >> 5] >> (g & 31)) & 1:
                g += 1
            assert g <= self.ng
            self.group[t0 + t] = g; self.ng = max(self.ng, g + 1)
            if t + 1 < b:
                c = _conflict(self.x[t0 + t + 1:t0 + b], self.z[t0 + t + 1:t0 + b], self.x[t0 + t], self.z[t0 + t], self.mode)
                bm[t + 1:b, g >> 5][c] |= np.uint32(1) << np.uint32(g & 31)

    def result(self):
        return self.group.copy(), self.ng

    def close(self):
        pass
