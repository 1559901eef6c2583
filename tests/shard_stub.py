"""TEST INFRASTRUCTURE: a tiny CPU stand-in for `sharded.CudaShard` (Python big-int rows) so that the host
driver of the row-sharded tableau -- window logic, ownership, and the three exchanges over torch.distributed --
can be exercised with world_size 2 on the gloo backend, where no GPU exists.  Never imported by the product."""
import numpy as np
import torch

NONE = 0x7F7F7F7F
H, S, SDG, X, Y, Z, CX, CZ, SWAP, M = range(10)


def g_sum(ax, az, bx, bz):
    """i-exponent of a*b (a left), ref: proj/src/pauli.cpp:189-205"""
    anti = (ax & bz) ^ (bx & az)
    plus = anti & ((ax & ~az & bx) | (ax & az & ~bx) | (~ax & az & ~bz))
    return plus.bit_count() - (anti & ~plus).bit_count()


class StubShard:
    def __init__(self, n, lo, hi):
        self.n, self.lo, self.hi = n, lo, hi
        self.W = (n + 63) // 64
        self.Wp = (self.W + 1) & ~1
        self.PW = 2 * self.Wp + 2
        k = hi - lo
        # rows: [x, z, sign]; stabilizers then destabilizers of the slots
        self.stab = [[0, 1 << (lo + i), 0] for i in range(k)]
        self.destab = [[1 << (lo + i), 0, 0] for i in range(k)]

    def close(self):
        pass

    # -- gates ------------------------------------------------------------
    @staticmethod
    def _h(r, q):
        x, z = (r[0] >> q) & 1, (r[1] >> q) & 1
        r[2] ^= x & z
        if x != z:
            r[0] ^= 1 << q; r[1] ^= 1 << q

    @staticmethod
    def _s(r, q):
        x, z = (r[0] >> q) & 1, (r[1] >> q) & 1
        r[2] ^= x & z
        r[1] ^= x << q

    @staticmethod
    def _cx(r, c, t):
        xc, zc, xt, zt = (r[0] >> c) & 1, (r[1] >> c) & 1, (r[0] >> t) & 1, (r[1] >> t) & 1
        r[2] ^= xc & zt & (xt ^ zc ^ 1)
        r[0] ^= xc << t; r[1] ^= zt << c

    def apply_gates(self, gates):
        for g in gates:
            k, a, b = int(g["kind"]), int(g["q0"]), int(g["q1"])
            for r in self.stab + self.destab:
                if k == H: self._h(r, a)
                elif k == S: self._s(r, a)
                elif k == SDG: self._s(r, a); self._s(r, a); self._s(r, a)
                elif k == Z: self._s(r, a); self._s(r, a)
                elif k == X: self._h(r, a); self._s(r, a); self._s(r, a); self._h(r, a)
                elif k == Y: self._s(r, a); self._s(r, a); self._h(r, a); self._s(r, a); self._s(r, a); self._h(r, a)
                elif k == CX: self._cx(r, a, b)
                elif k == CZ: self._h(r, b); self._cx(r, a, b); self._h(r, b)
                elif k == SWAP: self._cx(r, a, b); self._cx(r, b, a); self._cx(r, a, b)
                else: raise ValueError(k)

    # -- measurement pieces -----------------------------------------------------------------------
    def pivot_search(self, qubits):
        out = np.full(len(qubits), NONE, np.int32)
        for j, q in enumerate(qubits):
            for i, r in enumerate(self.stab):
                if (r[0] >> int(q)) & 1:
                    out[j] = self.lo + i; break
        return torch.from_numpy(out)

    def _pack(self, x, z, phase):
        w = np.zeros(self.PW, np.uint64)
        w[:self.W] = np.frombuffer(x.to_bytes(8 * self.W, "little"), np.uint64)
        w[self.Wp:self.Wp + self.W] = np.frombuffer(z.to_bytes(8 * self.W, "little"), np.uint64)
        w[2 * self.Wp] = phase
        return w.view(np.int64)

    def _unpack(self, w):
        w = np.ascontiguousarray(w.numpy()).view(np.uint64)
        return (int.from_bytes(w[:self.W].tobytes(), "little"), int.from_bytes(w[self.Wp:self.Wp + self.W].tobytes(), "little"), int(w[2 * self.Wp]))

    def det_partial(self, qubits):
        out = np.zeros((len(qubits), self.PW), np.int64)
        for j, q in enumerate(qubits):
            ax = az = e = 0
            for i, d in enumerate(self.destab):
                if (d[0] >> int(q)) & 1:
                    sx, sz, sr = self.stab[i]
                    e += g_sum(sx, sz, ax, az) + 2 * sr
                    ax ^= sx; az ^= sz
            out[j] = self._pack(ax, az, e & 3)
        return torch.from_numpy(out)

    def det_combine(self, gathered):
        G, m, _ = gathered.shape
        out = np.zeros(m, np.uint8)
        for j in range(m):
            ax = az = e = 0
            for g in range(G):
                sx, sz, ph = self._unpack(gathered[g, j])
                e += g_sum(sx, sz, ax, az) + ph
                ax ^= sx; az ^= sz
            assert e % 2 == 0
            out[j] = (e & 3) >> 1
        return out

    def pivot_row(self, p):
        x, z, r = self.stab[p - self.lo]
        return torch.from_numpy(self._pack(x, z, r))

    def new_row_buffer(self):
        return torch.zeros(self.PW, dtype=torch.int64)

    def random_update(self, q, p, row, outcome):
        px, pz, pr = self._unpack(row)
        pl = p - self.lo if self.lo <= p < self.hi else -1
        for half, rows in enumerate((self.stab, self.destab)):
            for i, r in enumerate(rows):
                if i == pl or not (r[0] >> q) & 1:
                    continue
                s = (2 * r[2] + 2 * pr + g_sum(px, pz, r[0], r[1])) & 3
                assert s % 2 == 0
                r[0] ^= px; r[1] ^= pz; r[2] = s >> 1
        if pl >= 0:
            self.destab[pl] = [px, pz, pr]
            self.stab[pl] = [0, 1 << q, outcome]

    # -- replicated elimination of a random block (same block layout as sk_shard_export_rows) ---------------
    def block_words(self, nloc=None):
        nloc = (self.hi - self.lo) if nloc is None else nloc
        return 4 * nloc * self.Wp + 2 * ((nloc + 63) // 64)

    def new_block(self, words):
        return torch.zeros(max(words, 1), dtype=torch.int64)

    def export_rows(self, buf):
        k = self.hi - self.lo
        w = np.zeros(buf.numel(), np.uint64)
        sw = (k + 63) // 64
        for half, rows in enumerate((self.stab, self.destab)):
            for i, r in enumerate(rows):
                base = (half * k + i) * 2 * self.Wp
                w[base:base + self.W] = np.frombuffer(r[0].to_bytes(8 * self.W, "little"), np.uint64)
                w[base + self.Wp:base + self.Wp + self.W] = np.frombuffer(r[1].to_bytes(8 * self.W, "little"), np.uint64)
                if r[2]: w[4 * k * self.Wp + half * sw + (i >> 6)] |= np.uint64(1) << np.uint64(i & 63)
        buf.copy_(torch.from_numpy(w.view(np.int64)))

    def import_rows(self, buf):
        k = self.hi - self.lo
        w = np.ascontiguousarray(buf.numpy()).view(np.uint64)
        sw = (k + 63) // 64
        for half, rows in enumerate((self.stab, self.destab)):
            for i in range(k):
                base = (half * k + i) * 2 * self.Wp
                x = int.from_bytes(w[base:base + self.W].tobytes(), "little"); z = int.from_bytes(w[base + self.Wp:base + self.Wp + self.W].tobytes(), "little")
                sg = int((int(w[4 * k * self.Wp + half * sw + (i >> 6)]) >> (i & 63)) & 1)
                rows[i] = [x, z, sg]

    def make_full(self):
        return StubFull(self.n)

    def download(self):
        k = self.hi - self.lo
        x = np.zeros((2 * k, self.W), np.uint64); z = np.zeros_like(x); r = np.zeros(2 * k, np.uint8)
        for i, row in enumerate(self.stab + self.destab):
            x[i] = np.frombuffer(row[0].to_bytes(8 * self.W, "little"), np.uint64)
            z[i] = np.frombuffer(row[1].to_bytes(8 * self.W, "little"), np.uint64)
            r[i] = row[2]
        return x, z, r


class StubFull:
    """Full tableau for the replicated block on CPU: the oracle's tableau (test infrastructure) fed with shard blocks."""

    def __init__(self, n):
        from oracle import oracle_py as orc
        self.orc, self.n, self.W = orc, n, (n + 63) // 64
        self.Wp = (self.W + 1) & ~1
        self.x = np.zeros((2 * n, self.W), np.uint64); self.z = np.zeros_like(self.x); self.r = np.zeros(2 * n, np.uint8)
        self.t = orc.Tableau(n)

    def import_block(self, lo, hi, buf):
        k = hi - lo
        w = np.ascontiguousarray(buf.numpy()).view(np.uint64)
        sw = (k + 63) // 64
        for half in range(2):
            for i in range(k):
                base = (half * k + i) * 2 * self.Wp
                row = half * self.n + lo + i
                self.x[row] = w[base:base + self.W]; self.z[row] = w[base + self.Wp:base + self.Wp + self.W]
                self.r[row] = (int(w[4 * k * self.Wp + half * sw + (i >> 6)]) >> (i & 63)) & 1

    def commit(self):
        self.t.set(self.x, self.z, self.r)

    def measure_batch(self, qubits, seed, ordinal0):
        gates = [(M, int(q), 0) for q in qubits]
        o, d, rc = self.t.sim(gates, seed, 1, ordinal0)
        assert rc == 0
        self.x, self.z, self.r = self.t.get()
        return o, d

    def export_block(self, lo, hi, buf):
        k = hi - lo
        w = np.zeros(buf.numel(), np.uint64)
        sw = (k + 63) // 64
        for half in range(2):
            for i in range(k):
                base = (half * k + i) * 2 * self.Wp
                row = half * self.n + lo + i
                w[base:base + self.W] = self.x[row]; w[base + self.Wp:base + self.Wp + self.W] = self.z[row]
                if self.r[row]: w[4 * k * self.Wp + half * sw + (i >> 6)] |= np.uint64(1) << np.uint64(i & 63)
        buf.copy_(torch.from_numpy(w.view(np.int64)))

    def close(self):
        pass
