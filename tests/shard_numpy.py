"""Test-only numpy shard engine with the CudaShard interface.

Drives paper_2311_04333_b200.sharded.sharded_coreness on CPU so the round /
level protocol and its collectives (gloo, world_size 2) are covered without a
GPU.  Sequential restatement of shard.cu: decrements skip vertices already at
or below the bound, the one that lands on the bound enrols the vertex.
"""
import numpy as np
import torch

UNSET = 0xFFFFFFFF


class NumpyShard:
    def __init__(self, offs, adj, bounds, rank):
        self.offs = np.asarray(offs, np.int64)
        self.adj = np.asarray(adj, np.int64)
        self.bounds = np.asarray(bounds, np.int64)
        self.P = len(bounds) - 1
        self.lo, self.hi = int(bounds[rank]), int(bounds[rank + 1])
        self.deg = (self.offs[self.lo + 1:self.hi + 1] - self.offs[self.lo:self.hi]).astype(np.int64)
        self.lab = np.full(self.hi - self.lo, UNSET, np.int64)
        self.front = np.zeros(0, np.int64)
        self.next = []

    @classmethod
    def from_rows(cls, n, bounds, rank, offs, adj):
        """The rank's own rows only (offs rebased to 0): nothing outside
        [lo, hi] of the global offsets is ever read."""
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        g = np.zeros(n + 1, np.int64)
        g[lo:hi + 1] = np.asarray(offs, np.int64)
        return cls(g, adj, bounds, rank)

    @property
    def n_local(self):
        return self.hi - self.lo

    def min_alive(self):
        alive = self.lab == UNSET
        return int(self.deg[alive].min()) if alive.any() else UNSET

    def collect(self, bound, label):
        sel = np.nonzero((self.lab == UNSET) & (self.deg <= bound))[0]
        self.lab[sel] = label
        self.front = sel
        return len(sel)

    def _arcs(self):
        if len(self.front) == 0:
            return np.zeros(0, np.int64)
        v = self.front + self.lo
        return np.concatenate([self.adj[self.offs[x]:self.offs[x + 1]] for x in v])

    def _owner(self, u):
        return np.searchsorted(self.bounds[1:], u, side="right")

    def count_remote(self):
        u = self._arcs()
        rem = u[(u < self.lo) | (u >= self.hi)]
        return np.bincount(self._owner(rem), minlength=self.P).astype(np.int64).tolist()

    def _dec(self, i, bound, label):
        if self.deg[i] <= bound:
            return
        self.deg[i] -= 1
        if self.deg[i] == bound:
            self.lab[i] = label
            self.next.append(i)

    def expand(self, bound, label, counts):
        u = self._arcs()
        self.next = []
        local = (u >= self.lo) & (u < self.hi)
        for x in u[local]:
            self._dec(int(x) - self.lo, bound, label)
        rem = u[~local]
        order = np.argsort(self._owner(rem), kind="stable")
        out = rem[order].astype(np.int32)
        assert len(out) == sum(counts)
        return torch.from_numpy(out)

    def apply(self, recv, bound, label):
        for x in recv.numpy().astype(np.int64):
            assert self.lo <= x < self.hi
            self._dec(int(x) - self.lo, bound, label)
        self.front = np.array(self.next, np.int64)
        return len(self.front)

    def labels(self):
        return self.lab.astype(np.uint32)
