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


def _block_views(buf, nl):
    """ctr u64[2] | deg | labels | q0 | q1 (u32[max(nl, 1)] each) -- the layout
    of the CUDA shard's peer block (shard.cu)."""
    w = max(nl, 1)
    ctr = np.frombuffer(buf, np.uint64, 2, 0)
    arr = np.frombuffer(buf, np.uint32, 4 * w, 16)
    return {"ctr": ctr, "deg": arr[:w], "lab": arr[w:2 * w], "q": [arr[2 * w:3 * w], arr[3 * w:]]}


class NumpyPeerShard:
    """Peer-mode restatement of dg_shard_expand_peer / dg_shard_finish_round:
    every decrement is applied AT THE OWNER's block (another shard object in
    this process, or a multiprocessing shared-memory block of another
    process -- the stand-in for CUDA IPC), crossings append to the owner's
    next queue.  Concurrent GPUs are modelled by any serial order: the set of
    crossings of a round does not depend on the order of its decrements."""

    def __init__(self, offs, adj, bounds, rank, shm=False):
        from multiprocessing import shared_memory
        self.offs = np.asarray(offs, np.int64)
        self.adj = np.asarray(adj, np.int64)
        self.bounds = np.asarray(bounds, np.int64)
        self.P = len(bounds) - 1
        self.rank = rank
        self.lo, self.hi = int(bounds[rank]), int(bounds[rank + 1])
        nl = self.hi - self.lo
        size = 16 + 16 * max(nl, 1)
        self._shm = shared_memory.SharedMemory(create=True, size=size) if shm else None
        self._buf = self._shm.buf if shm else bytearray(size)
        self.own = _block_views(self._buf, nl)
        self.own["ctr"][:] = 0
        self.own["deg"][:nl] = (self.offs[self.lo + 1:self.hi + 1] - self.offs[self.lo:self.hi])
        self.own["lab"][:nl] = UNSET
        self.peers = [None] * self.P
        self.peers[rank] = self.own
        self._opened = []
        self.cur = 0
        self.nfront = 0

    @classmethod
    def from_rows(cls, n, bounds, rank, offs, adj, shm=False):
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        g = np.zeros(n + 1, np.int64)
        g[lo:hi + 1] = np.asarray(offs, np.int64)
        return cls(g, adj, bounds, rank, shm)

    def close(self):
        import gc
        self.own = self.peers = None  # drop the numpy views before unmapping
        self._buf = None
        gc.collect()
        for s in self._opened:
            s.close()
        self._opened = []
        if self._shm is not None:
            self._shm.close()
            self._shm.unlink()
            self._shm = None

    @property
    def n_local(self):
        return self.hi - self.lo

    def ipc_handle(self):
        return self._shm.name.encode()

    def peer_open(self, r, handle):
        from multiprocessing import shared_memory
        s = shared_memory.SharedMemory(name=handle.decode())
        self._opened.append(s)
        self.peers[r] = _block_views(s.buf, int(self.bounds[r + 1] - self.bounds[r]))

    def peer_link(self, r, other):
        self.peers[r] = other.own

    def min_alive(self):
        nl = self.n_local
        alive = self.own["lab"][:nl] == UNSET
        return int(self.own["deg"][:nl][alive].min()) if alive.any() else UNSET

    def collect(self, bound, label):
        nl = self.n_local
        lab, deg = self.own["lab"][:nl], self.own["deg"][:nl]
        sel = np.nonzero((lab == UNSET) & (deg <= bound))[0]
        lab[sel] = label
        self.own["q"][self.cur][:len(sel)] = sel
        self.nfront = len(sel)
        return len(sel)

    def expand_peer(self, bound, label):
        self.own["ctr"][self.cur] = 0
        qn = self.cur ^ 1
        made = 0
        for x in self.own["q"][self.cur][:self.nfront].astype(np.int64):
            v = x + self.lo
            for u in self.adj[self.offs[v]:self.offs[v + 1]]:
                r = int(np.searchsorted(self.bounds[1:], u, side="right"))
                i = int(u - self.bounds[r])
                pv = self.peers[r]
                if pv["deg"][i] <= bound:
                    continue
                pv["deg"][i] -= 1
                if pv["deg"][i] == bound:
                    pv["lab"][i] = label
                    pv["q"][qn][int(pv["ctr"][qn])] = i
                    pv["ctr"][qn] += 1
                    made += 1
        return made

    def finish_round(self):
        self.nfront = int(self.own["ctr"][self.cur ^ 1])
        self.cur ^= 1
        return self.nfront

    def labels(self):
        return self.own["lab"][:self.n_local].astype(np.uint32)
