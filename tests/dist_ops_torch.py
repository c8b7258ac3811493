"""Host (torch CPU) restatement of CudaDistOps -- TEST INFRASTRUCTURE.

The distributed build's collective protocol (sharded_build.build_shards /
shard_get_core) runs unchanged over gloo on CPU tensors with these per-rank
steps standing in for the library's kernels (csrc/dist_build.cu); the CUDA
tests run the same protocol with CudaDistOps and compare both with the
oracle's CSR."""
import numpy as np
import torch

NONE32 = -1


class TorchDistOps:
    def max_id(self, u, v):
        keep = u != v
        if not bool(keep.any()):
            return 0
        return int(torch.maximum(u, v)[keep].max())

    def hist(self, u, v, shift, nb):
        keep = u != v
        a, b = u[keep], v[keep]
        h = torch.bincount(torch.clamp(a >> shift, max=nb - 1), minlength=nb)[:nb]
        h += torch.bincount(torch.clamp(b >> shift, max=nb - 1), minlength=nb)[:nb]
        return h.numpy().astype(np.int64)

    def route(self, u, v, bounds_id):
        keep = u != v
        a, b = u[keep], v[keep]
        src, dst = torch.cat([a, b]), torch.cat([b, a])
        bnd = torch.as_tensor(bounds_id[1:-1].astype(np.int64))
        o = torch.bucketize(src, bnd, right=True)
        keys = (src << 32) | dst
        order = torch.argsort(o, stable=True)
        P = len(bounds_id) - 1
        return keys[order], torch.bincount(o, minlength=P).tolist()

    def rows(self, keys):
        # keys hold (src << 32 | dst) with src < 2^32: compare as unsigned via the
        # order-preserving shift into signed range
        k = torch.unique(keys - (1 << 63)) + (1 << 63) if keys.numel() else keys
        src = (k >> 32) & 0xFFFFFFFF
        dst = (k & 0xFFFFFFFF).to(torch.int64)
        verts, deg = torch.unique_consecutive(src, return_counts=True)
        offs = torch.zeros(verts.numel() + 1, dtype=torch.int64)
        offs[1:] = torch.cumsum(deg, 0)
        return offs, verts, dst

    def unique(self, vals):
        u, inv = torch.unique(vals.to(torch.int64) & 0xFFFFFFFF, return_inverse=True)
        return u, inv

    def bucket_counts(self, vals, bounds_id):
        P = len(bounds_id) - 1
        bnd = torch.as_tensor(bounds_id[1:-1].astype(np.int64))
        o = torch.bucketize(vals.to(torch.int64), bnd, right=True)
        return torch.bincount(o, minlength=P).tolist()

    def lookup(self, verts, asked, base):
        return torch.searchsorted(verts, asked.to(torch.int64)) + int(base)

    def relabel(self, back, inv):
        return back[inv]

    def keep_map(self, labels, k, base):
        keep = labels.to(torch.int64) >= k
        new = torch.cumsum(keep.to(torch.int64), 0) - 1 + int(base)
        return torch.where(keep, new, torch.full_like(new, NONE32)), int(keep.sum())

    def core_rows(self, offs, adj, local_map, full_map):
        nl = offs.numel() - 1
        adj = adj.to(torch.int64) & 0xFFFFFFFF
        row = torch.repeat_interleave(torch.arange(nl), offs[1:] - offs[:-1],
                                      output_size=adj.numel())
        keep = local_map >= 0
        nadj = full_map.to(torch.int64)[adj]
        ka = keep[row] & (nadj >= 0)
        deg = torch.bincount(row[ka], minlength=nl)[keep]
        noffs = torch.zeros(deg.numel() + 1, dtype=torch.int64)
        noffs[1:] = torch.cumsum(deg, 0)
        return noffs, nadj[ka]

    def take(self, x, local_map, base, kept):
        return x[local_map >= 0]
