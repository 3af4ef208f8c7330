"""CPU stand-ins for the sharded-sortPR device primitives (test infrastructure):
exact numpy/torch versions of CudaShardOps, so the distributed protocol in
paper_2410_22764_b200/sharded.py runs under gloo on CPU.  `weak_first_seed`
makes the very first seed's hash tiny, forcing collisions -> exercises the
collision-void-and-retry path."""
import numpy as np
import torch

M64 = (1 << 64) - 1


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class CpuShardOps:
    device = torch.device("cpu")

    def __init__(self, weak_first_seed: bool = False):
        self.weak = weak_first_seed

    def signature(self, delta_local, block_full, lo, seed, ranks, pack_bits=0):
        d = delta_local.numpy().astype(np.int64)
        bf = block_full.numpy().astype(np.int64) & 0xFFFFFFFF  # int16 ids arrive signed
        if block_full.dtype == torch.int16:
            bf = bf & 0xFFFF
        n = d.shape[1]
        if pack_bits:  # exact packed key + 1, no rows
            key = bf[lo:lo + n].astype(np.uint64)
            for a in range(d.shape[0]):
                key = (key << np.uint64(pack_bits)) | bf[d[a]].astype(np.uint64)
            with np.errstate(over="ignore"):
                dest = (_mix(key ^ np.uint64(0xD1B54A32D192ED03)) % np.uint64(ranks)).astype(np.int32)
            return (torch.from_numpy((key + np.uint64(1)).view(np.int64).copy()), None,
                    torch.from_numpy(dest))
        rows = np.empty((n, d.shape[0] + 1), np.uint32)
        rows[:, 0] = bf[lo:lo + n]
        for a in range(d.shape[0]):
            rows[:, a + 1] = bf[d[a]]
        with np.errstate(over="ignore"):
            h = _mix(np.full(n, seed * 0x9E3779B97F4A7C15 & M64, np.uint64) + rows[:, 0].astype(np.uint64))
            for a in range(1, rows.shape[1]):
                h = _mix(h + np.uint64(0x9E3779B97F4A7C15) + rows[:, a].astype(np.uint64))
            if self.weak and seed == 0x5EED0001:
                h = h % np.uint64(3)  # deliberately colliding first attempt
            keys = h | np.uint64(1)
            dest = (_mix(keys ^ np.uint64(0xD1B54A32D192ED03)) % np.uint64(ranks)).astype(np.int32)
        return (torch.from_numpy(keys.view(np.int64).copy()), torch.from_numpy(rows.view(np.int32)),
                torch.from_numpy(dest))

    def route(self, dest, ranks):
        order = torch.argsort(dest, stable=True)
        counts = torch.bincount(dest.long(), minlength=ranks).tolist()
        return order, counts

    def group(self, keys, sig):
        if keys.numel() == 0:
            return torch.empty(0, dtype=torch.int32), 0, False
        k = keys.numpy()
        _, first, inv = np.unique(k, return_index=True, return_inverse=True)
        # collision: some key carries two different rows (exact packed keys: none)
        collision = False
        if sig is not None:
            rows = sig.numpy()
            collision = bool((rows != rows[first][inv]).any())
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(order.size)
        return torch.from_numpy(rank[inv].astype(np.int32)), int(first.size), collision

    def canonicalize(self, raw):
        r = raw.numpy()
        _, first, inv = np.unique(r, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty_like(order)
        rank[order] = np.arange(order.size)
        return torch.from_numpy(rank[inv].astype(np.int32)), int(first.size)
