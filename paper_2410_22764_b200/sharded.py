"""State-sharded sortPR over several GPUs.

The product path is the C++ driver in libdfm (csrc/shard_driver.cu, C-ABI
``dfm_sort_pr_sharded[_dev]``), reached here through :class:`ShardedEngine`: its
context owns an NCCL communicator (bootstrapped over torch.distributed: rank 0's
ncclUniqueId is broadcast) or, in the single-GPU tests, the in-process "local"
transport (ranks as threads sharing one device).

``sharded_sort_pr`` below is the same protocol written over torch.distributed
collectives and pluggable device ops: the CPU-testable specification of the
driver (tests/test_sharded_gloo.py runs it at world 2 and 3 over gloo).

One process per GPU.  Rank g owns the contiguous state range [lo_g, hi_g) and
its δ rows (global target ids).  Each refinement pass (min_sort.hpp:93-118):

  1. all-gather the owned block-id slices   -> full block vector on every rank
  2. signature rows + 64-bit keys of owned states (libdfm ``dfm_shard_signature``)
  3. route every (key, row) to the rank ``dest(key)`` that groups it:
     radix sort by destination (``dfm_sort_pairs``) + one all-to-all
  4. exact local grouping at the destination (``dfm_shard_group``); a hash
     collision anywhere voids the pass for all ranks (max all-reduce) and it is
     redone under a new seed — the partition stays exact
  5. all-gather of per-rank group counts -> dense global ids (rank offsets)
  6. reverse all-to-all of the new ids to the owners
  7. fixpoint when the global block count did not grow (the reference's
     ``fresh == num_blocks``), so pass counts equal the reference's.

Grouping is by exact key equality, independent of the number of ranks and of
the hashing, so the partition sequence is the reference's for any world size.

``Comm`` wraps torch.distributed (NCCL on GPU; gloo with host staging for the
CPU tests); ``ops`` supplies the device primitives (``CudaShardOps`` here, a CPU
stand-in in tests/) so the protocol itself is testable with gloo on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch
import torch.distributed as dist


class Comm:
    """torch.distributed collectives on 1-D tensors of the ops' device."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.stage = dist.is_initialized() and dist.get_backend(group) == "gloo"

    def _to(self, t):
        return t.cpu() if self.stage else t

    def all_gather(self, t: torch.Tensor, counts) -> torch.Tensor:
        """Concatenate every rank's `t` (rank r contributes counts[r] elements).  Narrow
        id vectors (uint8 / int16) travel as they are over NCCL (int16 as byte pairs);
        gloo (the CPU tests) lacks those types and gets int32."""
        if self.world == 1:
            return t
        if t.dtype in (torch.uint8, torch.int16) and self.stage:
            return self.all_gather(t.to(torch.int32), counts).to(t.dtype)
        if t.dtype == torch.int16:
            b = self.all_gather(t.contiguous().view(torch.uint8), [2 * int(c) for c in counts])
            return b.view(torch.int16)
        width = int(max(counts))  # collectives need equal sizes: pad, gather, trim
        src = self._to(t)
        if src.numel() < width:
            src = torch.cat([src, src.new_zeros(width - src.numel())])
        out = torch.empty(width * self.world, dtype=t.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        parts = [out[r * width:r * width + int(c)] for r, c in enumerate(counts)]
        return torch.cat(parts).to(t.device)

    def all_to_all(self, t: torch.Tensor, send_counts, recv_counts) -> torch.Tensor:
        if self.world == 1:
            return t.clone()
        src = self._to(t).contiguous()
        out = torch.empty(int(sum(recv_counts)), *t.shape[1:], dtype=t.dtype, device=src.device)
        dist.all_to_all_single(out, src, [int(x) for x in recv_counts],
                               [int(x) for x in send_counts], group=self.group)
        return out.to(t.device)

    def all_gather_ints(self, values) -> list:
        """Gather a short list of python ints from every rank -> list per rank."""
        v = torch.tensor(list(values), dtype=torch.int64)
        if self.world == 1:
            return [v.tolist()]
        dev = "cpu" if self.stage or not torch.cuda.is_available() else torch.device(
            "cuda", torch.cuda.current_device())
        v = v.to(dev)
        outs = [torch.empty_like(v) for _ in range(self.world)]
        dist.all_gather(outs, v, group=self.group)
        return [o.cpu().tolist() for o in outs]


class CudaShardOps:
    """libdfm device primitives on torch CUDA tensors (the product path)."""

    def __init__(self, engine):
        self.eng = engine
        self.lib = engine.lib
        # kernels must be ordered with the torch ops and NCCL collectives around them
        engine.set_stream(torch.cuda.current_stream(torch.device("cuda", engine.device)).cuda_stream)
        lib = self.lib
        vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
        lib.dfm_shard_signature.argtypes = [vp, vp, u64, u32, vp, u64, u64, u32, vp, vp, vp]
        lib.dfm_shard_signature_ex.argtypes = [vp, vp, u64, u32, vp, u32, u64, u64, u32, u32, vp,
                                                vp, vp]
        lib.dfm_shard_group.argtypes = [vp, vp, vp, u32, u64, vp, C.POINTER(u64),
                                        C.POINTER(C.c_int)]
        lib.dfm_sort_pairs.argtypes = [vp, vp, vp, u64, u32]
        lib.dfm_canonicalize_dev.argtypes = [vp, vp, u64, vp, C.POINTER(u32)]
        lib.dfm_random_dfa_slice_dev.argtypes = [vp, u64, u32, u64, C.c_double, u64, u64, vp, vp]
        for f in ("dfm_shard_signature", "dfm_shard_signature_ex", "dfm_shard_group",
                  "dfm_sort_pairs",
                  "dfm_canonicalize_dev", "dfm_random_dfa_slice_dev"):
            getattr(lib, f).restype = C.c_int

    @property
    def device(self):
        return torch.device("cuda", self.eng.device)

    def signature(self, delta_local, block_full, lo: int, seed: int, ranks: int,
                  pack_bits: int = 0):
        """Keys of the owned states; pack_bits > 0: exact packed keys, no rows (sig None).
        block_full may be uint8 / int16 / int32 (the narrowest width holding the ids)."""
        k, n_local = delta_local.shape
        keys = torch.empty(n_local, dtype=torch.int64, device=self.device)
        sig = None if pack_bits else torch.empty((n_local, k + 1), dtype=torch.int32,
                                                 device=self.device)
        dest = torch.empty(n_local, dtype=torch.int32, device=self.device)
        self.eng._check(self.lib.dfm_shard_signature_ex(
            self.eng.handle, delta_local.data_ptr(), n_local, k, block_full.data_ptr(),
            block_full.element_size(), lo, seed & (2 ** 64 - 1), ranks, pack_bits,
            keys.data_ptr(), sig.data_ptr() if sig is not None else None, dest.data_ptr()))
        return keys, sig, dest

    def route(self, dest, ranks: int):
        """Stable order of items by destination rank + per-rank counts (None = identity
        order at one rank).  Counts come from one reduction per rank: a bincount over a
        handful of bins serialises its atomics on a few addresses."""
        n = dest.numel()
        if ranks == 1 or n == 0:
            return None, [n] + [0] * (ranks - 1)
        counts = torch.stack([(dest == r).sum() for r in range(ranks)]).cpu().tolist()
        keys = dest.to(torch.int64).contiguous()
        order = torch.arange(n, dtype=torch.int32, device=self.device)
        bits = max(1, (ranks - 1).bit_length())
        self.eng._check(self.lib.dfm_sort_pairs(self.eng.handle, keys.data_ptr(),
                                                order.data_ptr(), n, bits))
        return order.long(), counts

    def group(self, keys, sig):
        n = keys.numel()
        words = sig.shape[1] if sig is not None else 0
        label = torch.empty(n, dtype=torch.int32, device=self.device)
        groups = C.c_uint64(0)
        coll = C.c_int(0)
        self.eng._check(self.lib.dfm_shard_group(self.eng.handle, keys.data_ptr(),
                                                 sig.data_ptr() if sig is not None else None,
                                                 words, n, label.data_ptr(), C.byref(groups),
                                                 C.byref(coll)))
        return label, int(groups.value), bool(coll.value)

    def canonicalize(self, raw):
        out = torch.empty_like(raw)
        nb = C.c_uint32(0)
        self.eng._check(self.lib.dfm_canonicalize_dev(self.eng.handle, raw.data_ptr(), raw.numel(),
                                                      out.data_ptr(), C.byref(nb)))
        return out, int(nb.value)

    def random_slice(self, n_total: int, k: int, seed: int, p: float, lo: int, count: int):
        delta = torch.empty((k, count), dtype=torch.int32, device=self.device)
        acc = torch.empty(count, dtype=torch.uint8, device=self.device)
        self.eng._check(self.lib.dfm_random_dfa_slice_dev(
            self.eng.handle, n_total, k, seed & (2 ** 64 - 1), p, lo, count, delta.data_ptr(),
            acc.data_ptr()))
        return delta, acc


@dataclass
class ShardedResult:
    block_local: torch.Tensor  # canonical labels of the owned states
    num_blocks: int
    iterations: int
    retries: int
    converged: bool = True  # False: stopped at max_passes before the fixpoint


def shard_bounds(n_total: int, world: int, rank: int):
    """Rank r owns [r*S, min(n, (r+1)*S)), S = ceil(n/world) rounded up to a multiple of
    32 (dfm_shard_bounds: a rank's slice of a bit-packed id vector is whole words)."""
    S = -(-(-(-n_total // world)) // 32) * 32
    lo = min(n_total, rank * S)
    return lo, min(n_total, lo + S)


def sharded_sort_pr(delta_local: torch.Tensor, acc_local: torch.Tensor, n_total: int, lo: int,
                    comm: Comm, ops, max_passes: int | None = None,
                    allow_packed: bool = True) -> ShardedResult:
    """sortPR over state shards.  delta_local: (k, n_local) int32 global targets;
    acc_local: (n_local,) uint8.  Returns this rank's canonical labels.
    allow_packed=False keeps hashed keys + verification in every pass (tests)."""
    world, rank = comm.world, comm.rank
    k, n_local = delta_local.shape
    sizes = [hi - lo_ for lo_, hi in (shard_bounds(n_total, world, r) for r in range(world))]
    # init, min_sort.hpp:80-88: two blocks iff both acceptance classes are non-empty
    n_acc = sum(v[0] for v in comm.all_gather_ints([int(acc_local.sum().item())]))
    split = 0 < n_acc < n_total
    block = ((acc_local == 0).to(torch.int32) if split
             else torch.zeros(n_local, dtype=torch.int32, device=acc_local.device))
    B = 2 if split else 1
    seed = 0x5EED0001
    iterations = retries = 0
    converged = False
    while True:
        if max_passes is not None and iterations >= max_passes:
            break
        # ids travel at the narrowest width holding B values; while the whole key
        # (block, k successor ids) fits 63 bits it is packed exactly (no rows)
        w = max(1, (B - 1).bit_length())
        pack = w if allow_packed and (k + 1) * w <= 63 else 0
        narrow = torch.uint8 if B <= 256 else torch.int16 if B <= 65536 else torch.int32
        block_full = comm.all_gather(block.to(narrow), sizes)
        keys, sig, dest = ops.signature(delta_local, block_full, lo, seed, world, pack)
        order, send_counts = ops.route(dest, world)
        if order is None:  # one rank: every key is grouped here, in place
            recv_counts = send_counts
            rkeys, rsig = keys, sig
        else:
            recv_counts = [c[rank] for c in comm.all_gather_ints(send_counts)]
            rkeys = comm.all_to_all(keys[order], send_counts, recv_counts)
            rsig = (comm.all_to_all(sig[order], send_counts, recv_counts)
                    if sig is not None else None)
        label, groups, collision = ops.group(rkeys, rsig)
        stats = comm.all_gather_ints([groups, int(collision)])
        if any(s[1] for s in stats):  # a collision on any rank voids the pass everywhere
            retries += 1
            seed = (seed * 0x9E3779B97F4A7C15 + 0x632BE59BD9B4E019) & (2 ** 64 - 1)
            continue
        offset = sum(s[0] for s in stats[:rank])
        B_new = sum(s[0] for s in stats)
        if order is None:
            new_block = (label + offset).to(block.dtype)
        else:
            back = comm.all_to_all(label + offset, recv_counts, send_counts)
            new_block = torch.empty_like(block)
            new_block[order] = back.to(new_block.dtype)
        iterations += 1
        block = new_block
        if B_new == B:  # fixpoint, min_sort.hpp:111-117
            converged = True
            break
        B = B_new
        if B == n_total:
            # every block is a singleton: the next pass sees n distinct keys (each holds
            # its own block id), grows nothing and ends the loop — count it, skip it
            iterations += 1
            converged = True
            break
    block_full = comm.all_gather(block, sizes)
    canon, nb = ops.canonicalize(block_full)
    return ShardedResult(canon[lo:lo + n_local].clone(), nb, iterations, retries, converged)


class ShardedEngine:
    """A libdfm context owning one rank of a communicator; runs the C++ sharded
    sortPR driver (dfm_sort_pr_sharded[_dev]).

    transport="nccl": one process per GPU; the NCCL id is created by rank 0 and
    broadcast over torch.distributed (any backend).  transport="local": ranks are
    threads of this process on one device meeting in `group` (tests)."""

    def __init__(self, device: int, rank: int, world: int, transport: str = "nccl",
                 group: str = "dfm", pg=None):
        import paper_2410_22764_b200 as dfm
        self.dfm = dfm
        lib = dfm._load()
        self.lib = lib
        h = C.c_void_p()
        if transport == "nccl":
            uid = (C.c_uint8 * 128)()
            if rank == 0:
                rc = lib.dfm_nccl_get_unique_id(uid)
                if rc != 0:
                    raise dfm.EngineError(rc, "ncclGetUniqueId failed")
            obj = [bytes(uid)]
            if world > 1:
                dist.broadcast_object_list(obj, src=0, group=pg)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
            rc = lib.dfm_ctx_create_sharded(device, rank, world, uid, C.byref(h))
        elif transport == "local":
            rc = lib.dfm_ctx_create_sharded_local(device, rank, world, group.encode(), C.byref(h))
        else:
            raise ValueError(transport)
        if rc != 0:
            raise dfm.EngineUnavailable(rc, (lib.dfm_last_error(None) or b"").decode())
        self.engine = dfm.Engine.__new__(dfm.Engine)  # profiling / stream plumbing
        self.engine.lib, self.engine.handle, self.engine.device = lib, h, device
        self.handle, self.device, self.rank, self.world = h, device, rank, world

    def bounds(self, n_total: int):
        lo, hi = C.c_uint64(0), C.c_uint64(0)
        self.lib.dfm_shard_bounds(n_total, self.world, self.rank, C.byref(lo), C.byref(hi))
        return int(lo.value), int(hi.value)

    def info(self):
        r, w, t = C.c_int(0), C.c_int(0), C.c_char_p()
        self.engine._check(self.lib.dfm_ctx_shard_info(self.handle, C.byref(r), C.byref(w),
                                                       C.byref(t)))
        return int(r.value), int(w.value), t.value.decode()

    def sort_pr(self, local, n_total: int, gather_all: bool = False, timeout_ms: int = 300_000):
        """local: dfm.Dfa of the owned states (GLOBAL targets).  Returns
        (labels, num_blocks, RunStats): this rank's canonical labels, or the whole
        partition with gather_all."""
        import numpy as np
        dfm = self.dfm
        cd, keep = dfm.Engine._cdfa(local)
        out = np.empty(n_total if gather_all else local.num_states, np.uint32)
        nb = C.c_uint32(0)
        st = dfm._CStats()
        self.engine._check(self.lib.dfm_sort_pr_sharded(
            self.handle, n_total, C.byref(cd), int(gather_all), out.ctypes.data, C.byref(nb),
            timeout_ms, C.byref(st)))
        return out, int(nb.value), dfm.Engine._stats(st)

    def sort_pr_device(self, delta, acc, n_total: int, out, timeout_ms: int = 300_000):
        """delta: (k, n_local) int32 CUDA tensor, acc: (n_local,) uint8, out: (n_local,)
        int32 — this rank's canonical labels are written there."""
        dfm = self.dfm
        k, nl = delta.shape
        nb = C.c_uint32(0)
        st = dfm._CStats()
        self.engine._check(self.lib.dfm_sort_pr_sharded_dev(
            self.handle, n_total, nl, k, delta.data_ptr(), acc.data_ptr(), out.data_ptr(),
            C.byref(nb), timeout_ms, C.byref(st)))
        return int(nb.value), dfm.Engine._stats(st)

    def close(self):
        if self.handle:
            self.lib.dfm_ctx_destroy(self.handle)
            self.handle = None
            self.engine.handle = None
