"""CPU, world_size 2 and 3 over gloo: the sharded sortPR protocol
(paper_2410_22764_b200/sharded.py) reproduces the oracle's partition and pass
count, including after forced hash collisions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, weak, q, max_passes=None):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2410_22764_b200.sharded import Comm, shard_bounds, sharded_sort_pr
    from tests.sharded_cpu_ops import CpuShardOps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for delta, acc in cases:
        n = acc.size
        lo, hi = shard_bounds(n, world, rank)
        # the forced-collision run keeps hashed keys in every pass (packed exact keys
        # of the early passes cannot collide)
        r = sharded_sort_pr(torch.from_numpy(delta[:, lo:hi].astype(np.int32)),
                            torch.from_numpy(acc[lo:hi]), n, lo, Comm(), CpuShardOps(weak),
                            max_passes=max_passes, allow_packed=not weak)
        out.append((lo, r.block_local.numpy().copy(), r.num_blocks, r.iterations, r.retries,
                    r.converged))
    q.put((rank, out))
    dist.destroy_process_group()


def _run(world, cases, weak=False, max_passes=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, weak, q, max_passes))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _cases():
    return [O.random_dfa(3000, 3, 11, 0.5), O.fib_dfa(9), O.bit_splitter(6), O.comb_dfa(40, 3),
            O.random_dfa(500, 2, 5, 1.0), O.vlts_dfa(50, 2000, 6)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_oracle(world):
    cases = _cases()
    res = _run(world, cases)
    for ci, (delta, acc) in enumerate(cases):
        ref = O.sort_pr(delta, acc)
        full = np.empty(acc.size, np.int64)
        for r in range(world):
            lo, blk, nb, it, _, conv = res[r][ci]
            full[lo:lo + blk.size] = blk
            assert (nb, it) == (ref.num_blocks, ref.iterations), (ci, r)
            assert conv, (ci, r)
        assert (full == ref.block).all(), ci


def test_sharded_collision_retry_is_exact():
    cases = _cases()[:2]
    res = _run(2, cases, weak=True)
    for ci, (delta, acc) in enumerate(cases):
        ref = O.sort_pr(delta, acc)
        full = np.empty(acc.size, np.int64)
        for r in range(2):
            lo, blk, nb, it, retries, _ = res[r][ci]
            full[lo:lo + blk.size] = blk
            assert it == ref.iterations and retries >= 1
        assert (full == ref.block).all()


def test_sharded_max_passes_reports_not_converged():
    """A run cut at max_passes before the fixpoint says so (ShardedResult.converged)."""
    delta, acc = O.fib_dfa(9)
    assert O.sort_pr(delta, acc).iterations > 2
    res = _run(2, [(delta, acc)], max_passes=2)
    for r in range(2):
        _, _, _, it, _, conv = res[r][0]
        assert it == 2 and not conv
