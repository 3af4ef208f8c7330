"""GPU: the sharded sortPR with the real libdfm device primitives
(CudaShardOps): world 1 over NCCL, and world 2 sharing one GPU over gloo
(host-staged collectives), against the oracle's partition and pass count."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, cases, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_2410_22764_b200 as dfm
    from paper_2410_22764_b200.sharded import Comm, CudaShardOps, shard_bounds, sharded_sort_pr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    eng = dfm.Engine(0)
    ops = CudaShardOps(eng)
    out = []
    for spec in cases:
        if spec[0] == "random-device":
            _, n, k, seed = spec
            lo, hi = shard_bounds(n, world, rank)
            delta, acc = ops.random_slice(n, k, seed, 0.5, lo, hi - lo)
        else:
            d, a = spec[1]
            n = a.size
            lo, hi = shard_bounds(n, world, rank)
            delta = torch.from_numpy(d[:, lo:hi].astype(np.int32)).cuda()
            acc = torch.from_numpy(a[lo:hi]).cuda()
        r = sharded_sort_pr(delta, acc, n, lo, Comm(), ops)
        out.append((lo, r.block_local.cpu().numpy(), r.num_blocks, r.iterations))
    q.put((rank, out))
    dist.destroy_process_group()


def _run(world, backend, cases):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, cases, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


CASES = [("host", O.random_dfa(20000, 3, 11, 0.5)), ("host", O.fib_dfa(11)),
         ("host", O.comb_dfa(200, 3)), ("host", O.vlts_dfa(100, 50000, 8)),
         ("random-device", 300000, 4, 1)]


def _check(res, world):
    for ci, spec in enumerate(CASES):
        if spec[0] == "random-device":
            d, a = O.random_dfa(spec[1], spec[2], spec[3], 0.5)
        else:
            d, a = spec[1]
        ref = O.sort_pr(d, a)
        full = np.empty(a.size, np.int64)
        for r in range(world):
            lo, blk, nb, it = res[r][ci]
            full[lo:lo + blk.size] = blk
            assert (nb, it) == (ref.num_blocks, ref.iterations), (ci, r)
        assert (full == ref.block).all(), ci


def test_sharded_world1_nccl():
    _check(_run(1, "nccl", CASES), 1)


def test_sharded_world2_one_gpu_gloo():
    _check(_run(2, "gloo", CASES), 2)
