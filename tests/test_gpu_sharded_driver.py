"""GPU: the C++ sharded sortPR driver (csrc/shard_driver.cu) through the C-ABI
(dfm_sort_pr_sharded[_dev]).

* world 2/3/4 with the in-process "local" transport: ranks are threads of this
  process on the one GPU, so the whole C++ protocol (narrow all-gathers, keys,
  routing, grouping, offsets, reverse exchange, canonical labels) runs exactly as
  over NCCL, minus the NCCL calls themselves;
* world 1 over a real NCCL communicator (ncclCommInitRank), with the protocol
  forced (DFM_SHARD_PROTOCOL=1) and with the single-GPU engine it delegates to.

Bar: bit-exact canonical partition, block count and pass count against the oracle
and the reference's config-size records (tests/golden/config_vectors.json)."""
import json
import os
import threading

import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O
from paper_2410_22764_b200.sharded import ShardedEngine
from tests.helpers import digest

pytestmark = pytest.mark.gpu
_group_id = [0]


def _local(world, delta, acc, gather_all=True, dev_side=False):
    """Run the driver at `world` local ranks; returns per-rank (labels, nb, stats)."""
    _group_id[0] += 1
    group = f"t{_group_id[0]}"
    n = acc.size
    k = delta.shape[0]
    res = [None] * world
    err = []

    def worker(r):
        try:
            se = ShardedEngine(0, r, world, "local", group)
            lo, hi = se.bounds(n)
            if dev_side:
                import torch
                d = torch.from_numpy(np.ascontiguousarray(delta[:, lo:hi]).view(np.int32)).cuda()
                a = torch.from_numpy(np.ascontiguousarray(acc[lo:hi])).cuda()
                out = torch.empty(max(hi - lo, 1), dtype=torch.int32, device="cuda")
                nb, st = se.sort_pr_device(d, a, n, out)
                torch.cuda.synchronize()
                res[r] = (out[:hi - lo].cpu().numpy().view(np.uint32), nb, st, lo)
            else:
                local = dfm.Dfa(hi - lo, k, np.ascontiguousarray(delta[:, lo:hi]),
                                np.ascontiguousarray(acc[lo:hi]), 0)
                lab, nb, st = se.sort_pr(local, n, gather_all=gather_all)
                res[r] = (lab, nb, st, lo)
            se.close()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    return res


def _check(res, ref, gather_all=True):
    full = None
    for lab, nb, st, lo in res:
        assert st.status == dfm.RunStatus.ok
        assert nb == ref.num_blocks
        assert st.iterations == ref.iterations
        if gather_all:
            assert (lab == ref.block).all()
            full = lab
    if not gather_all:
        full = np.concatenate([r[0] for r in sorted(res, key=lambda x: x[3])])
        assert (full == ref.block).all()
    return full


CASES = [
    ("random_5k3", lambda: O.random_dfa(5000, 3, 21, 0.5)),
    ("vlts_hashed", lambda: O.vlts_dfa(200, 20_000, 10)),   # B up to 196: hashed keys + rows
    ("comb", lambda: O.comb_dfa(300, 3)),
    ("fib12", lambda: O.fib_dfa(12)),
    ("tiny5", lambda: O.random_dfa(5, 2, 3, 0.5)),             # an empty shard at world 4
    ("all_accepting", lambda: O.random_dfa(3000, 2, 5, 1.0)),  # one block
    ("bits6", lambda: O.bit_splitter(6)),
]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("name,make", CASES, ids=[c[0] for c in CASES])
def test_local_transport_vs_oracle(world, name, make, monkeypatch):
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")  # world 1 runs the protocol too
    delta, acc = make()
    ref = O.sort_pr(delta, acc)
    _check(_local(world, delta, acc, gather_all=True), ref)
    _check(_local(world, delta, acc, gather_all=False), ref, gather_all=False)


def test_local_transport_device_path_c1(monkeypatch):
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    delta, acc = O.random_dfa(100_000, 2, 1, 0.5)
    ref = O.sort_pr(delta, acc)
    for world in (2, 3):
        _check(_local(world, delta, acc, dev_side=True), ref, gather_all=False)


def test_local_transport_config_vectors(monkeypatch):
    """The reference's records at config size: C1 seed 2 and vlts(1000, 1e6, 20) sort,
    through 2 and 3 local ranks."""
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    with open(os.path.join(os.path.dirname(__file__), "golden", "config_vectors.json")) as f:
        vec = {v["name"]: v for v in json.load(f)["vectors"]}
    for name, pair in (("c1_random_1e5_k2_s2", O.random_dfa(100_000, 2, 2, 0.5)),
                       ("c2_vlts_1000_1e6_20", O.vlts_dfa(1000, 1_000_000, 20))):
        exp = vec[name]["sort"]
        for world in (2, 3):
            res = _local(world, *pair, gather_all=True)
            for lab, nb, st, lo in res:
                assert (nb, st.iterations) == (exp["num_blocks"], exp["iterations"]), name
                assert digest(lab) == exp["sha256"], name


def test_nccl_world1(monkeypatch):
    """A real NCCL communicator of one rank; the protocol forced and the engine path."""
    delta, acc = O.vlts_dfa(200, 20_000, 10)
    ref = O.sort_pr(delta, acc)
    for forced in ("1", "0"):
        monkeypatch.setenv("DFM_SHARD_PROTOCOL", forced)
        se = ShardedEngine(0, 0, 1, "nccl")
        assert se.info() == (0, 1, "nccl")
        lab, nb, st = se.sort_pr(dfm.Dfa(acc.size, delta.shape[0], delta, acc, 0), acc.size)
        assert (lab == ref.block).all() and nb == ref.num_blocks
        assert st.iterations == ref.iterations
        se.close()


def test_out_of_range_target_rejected_on_every_rank(monkeypatch):
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    delta, acc = O.random_dfa(1000, 2, 9, 0.5)
    delta = delta.copy()
    delta[1, 700] = 5000  # owned by rank 1 of 2
    n = acc.size
    errs = []

    def worker(r):
        se = ShardedEngine(0, r, 2, "local", "bad_target")
        lo, hi = se.bounds(n)
        try:
            se.sort_pr(dfm.Dfa(hi - lo, 2, np.ascontiguousarray(delta[:, lo:hi]),
                               np.ascontiguousarray(acc[lo:hi]), 0), n)
        except dfm.EngineError as e:
            errs.append(str(e))
        se.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert len(errs) == 2 and all("out of range" in e for e in errs)


def _local_device_random(world, n, k, seed):
    """random_dfa slices generated on the device per rank; returns the whole
    canonical partition (gathered) and (nb, passes) of every rank."""
    import torch
    _group_id[0] += 1
    group = f"d{_group_id[0]}"
    res = [None] * world
    err = []

    def worker(r):
        try:
            import ctypes as C
            se = ShardedEngine(0, r, world, "local", group)
            lo, hi = se.bounds(n)
            d = torch.empty((k, max(hi - lo, 1)), dtype=torch.int32, device="cuda")
            a = torch.empty(max(hi - lo, 1), dtype=torch.uint8, device="cuda")
            f = se.lib.dfm_random_dfa_slice_dev
            f.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, C.c_uint64,
                          C.c_uint64, C.c_void_p, C.c_void_p]
            assert f(se.handle, n, k, seed, 0.5, lo, hi - lo, d.data_ptr(), a.data_ptr()) == 0
            d, a = d[:, :hi - lo].contiguous(), a[:hi - lo]
            out = torch.empty(max(hi - lo, 1), dtype=torch.int32, device="cuda")
            nb, st = se.sort_pr_device(d, a, n, out)
            torch.cuda.synchronize()
            res[r] = (lo, out[:hi - lo].cpu().numpy().view(np.uint32), nb, st.iterations)
            del d, a, out
            se.close()
        except Exception as e:  # pragma: no cover
            err.append(repr(e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not err, err
    full = np.concatenate([x[1] for x in sorted(res, key=lambda x: x[0])])
    return full, {(x[2], x[3]) for x in res}


@pytest.mark.parametrize("world", [1, 2, 3])
def test_blocked_shard_keys_match_single_engine(eng, monkeypatch, world):
    """32-bit id passes through the blocked builder over each rank's rows (targets =
    all states): same partition and pass count as the single-GPU engine."""
    import torch
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    n, k = 12_000_000, 4
    dd = eng.random_dfa_device(n, k, 41, 0.5)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = eng.run_device(dfm.Algo.sort, dd, block_out_ptr=out.data_ptr())
    ref = out.cpu().numpy().view(np.uint32)
    dd.free()
    full, stats = _local_device_random(world, n, k, 41)
    assert stats == {(nb, st.iterations)}
    assert (full == ref).all()


def test_blocked_shards_north_star_record(monkeypatch):
    """random_dfa(1e8, 4, 1) over 2 local ranks through the blocked shard builder
    against the reference's recorded result (tests/golden/config_vectors.json)."""
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    with open(os.path.join(os.path.dirname(__file__), "golden", "config_vectors.json")) as f:
        rec = {v["name"]: v for v in json.load(f)["vectors"]}["ns_random_1e8_k4_s1"]["sort"]
    full, stats = _local_device_random(2, 100_000_000, 4, 1)
    assert stats == {(rec["num_blocks"], rec["iterations"])}
    assert digest(full) == rec["sha256"]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_forced_hash_collisions_retry_exactly(world, monkeypatch):
    """DFM_SHARD_WEAK_HASH truncates the first seed's hashed keys: distinct signatures
    collide, the rows disagree on some rank, every rank voids the pass and redoes it
    under a new seed — the result is still the oracle's."""
    monkeypatch.setenv("DFM_SHARD_PROTOCOL", "1")
    monkeypatch.setenv("DFM_SHARD_WEAK_HASH", "6")
    for delta, acc in (O.vlts_dfa(200, 20_000, 10), O.random_dfa(30_000, 6, 13, 0.5)):
        ref = O.sort_pr(delta, acc)
        _check(_local(world, delta, acc, gather_all=True), ref)
