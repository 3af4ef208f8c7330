"""Pipelined host upload for sortPR (capi.cu upload_progressive): the rows land
chunk by chunk on a copy stream while the first pass and the layout build consume
them.  Must give exactly the device-resident result (itself pinned against the
oracle), and reject out-of-range targets like the one-shot upload does."""
import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _device_result(eng, dd, n):
    import torch
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = eng.run_device(dfm.Algo.sort, dd, block_out_ptr=out.data_ptr())
    assert st.status == dfm.RunStatus.ok
    return nb, st.iterations, out.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("n,k,seed", [(17_000_001, 4, 21), (40_000_000, 2, 22),
                                      (9_000_000, 8, 23), (70_000_003, 1, 24)])
def test_pipelined_upload_matches_device_run(eng, n, k, seed):
    dd = eng.random_dfa_device(n, k, seed, 0.5)
    nb, it, lab = _device_result(eng, dd, n)
    host = dd.download()
    dd.free()
    r = eng.sort_pr(host)
    assert r.stats.status == dfm.RunStatus.ok
    assert (r.partition.num_blocks, r.stats.iterations) == (nb, it)
    assert (r.partition.block == lab).all()


def test_pipelined_upload_non_identity_partition(eng):
    delta, acc = O.vlts_dfa(1000, 20_000_000, 4)
    d = dfm.Dfa(20_000_000, 4, delta, acc, 0)
    r = eng.sort_pr(d)
    dd = eng.upload(d)
    nb, it, lab = _device_result(eng, dd, 20_000_000)
    dd.free()
    assert r.partition.num_blocks == nb < 20_000_000 and r.stats.iterations == it
    assert (r.partition.block == lab).all()


def test_pipelined_upload_rejects_bad_target(eng):
    n, k = 17_000_000, 4
    delta, acc = O.random_dfa(n, k, 5, 0.5)
    delta[3, n - 1] = n  # last chunk, last row
    with pytest.raises(dfm.EngineError):
        eng.sort_pr(dfm.Dfa(n, k, delta, acc, 0))
    delta[3, n - 1] = 0
    r = eng.sort_pr(dfm.Dfa(n, k, delta, acc, 0))
    assert r.stats.status == dfm.RunStatus.ok


def test_pipelined_upload_timeout_then_reuse(eng):
    """A deadline that expires while the rows are still landing: timeout status,
    empty partition, and the engine (its copy stream drained) stays usable."""
    n, k = 40_000_000, 4
    delta, acc = O.random_dfa(n, k, 6, 0.5)
    d = dfm.Dfa(n, k, delta, acc, 0)
    r = eng.sort_pr(d, 1)
    assert r.stats.status == dfm.RunStatus.timeout and r.partition.block.size == 0
    r = eng.sort_pr(d)
    assert r.stats.status == dfm.RunStatus.ok and r.partition.num_blocks > 0


@pytest.mark.parametrize("p", [0.0, 1.0])
def test_pipelined_upload_single_initial_block(eng, p):
    """All states accepting (or none): one block after one pass, through the
    pipelined path as well."""
    n, k = 17_000_000, 4
    delta, acc = O.random_dfa(n, k, 7, p)
    r = eng.sort_pr(dfm.Dfa(n, k, delta, acc, 0))
    assert r.stats.status == dfm.RunStatus.ok
    assert (r.partition.num_blocks, r.stats.iterations) == (1, 1)
    assert not r.partition.block.any()


def test_pinned_and_pageable_rows_give_the_same_result(eng):
    """The same DFA from pageable rows (staged by the library through its pinned ring on
    a stager thread) and from pinned rows (DMA'd directly): identical results."""
    import torch
    n, k = 17_000_001, 4
    dd = eng.random_dfa_device(n, k, 31, 0.5)
    nb, it, lab = _device_result(eng, dd, n)
    host = dd.download()
    dd.free()
    pd = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
    pa = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pd.numpy()[:] = host.delta.view(np.int32)
    pa.numpy()[:] = host.accepting
    pinned = dfm.Dfa(n, k, pd.numpy().view(np.uint32), pa.numpy(), 0)
    for d in (host, pinned):
        r = eng.sort_pr(d)
        assert (r.partition.num_blocks, r.stats.iterations) == (nb, it)
        assert (r.partition.block == lab).all()
    # the one-shot upload (other algorithms) from both kinds of rows
    small = dfm.Dfa(n, k, host.delta, host.accepting, 0)
    for d in (small, pinned):
        dd2 = eng.upload(d)
        assert _device_result(eng, dd2, n)[2].tolist()[:1000] == lab.tolist()[:1000]
        dd2.free()


def test_concurrent_pageable_uploads_share_the_copy_pool(eng):
    """Two contexts on two host threads minimizing pageable DFAs at the same time: their
    staging copies take turns on the process's one host copy pool (capi.cu HostPool);
    each result equals its device-resident run.  A vlts input (non-identity partition,
    D2H) beside a random one (identity labels written by the speculative thread)."""
    import threading
    from paper_2410_22764_b200 import generators as G
    n1, k1 = 17_000_001, 4
    dd = eng.random_dfa_device(n1, k1, 41, 0.5)
    want1 = _device_result(eng, dd, n1)
    a = dd.download()
    dd.free()
    b = G.vlts_dfa(1000, 8_000_000, 6)
    db = eng.upload(b)
    want2 = _device_result(eng, db, b.num_states)
    db.free()
    engines = [eng, dfm.Engine(0)]
    got = [None, None]
    errs = []

    def run(i, d):
        try:
            for _ in range(2):
                got[i] = engines[i].sort_pr(d)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(0, a)), threading.Thread(target=run, args=(1, b))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r, (nb, it, lab) in zip(got, (want1, want2)):
        assert (r.partition.num_blocks, r.stats.iterations) == (nb, it)
        assert (r.partition.block == lab).all()
