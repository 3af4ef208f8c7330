"""GPU quotient / remove_unreachable against the oracle
restatement of core.hpp:152-187 / 256-290 (itself pinned against the reference in
tests/test_oracle.py::test_post_processing_vs_reference)."""
import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O
from tests.helpers import to_dfa

pytestmark = pytest.mark.gpu


def _dfa(pair, initial=0):
    d = to_dfa(pair)
    d.initial = initial
    return d


def test_quotient_matches_oracle(eng):
    rng = np.random.default_rng(77)
    for t in range(60):
        n = int(rng.integers(1, 400))
        k = int(rng.integers(0, 4))
        pair = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), [0, 0.1, 0.5, 1][t % 4])
        ini = int(rng.integers(0, n))
        ref = O.sort_pr(*pair)
        d = _dfa(pair, ini)
        q = eng.quotient(d, dfm.Partition(ref.block, ref.num_blocks))
        dq, aq, iq = O.quotient(*pair, ref.block, ref.num_blocks, ini)
        assert (q.delta == dq).all() and (q.accepting == aq).all() and q.initial == iq
        # the quotient is minimal
        assert eng.sort_pr(q).partition.num_blocks == ref.num_blocks


def test_quotient_errors_match_reference_messages(eng):
    rng = np.random.default_rng(78)
    for t in range(80):
        n = int(rng.integers(2, 80))
        pair = O.random_dfa(n, 2, int(rng.integers(1, 2 ** 62)), 0.5)
        raw = rng.integers(0, 4, n).astype(np.uint32)
        canon, nb = O.canonicalize(raw)
        for blk, nbb in ((raw, 4), (canon, nb), (canon, nb + 1)):
            want = None
            try:
                O.quotient(*pair, blk, nbb)
            except O.QuotientError as e:
                want = str(e)
            got = None
            try:
                eng.quotient(to_dfa(pair), dfm.Partition(blk, nbb))
            except ValueError as e:
                got = str(e)
            assert got == want, (t, got, want)


def test_quotient_at_scale_device(eng):
    """minimize on the device, quotient on the device, check minimality."""
    import torch
    n, k = 2_000_000, 3
    dd = eng.random_dfa_device(n, k, 5, 0.5)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    nb, st = eng.run_device(dfm.Algo.sort, dd, block_out_ptr=out.data_ptr())
    qd = dd.quotient(out.data_ptr(), nb)
    q = qd.download()
    host = dd.download()
    ref_q = O.quotient(host.delta, host.accepting, out.cpu().numpy().view(np.uint32), nb)
    assert (q.delta == ref_q[0]).all() and (q.accepting == ref_q[1]).all()
    qd.free()
    dd.free()


@pytest.mark.parametrize("case", ["random", "sparse", "chain", "comb", "k0"])
def test_remove_unreachable_matches_oracle(eng, case):
    rng = np.random.default_rng(79)
    for t in range(25):
        if case == "random":
            n = int(rng.integers(1, 3000))
            pair = O.random_dfa(n, int(rng.integers(1, 4)), int(rng.integers(1, 2 ** 62)), 0.5)
        elif case == "sparse":  # most states unreachable: targets drawn from a small prefix
            n = int(rng.integers(2, 3000))
            delta, acc = O.random_dfa(n, 2, int(rng.integers(1, 2 ** 62)), 0.5)
            delta = (delta % max(1, n // 7)).astype(np.uint32)
            pair = (delta, acc)
        elif case == "chain":
            pair = O.chain_dfa(int(rng.integers(1, 5000)))
        elif case == "comb":
            pair = O.comb_dfa(int(rng.integers(1, 300)), 3)
        else:
            n = int(rng.integers(1, 50))
            pair = (np.zeros((0, n), np.uint32), (rng.random(n) < 0.5).astype(np.uint8))
        n = pair[1].size
        ini = int(rng.integers(0, n))
        r = eng.remove_unreachable(_dfa(pair, ini))
        dq, aq, iq = O.remove_unreachable(*pair, ini)
        assert r.num_states == aq.size
        assert (r.delta == dq).all() and (r.accepting == aq).all() and r.initial == iq


def test_remove_unreachable_deep_chain(eng):
    """A 2^20-state chain: BFS depth n; the doubled alphabet finishes it in ~log n levels."""
    pair = O.chain_dfa(1 << 20)
    r = eng.remove_unreachable(_dfa(pair, 0))
    assert r.num_states == 1 << 20
    r = eng.remove_unreachable(_dfa(pair, (1 << 20) - 10))
    dq, aq, iq = O.remove_unreachable(*pair, (1 << 20) - 10)
    assert r.num_states == aq.size and (r.delta == dq).all() and r.initial == iq


def test_lts_pipeline_into_gpu_minimizers(eng):
    """VLTS front-end: parse -> determinize -> complete (host, libdfm)
    -> the GPU minimizers, against the reference's own pipeline and oracle."""
    import numpy as np
    from tests.test_ingest import det_lts_text, random_lts_text
    rng = np.random.default_rng(5)
    for text in (random_lts_text(rng, 40, 150, 3, 5), det_lts_text(rng, 3000, 4, 10)):
        d = dfm.complete(dfm.determinize(dfm.parse_lts(text)))
        r = O.ref_ingest(text)
        assert (d.delta == r["dfa"][0]).all() and (d.accepting == r["dfa"][1]).all()
        ref = O.sort_pr(*r["dfa"])
        got = eng.sort_pr(d)
        assert (got.partition.block == ref.block).all()
        assert got.stats.iterations == ref.iterations
        assert (eng.naive_pr(d, dfm.PrOptions(policy=dfm.RacePolicy.deterministic_min))
                .partition.block == ref.block).all()
