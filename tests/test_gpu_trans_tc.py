"""GPU: the tcgen05 int8 squaring engine of the Cho–Huynh closure against the
CUDA-core bit engine, the oracle and the reference pins (test_min_trans.cpp)."""
import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O
from tests.helpers import to_dfa

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tc():
    e = dfm.Engine(0)
    e.set_trans_engine("tensor")
    return e


@pytest.fixture(scope="module")
def bit():
    e = dfm.Engine(0)
    e.set_trans_engine("bit")
    return e


def test_tensor_engine_matches_oracle_small(tc):
    rng = np.random.default_rng(81)
    for rnd in range(60):
        n = int(rng.integers(1, 41))
        k = int(rng.integers(1, 4))
        pair = O.random_dfa(n, k, int(rng.integers(1, 2 ** 62)), [0.0, 0.1, 0.5, 1.0][rnd % 4])
        ref = O.trans_minimize(*pair, inspect=(ins := {}))
        tins = dfm.TransInspect()
        r = tc.trans_minimize(to_dfa(pair), inspect=tins)
        assert (r.partition.block == ref.block).all(), (rnd, n, k)
        assert r.stats.iterations == ref.iterations, (rnd, n, k)
        assert tins.apart_popcounts == ins["apart_popcounts"].tolist()


def test_tensor_engine_pins(tc, pins):
    for idx, passes in {**pins["trans"]["fib_passes"]["values"],
                        **pins["trans"]["fib_10_11"]["values"]}.items():
        d = to_dfa(O.fib_dfa(int(idx)))
        r = tc.trans_minimize(d)
        assert (r.stats.iterations, r.partition.num_blocks) == (passes, d.num_states), idx


def test_tensor_engine_matches_bit_engine_large(tc, bit):
    for n, k, seed in ((100, 2, 3), (128, 2, 1), (160, 1, 5), (200, 4, 7)):
        d = to_dfa(O.random_dfa(n, k, seed, 0.5))
        ti, bi = dfm.TransInspect(), dfm.TransInspect()
        a = tc.trans_minimize(d, inspect=ti)
        b = bit.trans_minimize(d, inspect=bi)
        assert (a.partition.block == b.partition.block).all(), n
        assert a.stats.iterations == b.stats.iterations
        assert ti.apart_popcounts == bi.apart_popcounts
        assert (ti.apart == bi.apart).all()


def test_tile_skipping_matches_dense(tc, monkeypatch):
    """The tensor squaring skips K blocks whose 128x128 tiles are all zero; forcing
    every tile occupied (DFM_TRANS_DENSE=1) gives the same partition, passes and
    apartness trace."""
    for pair in (O.fib_dfa(10), O.random_dfa(100, 2, 3, 0.5)):
        d = to_dfa(pair)
        ins = dfm.TransInspect()
        r = tc.trans_minimize(d, inspect=ins)
        monkeypatch.setenv("DFM_TRANS_DENSE", "1")
        ins0 = dfm.TransInspect()
        r0 = tc.trans_minimize(d, inspect=ins0)
        monkeypatch.delenv("DFM_TRANS_DENSE")
        assert (r.partition.block == r0.partition.block).all()
        assert r.stats.iterations == r0.stats.iterations
        assert ins.apart_popcounts == ins0.apart_popcounts
