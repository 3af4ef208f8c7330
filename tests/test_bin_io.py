"""Bulk input path: binary DFA files.  Host write/read needs no
GPU; the device load/save round trip and minimization of a loaded file do."""
import os

import numpy as np
import pytest

import paper_2410_22764_b200 as dfm
from oracle import oracle as O


def test_host_roundtrip(tmp_path):
    for n, k, ini in ((1, 0, 0), (5, 1, 3), (1001, 3, 17), (4096, 4, 4095)):
        delta, acc = O.random_dfa(n, max(k, 1), n + k, 0.5)
        delta = delta[:k]
        d = dfm.Dfa(n, k, np.ascontiguousarray(delta), acc, ini)
        p = str(tmp_path / f"d{n}.dfmb")
        dfm.write_dfa_bin(p, d)
        e = dfm.read_dfa_bin(p)
        assert (e.num_states, e.alphabet_size, e.initial) == (n, k, ini)
        assert (e.delta == delta).all() and (e.accepting == acc).all()
        assert os.path.getsize(p) == 24 + ((n + 3) & ~3) + 4 * n * k


def test_bad_files(tmp_path):
    p = tmp_path / "bad.dfmb"
    p.write_bytes(b"NOTADFA0" + bytes(16))
    with pytest.raises(ValueError):
        dfm.read_dfa_bin(str(p))


@pytest.mark.gpu
def test_device_load_save_and_minimize(tmp_path, eng):
    n, k = 3_000_000, 4
    dd = eng.random_dfa_device(n, k, 3, 0.5)
    p = str(tmp_path / "big.dfmb")
    dd.save_bin(p)
    host = dd.download()
    e = dfm.read_dfa_bin(p)
    assert (e.delta == host.delta).all() and (e.accepting == host.accepting).all()
    d2 = eng.load_bin(p)
    back = d2.download()
    assert (back.delta == host.delta).all() and (back.accepting == host.accepting).all()
    nb1, st1 = eng.run_device(dfm.Algo.sort, dd)
    nb2, st2 = eng.run_device(dfm.Algo.sort, d2)
    assert (nb1, st1.iterations) == (nb2, st2.iterations)
    # a corrupt target is rejected on load (core.hpp:104-119 validation)
    bad = e.delta.copy()
    bad[1, 7] = n + 5
    dfm.write_dfa_bin(p, dfm.Dfa(n, k, bad, e.accepting, 0))
    with pytest.raises(dfm.EngineError):
        eng.load_bin(p)
    dd.free()
    d2.free()
