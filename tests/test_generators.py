"""CPU: the product's host generators are bit-exact with the oracle restatement
(itself pinned to the reference generators in test_oracle.py)."""
import numpy as np

from oracle import oracle as O
from paper_2410_22764_b200 import generators as G


def same(d, pair):
    delta, acc = pair
    return d.delta.shape == delta.shape and (d.delta == delta).all() and (d.accepting == acc).all()


def test_families_bit_exact():
    for i in (2, 3, 5, 9, 15):
        assert same(G.fib_dfa(i), O.fib_dfa(i))
    for b in (1, 2, 3, 7, 12):
        assert same(G.bit_splitter(b), O.bit_splitter(b))
    for L in (2, 3, 100, 4097):
        assert same(G.chain_dfa(L), O.chain_dfa(L))
    for L, t in ((1, 1), (64, 3), (100, 2)):
        assert same(G.comb_dfa(L, t), O.comb_dfa(L, t))
    for m, n, k in ((10, 100, 3), (1000, 20000, 10), (50, 5000, 1)):
        assert same(G.vlts_dfa(m, n, k), O.vlts_dfa(m, n, k))
    assert same(G.random_dfa(777, 3, 5, 0.3), O.random_dfa(777, 3, 5, 0.3))
