"""Shared test helpers: build inputs with the ORACLE generators (the checker side)
and wrap them in the product's Dfa type."""
import hashlib

import numpy as np

from oracle import oracle as O
import paper_2410_22764_b200 as dfm


def to_dfa(pair) -> "dfm.Dfa":
    delta, acc = pair
    return dfm.Dfa(int(acc.size), int(delta.shape[0]), delta, acc, 0)


def gen(spec):
    kind = spec[0]
    if kind == "random":
        _, n, k, seed, p = spec
        return O.random_dfa(n, k, seed, p)
    if kind == "fib":
        return O.fib_dfa(spec[1])
    if kind == "bits":
        return O.bit_splitter(spec[1])
    if kind == "chain":
        return O.chain_dfa(spec[1])
    if kind == "comb":
        return O.comb_dfa(spec[1], spec[2])
    if kind == "vlts":
        _, m, n, k = spec
        return O.vlts_dfa(m, n, k)
    raise ValueError(kind)


def digest(block) -> str:
    return hashlib.sha256(np.ascontiguousarray(block, dtype="<u4").tobytes()).hexdigest()
