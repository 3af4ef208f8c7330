"""Host-side synthetic inputs (generators.hpp:16-145 plus the builder-defined
comb and VLTS-shaped families of SURVEY.md §8(d)).  Input synthesis only — the
minimizers never call these.  `random_dfa` lives in libdfm (multi-threaded,
and bit-exact on device too); the rest are numpy restatements, bit-exact with
the reference generators (checked in tests/test_generators.py)."""
from __future__ import annotations

import numpy as np

from . import Dfa, random_dfa  # noqa: F401  (re-exported)

_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _draws(seed: int, first: int, count: int) -> np.ndarray:
    """Draws first..first+count-1 of SplitMix64(seed) (counter-based, generators.hpp:21-26)."""
    with np.errstate(over="ignore"):
        j = np.arange(first + 1, first + count + 1, dtype=np.uint64)
        return _mix(np.uint64(seed) + j * _G)


class _SplitMix64:
    def __init__(self, seed: int):
        self.s = seed & (2 ** 64 - 1)

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        return z ^ (z >> 31)

    def below(self, b: int) -> int:
        return self.next() % b

    def unit(self) -> float:
        return (self.next() >> 11) * (1.0 / 9007199254740992.0)


def fib_word_bits(idx: int) -> np.ndarray:
    """w_0 = "1", w_1 = "0", w_{i} = w_{i-1} ++ w_{i-2} (generators.hpp:36-48)."""
    prev, cur = np.array([1], np.uint8), np.array([0], np.uint8)
    if idx == 0:
        return prev
    for _ in range(2, idx + 1):
        prev, cur = cur, np.concatenate([cur, prev])
    return cur


def fib_dfa(idx: int) -> Dfa:  # generators.hpp:53-68
    if idx < 2 or idx > 45:
        raise ValueError("fib_dfa needs 2 <= idx <= 45")
    acc = fib_word_bits(idx)
    n = acc.size
    delta = ((np.arange(n, dtype=np.uint64) + 1) % n).astype(np.uint32)[None, :]
    return Dfa(n, 1, delta, acc, 0)


def chain_dfa(length: int) -> Dfa:  # generators.hpp:111-125
    if length < 2 or length > 0x7FFFFFFF:
        raise ValueError("chain_dfa needs 2 <= len < 2^31")
    delta = np.minimum(np.arange(1, length + 1, dtype=np.uint32), length - 1)[None, :]
    acc = np.zeros(length, np.uint8)
    acc[-1] = 1
    return Dfa(length, 1, delta, acc, 0)


def bit_splitter(bits: int) -> Dfa:  # generators.hpp:76-107 (closed form, test_generators.cpp:17-23)
    if bits < 1 or bits > 26:
        raise ValueError("bit_splitter needs 1 <= bits <= 26")
    n = 1 << bits
    q = np.arange(n, dtype=np.uint32)
    delta = np.empty((bits - 1, n), np.uint32)
    for letter in range(bits - 1):
        m = letter + 1
        setb = ((q >> (m - 1)) & 1) != 0
        high = (q >> (m + 1)) << (m + 1)
        flipped = (((q >> m) & 1) ^ 1) << m
        delta[letter] = np.where(setb, high | flipped, q)
    acc = (q >= n // 2).astype(np.uint8)
    return Dfa(n, bits - 1, delta, acc, 0)


def comb_dfa(L: int, t: int) -> Dfa:
    """comb(L, t): spine 0..L-1 on a (last spine state loops and
    accepts), b from spine i to tooth L+i*t, teeth chain on b into the sink, last
    tooth state accepting, sink n-1 rejecting."""
    n = L * (t + 1) + 1
    sink = n - 1
    da = np.full(n, sink, np.uint32)
    db = np.full(n, sink, np.uint32)
    acc = np.zeros(n, np.uint8)
    i = np.arange(L, dtype=np.uint32)
    da[:L] = np.minimum(i + 1, L - 1)
    db[:L] = L + i * t
    acc[L - 1] = 1
    for j in range(t):
        s = L + i * t + j
        db[s] = s + 1 if j + 1 < t else sink
        if j + 1 == t:
            acc[s] = 1
    return Dfa(n, 2, np.vstack([da, db]), acc, 0)


def vlts_dfa(m: int, n: int, k: int, base_seed: int = 7, inflate_seed: int = 9, p: float = 0.4,
             window: int = 16) -> Dfa:
    """VLTS-shaped inflated quotient, SURVEY.md 8(d) C2 (<= m blocks)."""
    if m < 2 or k < 1 or n % m != 0:
        raise ValueError("vlts_dfa needs m >= 2, k >= 1, n % m == 0")
    bd = np.full((k, m), m - 1, np.uint32)
    ba = np.ones(m, np.uint8)
    ba[m - 1] = 0
    rng = _SplitMix64(base_seed)
    for q in range(m - 1):
        deg = 1
        while deg < k and rng.unit() > p:
            deg += 1
        for _ in range(deg):
            u1 = rng.unit()
            u2 = rng.unit()
            a = int(float(k) * u1 * u2)
            if rng.unit() < 0.8:
                tgt = (q + 1 + rng.below(window)) % (m - 1)
            else:
                tgt = rng.below(m - 1)
            bd[a, q] = tgt
    copies = n // m
    r = (_draws(inflate_seed, 0, n * k) % np.uint64(copies)).astype(np.uint32).reshape(n, k).T
    q = np.arange(n) % m
    delta = bd[:, q] + np.uint32(m) * r
    return Dfa(n, k, np.ascontiguousarray(delta), ba[q].copy(), 0)
