"""compute-sanitizer driver: a few small engine calls that
cover the cooperative / cluster / persistent kernels and a 1e6 sortPR, each
checked against the oracle so a silent corruption also fails.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --small
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2410_22764_b200 as dfm  # noqa: E402
from oracle import oracle as O  # noqa: E402

small = "--small" in sys.argv
eng = dfm.Engine(0)
MIN = dfm.PrOptions(policy=dfm.RacePolicy.deterministic_min, timeout_ms=3_600_000)
LIM = dfm.Limits(timeout_ms=3_600_000)
cases = [("random", O.random_dfa(3000, 3, 7, 0.5)),      # small sortPR kernel, fused naive
         ("fib", O.fib_dfa(9 if small else 12)),           # cluster naive (n <= 4096), trans
         ("comb", O.comb_dfa(300 if small else 2000, 3))]
if not small:
    cases.append(("random1e6", O.random_dfa(1_000_000, 4, 3, 0.5)))  # hash engine passes
    cases.append(("vlts", O.vlts_dfa(500, 200_000, 12)))              # hashed keys + rows
for name, (delta, acc) in cases:
    d = dfm.Dfa(acc.size, delta.shape[0], delta, acc, 0)
    ref = O.sort_pr(delta, acc)
    r = eng.sort_pr(d, dfm.SortOptions(timeout_ms=3_600_000))
    assert (r.partition.block == ref.block).all(), name
    if acc.size <= 300_000:
        rn = eng.naive_pr(d, MIN)
        rm = O.naive_pr(delta, acc, "min")
        assert (rn.partition.block == rm.block).all() and rn.stats.iterations == rm.iterations
        assert (eng.naive_pr_cas(d, timeout_ms=3_600_000).partition.block == ref.block).all(), name
        rt = eng.trans_pr(d, MIN, LIM)
        assert (rt.partition.block == ref.block).all(), name
    if acc.size <= 256:
        for engine in ("bit", "tensor"):
            eng.set_trans_engine(engine)
            rt = eng.trans_minimize(d, LIM)
            assert (rt.partition.block == ref.block).all(), (name, engine)
        eng.set_trans_engine("auto")
    print("ok", name, acc.size, flush=True)
if small:  # racecheck is ~1000x slower: the shared-memory kernels above are the target
    print("sanitize run complete")
    sys.exit(0)
rr = dfm.Engine(0)
rr.set_sortpr_engine("radix")
delta, acc = O.random_dfa(200_000, 2, 11, 0.5)
assert (rr.sort_pr(dfm.Dfa(acc.size, 2, delta, acc, 0)).partition.block ==
        O.sort_pr(delta, acc).block).all()
print("sanitize run complete")
