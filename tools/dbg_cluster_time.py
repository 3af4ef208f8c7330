import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_2410_22764_b200 as dfm
from oracle import oracle as O
eng = dfm.Engine(0)
MIN = dfm.RacePolicy.deterministic_min
for name, pair in [("rand8000", O.random_dfa(8000, 2, 4, 0.5)), ("fib17", O.fib_dfa(17)), ("rand20000", O.random_dfa(20000, 2, 5, 0.5))]:
    n = pair[1].size
    d = dfm.Dfa(n, pair[0].shape[0], pair[0], pair[1], 0)
    for c in ("1", "0"):
        os.environ["DFM_NAIVE_CLUSTER"] = c
        eng.naive_pr(d, dfm.PrOptions(policy=MIN))
        t = time.perf_counter()
        for _ in range(5):
            r = eng.naive_pr(d, dfm.PrOptions(policy=MIN))
        print(name, n, "cluster" if c == "1" else "global", r.stats.iterations, "%.2f ms" % ((time.perf_counter() - t) / 5 * 1e3))
