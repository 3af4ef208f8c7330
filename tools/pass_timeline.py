"""Per-pass host timestamps of sortPR on random_dfa(1e8, 4) (DFM_SORTPR_PASS_TIMING=1:
the library syncs at each pass end and prints the elapsed time and whether the
side-stream layout is ready) under a few route switches; timing syncs distort the
totals slightly, they are for the shape of the critical path."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, time
sys.path.insert(0, %r)
import paper_2410_22764_b200 as dfm
eng = dfm.Engine(0)
dd = eng.random_dfa_device(100_000_000, 4, 1, 0.5)
for _ in range(3):
    nb, st = eng.run_device(dfm.Algo.sort, dd)
    print("total", st.elapsed_ms, file=sys.stderr, flush=True)
''' % ROOT
for env in ({}, {"DFM_SORTPR_LAYOUT_OVERLAP": "0"}, {"DFM_SORTPR_DIRECT": "1"},
            {"DFM_SORTPR_DIRECT": "1", "DFM_SORTPR_LAYOUT_OVERLAP": "0"}):
    e = dict(os.environ, DFM_SORTPR_PASS_TIMING="1", **env)
    r = subprocess.run([sys.executable, "-c", CODE], env=e, capture_output=True, text=True)
    print("==", env or "default")
    print("\n".join(r.stderr.strip().splitlines()[-5:]))
