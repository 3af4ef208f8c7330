"""e2e of the host-buffer sortPR on random_dfa(1e8, 4) with PAGEABLE rows (the
reference's std::vector Dfa) for several staging thread counts (DFM_STAGE_THREADS),
and with pinned rows, plus the raw pageable->pinned memcpy and H2D rates."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_22764_b200 as dfm  # noqa: E402

n, k = 100_000_000, 4
eng = dfm.Engine(0)
dd = eng.random_dfa_device(n, k, 1, 0.5)
host = dd.download()
dd.free()
page = dfm.Dfa(n, k, np.ascontiguousarray(host.delta), np.ascontiguousarray(host.accepting), 0)
out = np.empty(n, np.uint32)
res = {}
# the staging pool is sized once per process: one T per run (argv[1])
Ts = [int(a) for a in sys.argv[1:]] or [int(os.environ.get("DFM_STAGE_THREADS", "12"))]
for T in Ts:
    os.environ["DFM_STAGE_THREADS"] = str(T)
    eng.sort_pr(page, out=out)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        eng.sort_pr(page, out=out)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[f"pageable_T{T}"] = min(ts)
pin_d = torch.empty((k, n), dtype=torch.int32, pin_memory=True)
pin_a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pin_d.numpy()[:] = host.delta.view(np.int32)
pin_a.numpy()[:] = host.accepting
pin = dfm.Dfa(n, k, pin_d.numpy().view(np.uint32), pin_a.numpy(), 0)
eng.sort_pr(pin, out=out)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    eng.sort_pr(pin, out=out)
    ts.append((time.perf_counter() - t0) * 1e3)
res["pinned"] = min(ts)
buf = np.empty(host.delta.size, np.uint32)
t0 = time.perf_counter()
np.copyto(buf.reshape(host.delta.shape), host.delta)
res["numpy_copy_GBs_1thread"] = host.delta.nbytes / (time.perf_counter() - t0) / 1e9
print(res)
