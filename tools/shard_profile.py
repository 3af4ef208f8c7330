"""Stage timing of the state-sharded sortPR driver at world 1 (1e8 states, k=4)."""
import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2410_22764_b200 as dfm
from paper_2410_22764_b200 import sharded as S

eng = dfm.Engine(0)
ops = S.CudaShardOps(eng)
comm = S.Comm()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
delta, acc = ops.random_slice(n, 4, 1, 0.5, 0, n)
times = {}
orig = {name: getattr(ops, name) for name in ("signature", "route", "group", "canonicalize")}
def wrap(name, f):
    def g(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); times[name] = times.get(name, 0) + time.perf_counter() - t
        return r
    return g
for name, f in orig.items():
    setattr(ops, name, wrap(name, f))
for c in ("all_gather", "all_to_all", "all_gather_ints"):
    setattr(comm, c, wrap(c, getattr(comm, c)))
S.sharded_sort_pr(delta, acc, n, 0, comm, ops)
times.clear()
torch.cuda.synchronize(); t = time.perf_counter()
r = S.sharded_sort_pr(delta, acc, n, 0, comm, ops)
torch.cuda.synchronize(); total = time.perf_counter() - t
print("total %.1f ms, passes %d" % (total * 1e3, r.iterations))
for k, v in sorted(times.items(), key=lambda kv: -kv[1]):
    print("  %-16s %.1f ms" % (k, v * 1e3))
