"""Measured dense int8 tensor-core throughput on this B200 (the roofline peak for the
Cho-Huynh tcgen05 kind::i8 squaring): cuBLASLt through torch._int_mm, int8 x int8 ->
int32, 8192^3 and 16384^3, best of 10 (burst), CUDA events.  Writes profiles/int8_peak.json."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
best = {}
for n in (8192, 16384):
    a = torch.randint(-2, 3, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-2, 3, (n, n), dtype=torch.int8, device="cuda")
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    best[n] = 2.0 * n ** 3 / (min(ts) / 1e3) / 1e12
out = {"int8_tops": max(best.values()), "by_size": {str(k): v for k, v in best.items()},
       "how": "torch._int_mm (cuBLASLt int8 IMMA) n^3, 2*n^3 ops, best of 10 per size, CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
if "--write" in sys.argv:
    with open(os.path.join(ROOT, "profiles", "int8_peak.json"), "w") as f:
        json.dump(out, f, indent=1)
