"""H2D bandwidth from pinned host memory: one copy vs split across streams."""
import torch, time
N = 1600 << 20
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        part = N // streams
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"streams={streams}: {N / best / 1e9:.1f} GB/s ({best * 1e3:.1f} ms for {N >> 20} MiB)")
dd = torch.empty(N, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
h.copy_(dd, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H: {N / (time.perf_counter() - t) / 1e9:.1f} GB/s")
