"""Top CUDA source lines of one kernel by warp-stall samples, from an ncu report
(--page source --print-source cuda,sass).
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
fname = ""
h = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        h = r
        si = h.index("Warp Stall Sampling (All Samples)")
        stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if h is None or len(r) != len(h) or not r[0]:
        continue  # sass rows have an empty line number
    key = f"{fname}:{r[0]}  {r[1].strip()[:60]}"
    a = agg.setdefault(key, [0.0, {}])
    a[0] += float(r[si] or 0)
    for i in stalls:
        a[1][h[i][6:]] = a[1].get(h[i][6:], 0) + float(r[i] or 0)
tot = sum(v[0] for v in agg.values()) or 1
for k, (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = sorted(((v, nm) for nm, v in st.items()), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}%  {k:80s} " + " ".join(f"{nm}={v:.0f}" for v, nm in top if v > 0))
