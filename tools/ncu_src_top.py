"""Top source lines by warp-stall samples from an `ncu --page source --csv` export
(several kernels concatenated): python tools/ncu_src_top.py file.csv [kernel-substr] [n]"""
import csv
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
kern, hdr, rows = None, None, {}
for r in csv.reader(open(path)):
    if r and r[0] == "Kernel Name":
        kern, hdr = r[1], None
        continue
    if hdr is None:
        hdr = r
        continue
    if want not in (kern or ""):
        continue
    rows.setdefault(kern, []).append(dict(zip(hdr, r)))
for k, rs in rows.items():
    tot = sum(float(x.get("Warp Stall Sampling (All Samples)") or 0) for x in rs)
    print(f"== {k[:100]}  samples {tot:.0f}")
    stalls = [h for h in (hdr or []) if h.startswith("stall_") and "Not Issued" not in h]
    for x in sorted(rs, key=lambda x: -float(x.get("Warp Stall Sampling (All Samples)") or 0))[:top]:
        s = float(x.get("Warp Stall Sampling (All Samples)") or 0)
        br = sorted(((float(x.get(h) or 0), h[6:]) for h in stalls), reverse=True)[:3]
        print(f"{100 * s / max(tot, 1):5.1f}%  {x.get('Address', x.get('#', ''))[:6]:>6} "
              f"{x.get('Source', '')[:70]:70s} {' '.join(f'{b}:{v:.0f}' for v, b in br)}")
