"""Per-family DRAM bytes of one sortPR step from an ncu --set full report of
`python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline` (all kernels):
writes the summary bench.py reports as roofline.traffic.
usage: python tools/ncu_traffic.py report.ncu-rep|raw.csv out.json"""
import csv
import io
import json
import re
import subprocess
import sys

FAMILY = [  # kernel-name regex -> bench.py ProfScope family
    (r"insert_small_kernel|lay_gather_kernel|lay_sig_kernel", "sig"),
    (r"insert_kernel|filt_set_kernel|filt_mark_kernel|PresentIn|CandIn", "insert"),
    (r"rip_groups_kernel|rip_hashed_kernel|resolve_kernel|ActIn", "scan"),
    (r"apply_kernel|rip_flag_kernel", "relabel"),
    (r"lay_count_kernel|lay_transpose_kernel|LayOffIn|lay_scatter_kernel", "layout"),
    (r"init_kernel|first_states_kernel|sanitize_rows_kernel", "init"),
    (r"mirror_kernel", "mirror"),
    (r"iota_kernel|canon_gather_kernel|LeadIn", "canon"),
]

rep, out = sys.argv[1], sys.argv[2]
if rep.endswith(".csv"):  # the raw page saved next to the run (tools/gpu_suite.sh)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki = h.index("Kernel Name")
rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(r, i):
    return float(r[i].replace(",", "")) * scale.get(units[i], 1)


fam, detail = {}, {}
for r in rows[2:]:
    name = r[ki]
    f = next((f for pat, f in FAMILY if re.search(pat, name)), None)
    if f is None:
        continue
    b = val(r, rd) + val(r, wr)
    fam[f] = fam.get(f, 0.0) + b
    short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", "").replace("dfm::", ""))
    detail.setdefault(f, []).append(f"{short[:60]} {b / 1e9:.2f} GB")
old = json.load(open(out)) if out else {}
res = {"_doc": old.get("_doc", "") if out else "", **{k: round(v, -7) for k, v in fam.items()}}
if "gemm" in old:
    res["gemm"] = old["gemm"]
res["_detail"] = {k: "; ".join(v) for k, v in detail.items()}
if "gemm" in old.get("_detail", {}):
    res["_detail"]["gemm"] = old["_detail"]["gemm"]
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
