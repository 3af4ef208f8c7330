"""Per-family and whole-step DRAM bytes of ONE sortPR step, from an ncu launch list
captured with
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv \
        python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
(one row per kernel and metric; the generator kernels before the step are skipped).
Writes profiles/ncu_traffic.json, which bench.py reports as roofline.traffic (key
"step") and families[*].ncu_dram_bytes_per_step.
usage: python tools/ncu_step_traffic.py launches.csv profiles/ncu_traffic.json"""
import csv
import json
import re
import sys

FAMILY = [  # kernel-name regex -> bench.py ProfScope family (csrc/sortpr_hash.cu)
    (r"insert_small_kernel|lay_gather_kernel|lay_sig_kernel|direct_keys_kernel", "sig"),
    (r"insert_kernel|filt_set_kernel|filt_mark_kernel|PresentIn|CandIn", "insert"),
    (r"rip_groups_kernel|rip_hashed_kernel|resolve_kernel|ActIn", "scan"),
    (r"apply_kernel|rip_flag_kernel", "relabel"),
    (r"lay_count_kernel|lay_transpose_kernel|LayOffIn|lay_scatter_kernel", "layout"),
    (r"init_kernel|first_states_kernel|sanitize_rows_kernel", "init"),
    (r"mirror_kernel|mirror_packed_kernel", "mirror"),
    (r"iota_kernel|canon_gather_kernel|LeadIn", "canon"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}


def main(src, out):
    lines = open(src).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    per = {}
    for r in csv.DictReader(lines[start:]):
        k = (int(r["ID"]), r["Kernel Name"])
        per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * \
            SCALE.get(r["Metric Unit"], 1)
    fam, ms, detail = {}, {}, {}
    for (i, name), m in sorted(per.items()):
        f = next((f for pat, f in FAMILY if re.search(pat, name)), None)
        if f is None:
            continue
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        fam[f] = fam.get(f, 0.0) + b
        ms[f] = ms.get(f, 0.0) + m.get("gpu__time_duration.sum", 0) / 1e6
        short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", ""))
        detail.setdefault(f, []).append(f"{short[:60]} {b / 1e9:.2f} GB")
    old = {}
    try:
        old = json.load(open(out))
    except Exception:
        pass
    res = {"_doc": "DRAM bytes (read+write) of each kernel family for ONE step (one complete "
                   "minimization of random_dfa(1e8,4,1)) and the whole step ('step'), from "
                   f"the ncu launch list {src} (tools/ncu_step_traffic.py; cold caches, "
                   "serialised launches); bench.py reports them beside the algorithmic bytes.",
           "step": round(sum(fam.values()), -7),
           **{k: round(v, -7) for k, v in fam.items()},
           "_serialised_ms": {k: round(v, 3) for k, v in ms.items()}}
    if "gemm" in old:
        res["gemm"] = old["gemm"]
    res["_detail"] = {k: "; ".join(v) for k, v in detail.items()}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
