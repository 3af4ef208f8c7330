"""Generate tests/golden/config_vectors.json: the UNMODIFIED reference's results at
the BASELINE.json config sizes (SURVEY.md §8(c)/(d), C1–C4 and the 1e8 north star).

TEST INFRASTRUCTURE ONLY.  Runs oracle/_ref/libdfamin_ref.so (compiled from
/root/reference/proj/include by oracle/Makefile) multi-threaded in the CPU
container and records, per (input, algorithm): sha256 of the canonical
partition (u32 little-endian), block count, pass count, closure steps, the
reference's peak-memory estimate, sortPR's per-pass block counts, and the
reference's own elapsed time and worker count (informational).

Inputs come from the reference's own generators where one exists
(random_dfa / fib_dfa / chain_dfa, generators.hpp:36-145) and from the
builder-defined comb / VLTS generators of SURVEY.md §8(d) otherwise (oracle
restatement; no reference counterpart).  The GPU tests
(tests/test_gpu_configs.py) regenerate the same inputs on the device or from
the product's bit-exact generators and compare.

    make -C oracle && python tests/golden/make_config_golden.py [--only NAME ...]

C5 (random_dfa(1e9, 4)) is not here: the reference needs ~50 GB of host RAM
plus a second copy in the shim; the sharded path is pinned at 1e8 against this
file and by size-independent properties at 1e9.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_vectors.json")


def digest(block: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(block, dtype="<u4").tobytes()).hexdigest()


# (name, config tag, spec, algorithms)
CASES = [
    ("c1_random_1e5_k2_s1", "C1", ("random", 100_000, 2, 1, 0.5), ("sort", "naive_min")),
    ("c1_random_1e5_k2_s2", "C1", ("random", 100_000, 2, 2, 0.5), ("sort", "naive_min")),
    ("c1_random_1e5_k2_s3", "C1", ("random", 100_000, 2, 3, 0.5), ("sort", "naive_min")),
    ("c2_vlts_1000_1e6_10", "C2", ("vlts", 1000, 1_000_000, 10), ("sort", "naive_min")),
    ("c2_vlts_1000_1e6_20", "C2", ("vlts", 1000, 1_000_000, 20), ("sort", "naive_min")),
    ("c2_vlts_1000_1e6_100", "C2", ("vlts", 1000, 1_000_000, 100), ("sort",)),
    ("c2_vlts_5000_1e6_50", "C2", ("vlts", 5000, 1_000_000, 50), ("sort",)),
    ("c2_vlts_1000_1e7_10", "C2", ("vlts", 1000, 10_000_000, 10), ("sort",)),
    ("c2_vlts_1000_1e7_100", "C2", ("vlts", 1000, 10_000_000, 100), ("sort",)),
    ("c3_chain_1048576", "C3", ("chain", 1 << 20), ("transpr_min",)),
    ("c3_chain_1e6", "C3", ("chain", 1_000_000), ("transpr_min",)),
    ("c3_chain_1e7", "C3", ("chain", 10_000_000), ("transpr_min",)),
    ("c3_comb_1e6_3", "C3", ("comb", 1_000_000, 3), ("transpr_min",)),
    ("c3_fib_21", "C3", ("fib", 21), ("transpr_min", "naive_min", "sort")),
    ("c4_fib_10", "C4", ("fib", 10), ("trans",)),
    ("c4_fib_11", "C4", ("fib", 11), ("trans",)),
    ("c4_fib_12", "C4", ("fib", 12), ("trans",)),
    ("c4_random_64_k2", "C4", ("random", 64, 2, 1, 0.5), ("trans",)),
    ("c4_random_128_k2", "C4", ("random", 128, 2, 1, 0.5), ("trans",)),
    ("c4_random_192_k2", "C4", ("random", 192, 2, 1, 0.5), ("trans",)),
    ("c4_random_256_k2", "C4", ("random", 256, 2, 1, 0.5), ("trans",)),
    ("c4_random_256_k1", "C4", ("random", 256, 1, 1, 0.5), ("trans",)),
    ("c4_random_256_k4", "C4", ("random", 256, 4, 1, 0.5), ("trans",)),
    ("ns_random_1e8_k4_s1", "north-star", ("random", 100_000_000, 4, 1, 0.5), ("sort",)),
]


def make_input(R, spec):
    kind = spec[0]
    if kind == "random":
        _, n, k, seed, p = spec
        return R.random_dfa(n, k, seed, p)  # the reference's own generator
    if kind == "fib":
        return R.fib_dfa(spec[1])
    if kind == "chain":
        return R.chain_dfa(spec[1])
    if kind == "comb":
        return O.comb_dfa(spec[1], spec[2])
    if kind == "vlts":
        _, m, n, k = spec
        return O.vlts_dfa(m, n, k)
    raise ValueError(kind)


def run(R, algo, delta, acc):
    tc = []
    if algo == "sort":
        r = R.sort_pr(delta, acc, timeout_ms=3_600_000, trace_counts=tc)
    elif algo == "naive_min":
        r = R.naive_pr(delta, acc, "min", timeout_ms=3_600_000)
    elif algo == "transpr_min":
        r = R.trans_pr(delta, acc, "min", timeout_ms=3_600_000, max_memory_bytes=48 << 30)
    elif algo == "trans":
        r = R.trans_minimize(delta, acc, timeout_ms=3_600_000, max_memory_bytes=48 << 30)
    else:
        raise ValueError(algo)
    assert r.status == "ok", (algo, r.status)
    e = {"num_blocks": r.num_blocks, "iterations": r.iterations,
         "closure_steps": r.closure_steps, "peak_memory_estimate": r.peak_memory_estimate,
         "sha256": digest(r.block), "ref_elapsed_ms": r.elapsed_ms}
    if algo == "sort":
        e["trace_counts"] = tc
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    R = O.Reference()
    R.set_threads(args.threads)
    old = {}
    if os.path.exists(PATH):
        with open(PATH) as f:
            old = {v["name"]: v for v in json.load(f)["vectors"]}
    out = []
    for name, tag, spec, algos in CASES:
        if args.only and name not in args.only and name in old:
            out.append(old[name])
            continue
        t0 = time.time()
        delta, acc = make_input(R, spec)
        rec = {"name": name, "config": tag, "spec": list(spec), "n": int(acc.size),
               "k": int(delta.shape[0]), "input_sha256": hashlib.sha256(
                   delta.tobytes() + acc.tobytes()).hexdigest()}
        for a in algos:
            rec[a] = run(R, a, delta, acc)
        del delta, acc
        out.append(rec)
        print(f"{name}: {time.time() - t0:.1f} s "
              + " ".join(f"{a}={rec[a]['iterations']}/{rec[a]['num_blocks']}" for a in algos),
              flush=True)
    with open(PATH, "w") as f:
        json.dump({"generator": "tests/golden/make_config_golden.py",
                   "reference": "oracle/_ref (unmodified dfamin headers)",
                   "threads": R.worker_count(), "vectors": out}, f, indent=1)
    print(f"wrote {PATH}: {len(out)} vectors")


if __name__ == "__main__":
    main()
