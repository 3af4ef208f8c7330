#!/bin/bash
# One GPU session: parity tests, bench lines for every §8 row, launch list + ncu captures.
# Usage (on the GPU box via gpurun): bash tools/gpu_suite.sh <tag> [tests|bench|ncu ...]
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-"tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
if [[ " $WHAT " == *" tests "* ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/gpu_tests.txt 2>&1
  echo "tests rc=$?" >> $OUT/gpu_tests.txt; tail -4 $OUT/gpu_tests.txt
fi
if [[ " $WHAT " == *" bench "* ]]; then
  python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 600 $OUT/bench_default.json
  python bench.py --sortpr-engine radix --no-e2e --no-cpu-baseline > $OUT/bench_radix.json 2>&1
  python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2>&1
  python bench.py --algo naive --n 100000 --k 2 --steps 5 --warmup 2 --no-e2e > $OUT/bench_c1_naive.json 2>&1
  python bench.py --algo sort --n 100000 --k 2 --steps 10 --warmup 3 --no-e2e > $OUT/bench_c1_sort.json 2>&1
  python bench.py --algo sort --family vlts --n 10000000 --k 100 --steps 5 --warmup 2 --no-e2e > $OUT/bench_c2_sort.json 2>&1
  python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 3 --warmup 1 --no-e2e > $OUT/bench_c2_naive.json 2>&1
  python bench.py --algo transpr --family chain --n 10000000 --k 1 --steps 3 --warmup 1 --no-e2e > $OUT/bench_c3_chain.json 2>&1
  python bench.py --algo transpr --family comb --n 1000000 --k 2 --steps 3 --warmup 1 --no-e2e > $OUT/bench_c3_comb.json 2>&1
  python bench.py --algo trans --family fib --n 12 --k 1 --steps 3 --warmup 1 --no-e2e > $OUT/bench_c4_fib12.json 2>&1
  python bench.py --algo trans --family random --n 256 --k 2 --steps 3 --warmup 1 --no-e2e > $OUT/bench_c4_rand256.json 2>&1
  for f in $OUT/bench_*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    print(f.split("/")[-1], "ms/step=%.3f" % d["ms_per_step"], "value=%.3e" % d["value"],
          "passes=%s" % d["config"].get("passes"), "blocks=%s" % d["config"].get("blocks"),
          "dominant=%s frac=%.3f" % (r.get("kernel"), r.get("frac") or 0))
except Exception as e:
    print(f, "ERR", e, open(f).read()[-400:])
PY
  done
fi
if [[ " $WHAT " == *" ncu "* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_default.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -c 60 \
      -o $OUT/prof_default python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"square_kernel" -c 2 \
      -o $OUT/prof_trans python bench.py --algo trans --family fib --n 12 --k 1 --steps 1 --warmup 0 --no-e2e > $OUT/ncu_trans.log 2>&1
  # the reports themselves can exceed gpurun's 64 MiB copy-back: keep their raw pages
  for r in default trans; do
    if [ -f $OUT/prof_$r.ncu-rep ]; then
      ncu -i $OUT/prof_$r.ncu-rep --page raw --csv > $OUT/prof_${r}_raw.csv 2>/dev/null
      rm -f $OUT/prof_$r.ncu-rep
    fi
  done
  ls -la $OUT
fi
