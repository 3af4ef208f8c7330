#!/bin/bash
# One GPU session: parity tests, bench lines for every §8 config (with same-run CPU
# baselines), the reference arm, the sharded C5 line, ncu launch list + DRAM traffic,
# compute-sanitizer.  Usage (on the GPU box via gpurun):
#   bash tools/gpu_suite.sh <tag> [tests bench ref c5 ncu sanitize]
set -u
TAG=${1:-r02}; shift || true
WHAT=${*:-"tests bench ref c5 ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv; nproc; free -g;
  lscpu | grep "Model name"; } > $OUT/gpu.txt 2>&1
summ() {
  for f in "$@"; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = d.get("roofline") or {}
    c = d.get("cpu_baseline") or {}
    e = d.get("e2e") or {}
    print(f.split("/")[-1], "ms/step=%.3f" % d["ms_per_step"], "value=%.3e" % d["value"],
          "passes=%s" % d["config"].get("passes"), "blocks=%s" % d["config"].get("blocks"),
          "frac=%.3f" % (r.get("frac") or 0), "e2e_ms=%s" % e.get("ms_per_step"),
          "cpu=%s" % c.get("value"))
except Exception as e:
    print(f, "ERR", e, open(f).read()[-400:])
PY
  done
}
if [[ " $WHAT " == *" tests "* ]]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $OUT/gpu_tests.txt 2>&1
  echo "tests rc=$?" >> $OUT/gpu_tests.txt; tail -4 $OUT/gpu_tests.txt
fi
if [[ " $WHAT " == *" bench "* ]]; then
  timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
  B="--no-e2e"
  timeout 600 python bench.py --sortpr-engine radix $B --no-cpu-baseline > $OUT/bench_radix.json 2>&1
  timeout 900 python bench.py --algo sort --n 100000 --k 2 --steps 10 --warmup 3 $B > $OUT/bench_c1_sort.json 2>&1
  timeout 900 python bench.py --algo naive --n 100000 --k 2 --steps 5 --warmup 2 $B > $OUT/bench_c1_naive.json 2>&1
  timeout 900 python bench.py --algo sort --family vlts --n 10000000 --k 100 --steps 5 --warmup 2 > $OUT/bench_c2_sort.json 2>&1
  timeout 900 python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 3 --warmup 1 $B > $OUT/bench_c2_naive.json 2>&1
  timeout 900 python bench.py --algo transpr --family chain --n 10000000 --k 1 --steps 3 --warmup 1 $B > $OUT/bench_c3_chain.json 2>&1
  timeout 900 python bench.py --algo transpr --family comb --n 1000000 --k 2 --steps 3 --warmup 1 $B > $OUT/bench_c3_comb.json 2>&1
  timeout 900 python bench.py --algo trans --family fib --n 12 --k 1 --steps 3 --warmup 1 $B > $OUT/bench_c4_fib12.json 2>&1
  timeout 900 python bench.py --algo trans --family random --n 256 --k 2 --steps 3 --warmup 1 $B > $OUT/bench_c4_rand256.json 2>&1
  summ $OUT/bench_*.json
fi
if [[ " $WHAT " == *" ref "* ]]; then
  timeout 1200 python bench.py --impl reference --steps 8 --warmup 1 > $OUT/reference_default.json 2>&1
  tail -c 1500 $OUT/reference_default.json
fi
if [[ " $WHAT " == *" c5 "* ]]; then
  timeout 1200 python bench.py --sharded --n 1000000000 --steps 3 --warmup 1 --e2e-steps 1 > $OUT/bench_c5_sharded_n1.json 2> $OUT/bench_c5_sharded_n1.err
  timeout 1200 python bench.py --sharded --n 100000000 --steps 5 --warmup 2 --e2e-steps 2 > $OUT/bench_sharded_1e8_n1.json 2> $OUT/bench_sharded_1e8_n1.err
  summ $OUT/bench_c5_sharded_n1.json $OUT/bench_sharded_1e8_n1.json
fi
if [[ " $WHAT " == *" ncu "* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $OUT/launches_default.csv \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
  python tools/ncu_step_traffic.py $OUT/launches_default.csv $OUT/ncu_traffic.json > /dev/null
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lay_sig_kernel" -s 1 -c 1 \
      -o $OUT/prof_laysig python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"square_persistent" -c 3 \
      -o $OUT/prof_trans python bench.py --algo trans --family fib --n 12 --k 1 --steps 1 --warmup 0 --no-e2e > $OUT/ncu_trans.log 2>&1
  for r in laysig trans; do
    if [ -f $OUT/prof_$r.ncu-rep ]; then
      ncu -i $OUT/prof_$r.ncu-rep --page raw --csv > $OUT/prof_${r}_raw.csv 2>/dev/null
      rm -f $OUT/prof_$r.ncu-rep
    fi
  done
fi
if [[ " $WHAT " == *" sanitize "* ]]; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > $OUT/sanitize_memcheck.txt 2>&1
  echo "rc=$?" >> $OUT/sanitize_memcheck.txt
  timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py --small > $OUT/sanitize_racecheck.txt 2>&1
  echo "rc=$?" >> $OUT/sanitize_racecheck.txt
  tail -3 $OUT/sanitize_memcheck.txt $OUT/sanitize_racecheck.txt
fi
ls $OUT
