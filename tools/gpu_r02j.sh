set -u
OUT=gpurun_out/r02j; mkdir -p $OUT
for O in 0 1; do
DFM_NAIVE_OWN_LABEL=$O python bench.py --algo naive --n 100000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c1_naive_own$O.json 2>&1
DFM_NAIVE_OWN_LABEL=$O python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c2_naive_own$O.json 2>&1
DFM_NAIVE_OWN_LABEL=$O python bench.py --algo transpr --family comb --n 1000000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c3_comb_own$O.json 2>&1
done
for f in $OUT/*.json; do python - $f <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d["ms_per_step"],3), d["config"]["passes"])
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[1]).read()[-300:])
PY
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "naive or golden or c1 or transpr or comb or chain or fib" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
