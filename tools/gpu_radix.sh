# radix engine: parity subset + bench + per-kernel launch times: bash tools/gpu_radix.sh <tag>
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "radix or config or sort" > $OUT/tests.txt 2>&1; tail -2 $OUT/tests.txt
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --sortpr-engine radix > $OUT/radix.json 2>&1
python - $OUT/radix.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("radix", d["ms_per_step"], {k:round(v["ms_per_step"],2) for k,v in d["roofline"]["families"].items()})
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --sortpr-engine radix > /dev/null 2>&1
python tools/launches.py $OUT/launches.csv | grep -E "onesweep|total" | head -40
