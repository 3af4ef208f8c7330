set -u
OUT=gpurun_out/${1:-r02q}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_sharded_driver.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.json 2>&1
python - $OUT/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("default", d["ms_per_step"], {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1; python tools/launches.py $OUT/launches.csv | grep -E "lay_|total"
