set -u
OUT=gpurun_out/r02m; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_sharded_driver.py tests/test_gpu_sharded.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
timeout 900 python bench.py --sharded --n 100000000 --steps 5 --warmup 2 --no-e2e > $OUT/sharded_1e8.json 2> $OUT/sharded_1e8.err
timeout 1500 python bench.py --sharded --n 1000000000 --steps 3 --warmup 1 --no-e2e > $OUT/sharded_1e9.json 2> $OUT/sharded_1e9.err
for f in $OUT/sharded_1e8.json $OUT/sharded_1e9.json; do python - $f <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d["ms_per_step"], d.get("single_gpu_engine"), {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[1]).read()[-500:])
PY
done
DFM_SHARD_PROTOCOL=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/shard_launches.csv python bench.py --sharded --n 100000000 --steps 1 --warmup 0 --no-e2e > /dev/null 2>&1; python tools/launches.py $OUT/shard_launches.csv | sed -n 2,33p
