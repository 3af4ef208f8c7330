set -u
OUT=gpurun_out/r02k; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_sharded_driver.py tests/test_gpu_sharded.py tests/test_cpp_shim.py -q -p no:cacheprovider -x --durations=8 > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -12 $OUT/tests.txt
for B in 0 1; do
DFM_SHARD_BLOCKED=$B timeout 900 python bench.py --sharded --n 100000000 --steps 5 --warmup 2 --no-e2e > $OUT/sharded_1e8_b$B.json 2> $OUT/sharded_1e8_b$B.err
python - $OUT/sharded_1e8_b$B.json <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d["ms_per_step"], d.get("single_gpu_engine"), {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[1]).read()[-500:])
PY
done
tail -3 $OUT/sharded_1e8_b1.err
