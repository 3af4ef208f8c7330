set -u
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sharded_driver.py tests/test_gpu_sharded.py tests/test_cpp_shim.py tests/test_gpu_post.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -x -k "radix or golden or config or oracle_agreement or full_size" > $OUT/tests_radix.txt 2>&1; echo "rc=$?" >> $OUT/tests_radix.txt; tail -3 $OUT/tests_radix.txt
python bench.py --sortpr-engine radix --no-e2e --no-cpu-baseline > $OUT/bench_radix.json 2>&1
python - $OUT/bench_radix.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print("radix", d["ms_per_step"], {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
PY
timeout 1500 python bench.py --sharded --n 1000000000 --steps 3 --warmup 1 --e2e-steps 1 > $OUT/bench_c5_sharded_n1.json 2> $OUT/bench_c5_sharded_n1.err
timeout 900 python bench.py --sharded --n 100000000 --steps 5 --warmup 2 --e2e-steps 2 > $OUT/bench_sharded_1e8_n1.json 2> $OUT/bench_sharded_1e8_n1.err
for f in $OUT/bench_c5_sharded_n1.json $OUT/bench_sharded_1e8_n1.json; do python - $f <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d["ms_per_step"], d.get("single_gpu_engine"), {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()}, (d.get("e2e") or {}).get("ms_per_step"))
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[1]).read()[-300:])
PY
done
tail -3 $OUT/bench_c5_sharded_n1.err
timeout 900 python tools/e2e_stage.py > $OUT/e2e_stage.txt 2>&1; cat $OUT/e2e_stage.txt | tail -2
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py --small > $OUT/sanitize_racecheck.txt 2>&1; echo "rc=$?" >> $OUT/sanitize_racecheck.txt; tail -n 4 $OUT/sanitize_racecheck.txt
