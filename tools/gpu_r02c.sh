set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bench tools/l2_bench.cu && /tmp/l2_bench > $OUT/l2_bench.txt 2>&1
cat $OUT/l2_bench.txt
for D in 0 1; do
DFM_SORTPR_DIRECT=$D python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_direct$D.json 2>&1
python - $OUT/bench_direct$D.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
PY
done
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py $OUT/launches_default.csv 2>/dev/null | tail -40
