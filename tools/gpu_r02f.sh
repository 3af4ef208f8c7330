set -u
OUT=gpurun_out/r02f; mkdir -p $OUT
for F in 0 1; do
DFM_SORTPR_FILT_FUSED=$F python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_f$F.json 2>&1
python - $OUT/bench_f$F.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
PY
done
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_default.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
