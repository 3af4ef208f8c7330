set -u
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_trans_tc.py tests/test_gpu_configs.py -k "trans or c4" tests/test_gpu_parity.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
for P in 0 1; do
DFM_TRANS_PERSIST=$P python bench.py --algo trans --family random --n 256 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c4_rand256_p$P.json 2>&1
DFM_TRANS_PERSIST=$P python bench.py --algo trans --family fib --n 12 --k 1 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c4_fib12_p$P.json 2>&1
done
for f in $OUT/*.json; do python - $f <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d["roofline"]; print(sys.argv[1], round(d["ms_per_step"],3), d["config"]["passes"], r["families"].get("gemm"))
except Exception as e: print(sys.argv[1], "ERR", open(sys.argv[1]).read()[-500:])
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"square|dead_copy" --log-file $OUT/ncu_trans_rand256.csv python bench.py --algo trans --family random --n 256 --k 2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"square|dead_copy" --log-file $OUT/ncu_trans_fib12.csv python bench.py --algo trans --family fib --n 12 --k 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv,glob
for f in sorted(glob.glob("gpurun_out/r02e/ncu_*.csv")):
    lines=open(f).read().splitlines(); i=[j for j,l in enumerate(lines) if l.startswith('"ID"')]
    if not i: print(f,"no data"); continue
    rows=list(csv.DictReader(lines[i[0]:])); agg={}
    for r in rows:
        k=(r["ID"], r["Kernel Name"][:40]); agg.setdefault(k,{})[r["Metric Name"]]=r["Metric Value"]
    print(f)
    for k,v in list(agg.items())[:40]: print(k, v)
PY
