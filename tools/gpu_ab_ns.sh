#!/bin/bash
# sortPR parity (configs incl. the 1e8 record) + north-star A/B over an env switch:
#   VAR=DFM_SORTPR_FILT_CKEYS bash tools/gpu_ab_ns.sh <tag>
set -u
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "sort or ns_ or c2_ or collision or golden" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -n 2 $OUT/tests.txt
for r in 1 2; do for v in 1 0; do
  env $VAR=$v timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ns_${v}_$r.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['roofline']['families'].items()})" $OUT/ns_${v}_$r.json
done; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
