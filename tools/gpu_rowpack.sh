#!/bin/bash
# packed signature rows: parity (incl. C2 config records) + C2 sort A/B
set -u
OUT=gpurun_out/${1:-rowpack}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -x -k "packed or c2_ or c1_ or golden or collision or vlts or random" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -n 2 $OUT/tests.txt
for v in 1; do
  DFM_SORTPR_ROW_PACK=$v timeout 900 python bench.py --algo sort --family vlts --n 10000000 --k 100 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/c2_sort_$v.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step'],3), d['config']['passes'], d['config']['blocks'], {k:round(v['ms_per_step'],3) for k,v in d['roofline']['families'].items()})" $OUT/c2_sort_$v.json
done
