#!/bin/bash
# thread-per-state naivePR CTAs spread over all SMs: parity + C1 naive / C3 A/B
set -u
OUT=gpurun_out/${1:-spread}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -x -k "naive or c1_ or c3_ or trans_pr or transpr" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -n 2 $OUT/tests.txt
for v in 1 0; do
  DFM_NAIVE_SPREAD=$v timeout 600 python bench.py --algo naive --n 100000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c1_naive_$v.json 2>&1
  DFM_NAIVE_SPREAD=$v timeout 600 python bench.py --algo transpr --family comb --n 1000000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c3_comb_$v.json 2>&1
  DFM_NAIVE_SPREAD=$v timeout 600 python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c2_naive_$v.json 2>&1
  for f in c1_naive c3_comb c2_naive; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['ms_per_step'],3), d['config'].get('passes'), d['config'].get('blocks'))" $OUT/${f}_$v.json; done
done
