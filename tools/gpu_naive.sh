#!/bin/bash
# naivePR parity + C1/C2 naive bench lines (A/B over DFM_NAIVE_QUEUE), host-register probe
set -u
OUT=gpurun_out/${1:-naive}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -p no:cacheprovider -x -k "naive or c2 or c1" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -3 $OUT/tests.txt
for q in ${QS:-1 0}; do
  DFM_NAIVE_QUEUE=$q timeout 600 python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c2_naive_q$q.json 2>&1
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['config'].get('passes'), d['config'].get('blocks'))" $OUT/c2_naive_q$q.json
done
timeout 300 python tools/host_register_probe.py > $OUT/host_register.txt 2>&1; cat $OUT/host_register.txt
if [ -n "${MORE:-}" ]; then
  timeout 600 python bench.py --algo naive --n 100000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c1_naive.json 2>&1
  timeout 600 python bench.py --algo transpr --family comb --n 1000000 --k 2 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c3_comb.json 2>&1
  timeout 600 python bench.py --algo transpr --family chain --n 10000000 --k 1 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/c3_chain.json 2>&1
  for f in c1_naive c3_comb c3_chain; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], d['ms_per_step'], d['config'].get('passes'), d['config'].get('blocks'))" $OUT/$f.json; done
fi
