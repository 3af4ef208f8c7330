#!/bin/bash
# dynamic-row/queue naive parity test + pageable staging A/B (pool size per process) + default bench e2e
set -u
OUT=gpurun_out/${1:-stage}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "dynamic_rows or work_efficient" > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -n 2 $OUT/tests.txt
for T in 8 12 16; do timeout 600 python tools/e2e_stage.py $T > $OUT/e2e_stage_T$T.txt 2>&1; tail -n 1 $OUT/e2e_stage_T$T.txt; done
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['e2e']; print('step', d['ms_per_step'], 'e2e', e['ms_per_step'], 'pinned', e['pinned']['ms_per_step'], 'cpp', e.get('cpp_reference_types',{}).get('ms_min'))" $OUT/bench_default.json
