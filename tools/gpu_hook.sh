#!/bin/bash
# C++ shim / out-ready hook tests + default bench (e2e incl. the C++ reference-types line)
set -u
OUT=gpurun_out/${1:-hook}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_cpp_shim.py tests/test_e2e_ref_tool.py tests/test_gpu_pipeline.py tests/test_cabi.py -q -p no:cacheprovider -x > $OUT/tests.txt 2>&1; echo "rc=$?" >> $OUT/tests.txt; tail -n 2 $OUT/tests.txt
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['e2e']; print('step', d['ms_per_step'], 'e2e', e['ms_per_step'], 'pinned', e['pinned']['ms_per_step'], 'cpp', e.get('cpp_reference_types',{}).get('ms_min'))" $OUT/bench_default.json
