set -u
OUT=gpurun_out/r02a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; free -g >> $OUT/gpu.txt; lscpu | grep "Model name" >> $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 -x > $OUT/gpu_tests.txt 2>&1; echo "tests rc=$?" >> $OUT/gpu_tests.txt
tail -5 $OUT/gpu_tests.txt
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; tail -c 3000 $OUT/bench_default.json
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > $OUT/sanitize_memcheck.txt 2>&1; echo "rc=$?" >> $OUT/sanitize_memcheck.txt
tail -5 $OUT/sanitize_memcheck.txt
