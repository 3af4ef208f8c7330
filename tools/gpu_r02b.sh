set -u
OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sharded_driver.py tests/test_cpp_shim.py tests/test_gpu_sharded.py -q -p no:cacheprovider -x --durations=10 > $OUT/tests_sharded.txt 2>&1; echo "rc=$?" >> $OUT/tests_sharded.txt
tail -15 $OUT/tests_sharded.txt
timeout 600 python bench.py --sharded --n 100000000 --steps 5 --warmup 2 --e2e-steps 2 > $OUT/bench_sharded_1e8.json 2> $OUT/bench_sharded_1e8.err; tail -c 2500 $OUT/bench_sharded_1e8.json; tail -5 $OUT/bench_sharded_1e8.err
