# one ncu --set full capture of the kernels matching $2 in a 1-step bench (extra bench args in $3)
# bash tools/ncu_one.sh <tag> <kernel-regex> "<bench args>" [count]
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c ${4:-3} -o $OUT/prof python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline $3 > $OUT/ncu.log 2>&1
ncu -i $OUT/prof.ncu-rep --page details --csv > $OUT/details.csv
ncu -i $OUT/prof.ncu-rep --page source --csv > $OUT/source.csv 2>/dev/null
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source cuda > $OUT/source_cuda.csv 2>/dev/null
rm -f $OUT/prof.ncu-rep
