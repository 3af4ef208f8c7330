#!/bin/bash
# ncu --set full of C1 naive's thread-per-state fused kernel (one launch of 1024 passes)
set -u
OUT=gpurun_out/${1:-c1_ncu}; mkdir -p $OUT
B="python bench.py --algo naive --n 100000 --k 2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_pr_kernel" -s 6 -c 1 -o $OUT/prof_c1 $B > $OUT/ncu_c1.log 2>&1
if [ -f $OUT/prof_c1.ncu-rep ]; then
  ncu -i $OUT/prof_c1.ncu-rep --page raw --csv > $OUT/prof_c1_raw.csv 2>/dev/null
  ncu -i $OUT/prof_c1.ncu-rep --page details > $OUT/prof_c1_details.txt 2>/dev/null
  ncu -i $OUT/prof_c1.ncu-rep --page source --csv > $OUT/prof_c1_source.csv 2>/dev/null
  rm -f $OUT/prof_c1.ncu-rep
fi
ls $OUT
