#!/bin/bash
# ncu --set full of the masked naivePR pass kernels on C2 (vlts(1000, 1e6, 20)):
# the grid-stride fused_pr_kernel<kMask> and queue_pr_kernel (one launch = 128 passes)
set -u
OUT=gpurun_out/${1:-naive_ncu}; mkdir -p $OUT
B="python bench.py --algo naive --family vlts --n 1000000 --k 20 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
DFM_NAIVE_QUEUE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_pr_kernel" -s 3 -c 1 -o $OUT/prof_fused $B > $OUT/ncu_fused.log 2>&1
DFM_NAIVE_QUEUE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"queue_pr_kernel" -c 1 -o $OUT/prof_queue $B > $OUT/ncu_queue.log 2>&1
for r in fused queue; do
  if [ -f $OUT/prof_$r.ncu-rep ]; then
    ncu -i $OUT/prof_$r.ncu-rep --page raw --csv > $OUT/prof_${r}_raw.csv 2>/dev/null
    ncu -i $OUT/prof_$r.ncu-rep --page details > $OUT/prof_${r}_details.txt 2>/dev/null
    ncu -i $OUT/prof_$r.ncu-rep --page source --csv > $OUT/prof_${r}_source.csv 2>/dev/null
    rm -f $OUT/prof_$r.ncu-rep
  fi
done
ls -la $OUT; tail -3 $OUT/ncu_*.log
