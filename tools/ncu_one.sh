OUT=gpurun_out/r02r; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lay_sig_kernel|lay_scatter" -c 3 -o $OUT/laysig python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
ncu -i $OUT/laysig.ncu-rep --page details --csv > $OUT/laysig_details.csv
ncu -i $OUT/laysig.ncu-rep --page source --csv > $OUT/laysig_source.csv 2>/dev/null
rm -f $OUT/laysig.ncu-rep
