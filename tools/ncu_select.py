"""Select a few columns of an ncu raw-page CSV (tools/gpu_suite.sh keeps the raw
pages): kernel, grid/block, registers, time, DRAM bytes, throughputs, L2 hit rate,
tensor-pipe activity.  usage: python tools/ncu_select.py raw.csv out.csv"""
import csv
import sys

COLS = ["ID", "Kernel Name", "Block Size", "Grid Size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active"]

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
idx = [h.index(c) for c in COLS if c in h]
with open(sys.argv[2], "w", newline="") as f:
    w = csv.writer(f, quoting=csv.QUOTE_ALL)
    for r in rows:
        if len(r) == len(h):
            w.writerow([r[i] for i in idx])
