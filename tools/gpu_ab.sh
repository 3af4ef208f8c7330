# A/B of env switches on the north-star bench: bash tools/gpu_ab.sh <tag> "ENV=1 ENV2=x" ...
# (the empty string is the default); per variant the ms/step of a 10-step bench and
# the ncu launch list of one step.
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
i=0
for v in "$@"; do
  i=$((i+1))
  env $v python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > $OUT/bench_$i.json 2>&1
  python - "$v" $OUT/bench_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); print(f"[{sys.argv[1]}]", round(d["ms_per_step"],3), {k:round(v["ms_per_step"],3) for k,v in d["roofline"]["families"].items()})
PY
  [ -n "${NO_NCU:-}" ] || env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$i.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1
done
