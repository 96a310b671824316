# Warm per-launch kernel times (ncu --cache-control none) for one bench config.
# usage: bash tools/prof_launches_warm.sh TAG CONFIG SKIP COUNT [ENV=V ...]
TAG=$1; CFG=$2; SKIP=$3; CNT=$4; shift 4
C="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
env "$@" $C > gpurun_out/lw_${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/lw_${TAG}_plain.log; exit 1; }
python -c "import json;d=json.loads(open('gpurun_out/lw_${TAG}_plain.log').read().strip().splitlines()[-1]);print('$TAG', d['ms_per_step'], d['roofline']['frac'])"
env "$@" ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active \
   -k regex:sfft -s $SKIP -c $CNT --csv $C 2>/dev/null | python -c "
import csv, sys
rows = [r for r in csv.reader(sys.stdin) if len(r) > 12]
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r)); print('$TAG', d['ID'], d['Kernel Name'][:60], d['Metric Name'], d['Metric Value'])
"
