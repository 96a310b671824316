# Warm per-launch kernel times (ncu --cache-control none) for one bench config.
# usage: bash tools/prof_launches_warm.sh TAG CONFIG SKIP COUNT [bench args...]
TAG=$1; CFG=$2; SKIP=$3; CNT=$4; shift 4
C="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $*"
$C > gpurun_out/lw_${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/lw_${TAG}_plain.log; exit 1; }
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed \
   -k regex:sfft -s $SKIP -c $CNT --csv $C 2>/dev/null | python tools/ncu_csv.py $TAG
