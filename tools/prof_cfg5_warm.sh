# Warm per-launch times of the N = 2^28 pass groups (ncu --cache-control none:
# the twiddle tables stay cached as in a real run), plus --set full of the
# last group.  usage: bash tools/prof_cfg5_warm.sh TAG [ENV=V ...]
TAG=$1; shift
C="python bench.py --config cfg5_n2p28_f32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
env "$@" $C > gpurun_out/warm_${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/warm_${TAG}_plain.log; exit 1; }
env "$@" ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
   -k regex:sfft -s 16 -c 8 --csv $C > gpurun_out/warm_${TAG}_launches.csv 2> gpurun_out/warm_${TAG}_launches.err
env "$@" ncu --set full --import-source on --cache-control none --clock-control none -k regex:sfft -s 19 -c 1 -o gpurun_out/warm_${TAG}_g3 $C > gpurun_out/warm_${TAG}_g3.log 2>&1
python - "$TAG" <<'PY'
import csv, sys
tag = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/warm_{tag}_launches.csv")) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
for r in rows[1:]:
    print(tag, r[0], r[ki][:60], r[mi], r[vi])
PY
