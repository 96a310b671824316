# Round-end measurement pass: bench lines for every config + the reference
# arm, the launch list of the default bench command, and one ncu --set full
# capture of the top kernel per config (cfg5: its 4 pass launches).
# usage: bash tools/round_profiles.sh TAG
set -u
TAG=$1
bash tools/bench_all.sh $TAG
python bench.py --steps 3 --warmup 3 > gpurun_out/default_${TAG}.json 2> gpurun_out/default_${TAG}.err || echo "default bench failed"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launches_${TAG}.log 2>&1 || echo "launch list failed"
bash tools/prof_cfgs.sh $TAG cfg2_n64_f32 cfg3_n1024_f32 cfg3_n1024_f64 cfg4_n4096_f32
C5="python bench.py --config cfg5_n2p28_f32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C5 > gpurun_out/plain_${TAG}_cfg5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sfft -s 4 -c 4 -o gpurun_out/prof_${TAG}_cfg5_n2p28_f32 $C5 \
    > gpurun_out/ncu_${TAG}_cfg5.log 2>&1
echo done
