# Round-end measurement pass (run under gpurun from the repo root):
#   bash tools/run_final.sh TAG
# 1. the full GPU test suite; 2. one bench line per BASELINE config + the
# reference arm; 3. the default bench line (the driver's command) and its
# ncu launch list; 4. one ncu --set full capture per fused config + config 5
# (kernel-source hash recorded for bench.py's roofline.traffic).
set -u
TAG=$1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
tail -3 gpurun_out/${TAG}_gpu_tests.txt
python bench.py > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err || echo "default bench failed"
bash tools/bench_all.sh $TAG
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_${TAG}.log 2>&1 || echo "launch list failed"
bash tools/prof_cfgs.sh $TAG cfg3_n1024_f64 cfg2_n64_f32 cfg3_n1024_f32 cfg4_n4096_f32
C5="python bench.py --config cfg5_n2p28_f32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C5 > gpurun_out/plain_${TAG}_cfg5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sfft -s 4 -c 4 -o gpurun_out/prof_${TAG}_cfg5_n2p28_f32 $C5 \
    > gpurun_out/ncu_${TAG}_cfg5.log 2>&1
echo done
