# r02bb: re-capture after the layout-header change (new kernel-source hash): TMA parity subset, default + cfg2 bench lines, launch list, ncu --set full per config
set -u
T=r02bb
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -x -q -k "tma or known or f32_rel or edges or empty or ragged" > gpurun_out/${T}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.txt
tail -2 gpurun_out/${T}_tests.txt
python bench.py > gpurun_out/${T}_default.json 2> gpurun_out/${T}_default.err
timeout 300 python bench.py --config cfg2_n64_f32 --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_${T}_cfg2_n64_f32.json 2> gpurun_out/bench_${T}_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${T}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_${T}.log 2>&1 || echo "launch list failed"
bash tools/prof_cfgs.sh $T cfg3_n1024_f64 cfg2_n64_f32 cfg3_n1024_f32 cfg4_n4096_f32
C5="python bench.py --config cfg5_n2p28_f32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C5 > gpurun_out/plain_${T}_cfg5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sfft -s 4 -c 4 -o gpurun_out/prof_${T}_cfg5_n2p28_f32 $C5 > gpurun_out/ncu_${T}_cfg5.log 2>&1
echo done
