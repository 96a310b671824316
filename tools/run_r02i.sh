# r02i: ncu of the warp kernel (DIT vs DIF), pair probe, 3-group cfg5 splits, cfg4 X2 A/B
set -u
B="python bench.py --config cfg3_n1024_f64 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
for A in dit dif; do
  $B --algorithm $A > gpurun_out/plain_r02i_$A.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:tmaw -s 2 -c 1 -o gpurun_out/prof_r02i_tmaw_$A $B --algorithm $A > gpurun_out/ncu_r02i_$A.log 2>&1
done
timeout 300 ./build/tools/pattern_probe_pairs > gpurun_out/r02i_pairs.txt 2>&1
C5="python bench.py --config cfg5_n2p28_f32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
for S in default 10,9,9 9,10,9 9,9,10; do
  for A in dit dif; do
    if [ $S = default ]; then E=""; else E="SFFT_PASS_SPLIT=$S"; fi
    env $E $C5 --algorithm $A 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$S', '$A', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'))" >> gpurun_out/r02i_cfg5_splits.txt 2>&1
  done
done
VARIANTS="x2||-DSFFT_FUSED_X2" CONFIGS="cfg4_n4096_f32 cfg3_n1024_f32" ALGOS="dit dif" REPS=2 timeout 1200 bash tools/ab_build.sh > gpurun_out/r02i_ab_x2.txt 2>&1
cat gpurun_out/r02i_pairs.txt gpurun_out/r02i_cfg5_splits.txt gpurun_out/r02i_ab_x2.txt
