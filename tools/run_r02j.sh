# r02j: TMEM-factor warp kernel + X2 exchange default: parity, A/B, ncu of the new DIT kernel
set -u
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r02j_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02j_tests.txt
tail -3 gpurun_out/r02j_tests.txt
VARIANTS="regf|SFFT_TMAW=f64:10:7,3,0|;;old|SFFT_AUTO_OVERRIDE=f64:10:tma,3|;;tm6|SFFT_TMAW=f64:10:6,3,1|" CONFIGS=cfg3_n1024_f64 ALGOS="dit dif" REPS=2 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02j_ab.txt 2>&1
cat gpurun_out/r02j_ab.txt
B="python bench.py --config cfg3_n1024_f64 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_r02j_dit.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tmaw -s 2 -c 1 -o gpurun_out/prof_r02j_tmaw_dit $B > gpurun_out/ncu_r02j_dit.log 2>&1
echo done
