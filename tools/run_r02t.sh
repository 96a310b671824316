# r02t: fp32 N=4096 signal-group kernel (2 warps per signal, radix 64, slot ring): parity + A/B
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tma_kernel_many_tiles or warp_kernel or auto_batch or every_radix" > gpurun_out/r02t_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02t_tests.txt
tail -3 gpurun_out/r02t_tests.txt
VARIANTS="g64|SFFT_AUTO_OVERRIDE=f32:12:tma,6|;;g64x3|SFFT_AUTO_OVERRIDE=f32:12:tma,6 SFFT_TMAW=f32:12:8,0,0,1,3,2|" CONFIGS="cfg4_n4096_f32" ALGOS="dit dif" REPS=3 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02t_ab.txt 2>&1
cat gpurun_out/r02t_ab.txt
B="python bench.py --config cfg4_n4096_f32 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
(cd /tmp/ab_g64 && $B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tmaw -s 2 -c 1 -o $GRAFT_REPO_ROOT/gpurun_out/prof_r02t_cfg4_g64 $B > $GRAFT_REPO_ROOT/gpurun_out/ncu_r02t.log 2>&1)
echo done
