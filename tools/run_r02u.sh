# r02u: fp32 N=4096 signal-group kernel with second-pass factors in TMEM: parity + A/B
set -u
VARIANTS="g64|SFFT_AUTO_OVERRIDE=f32:12:tma,6|;;g64tm|SFFT_AUTO_OVERRIDE=f32:12:tma,6 SFFT_TMAW=f32:12:8,0,1,1,2,2|" CONFIGS="cfg4_n4096_f32" ALGOS="dit dif" REPS=3 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02u_ab.txt 2>&1
cat gpurun_out/r02u_ab.txt
(cd /tmp/ab_g64tm && timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tma_kernel_many_tiles and f32 and 12") > gpurun_out/r02u_tests.txt 2>&1
tail -1 gpurun_out/r02u_tests.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or (tma_kernel_many_tiles and 10) or auto_batch" >> gpurun_out/r02u_tests.txt 2>&1
tail -1 gpurun_out/r02u_tests.txt
B="python bench.py --config cfg4_n4096_f32 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
(cd /tmp/ab_g64tm && $B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tmaw -s 2 -c 1 -o $GRAFT_REPO_ROOT/gpurun_out/prof_r02u_cfg4_g64tm $B > $GRAFT_REPO_ROOT/gpurun_out/ncu_r02u.log 2>&1)
python tools/pcie_probe.py > gpurun_out/r02u_pcie.txt 2>&1
echo done
