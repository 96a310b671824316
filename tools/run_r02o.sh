# r02o: cfg4 occupancy A/B (min 5 CTAs/SM for the 256-thread fused kernels), batch-switch test
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "auto_batch_switch or warp_kernel" > gpurun_out/r02o_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02o_tests.txt
tail -2 gpurun_out/r02o_tests.txt
VARIANTS="minb5||-DSFFT_FUSED_MINB=5" CONFIGS="cfg4_n4096_f32" ALGOS="dit dif" REPS=3 timeout 1200 bash tools/ab_build.sh > gpurun_out/r02o_ab.txt 2>&1
cat gpurun_out/r02o_ab.txt
grep -A2 "Li12ELi4ELb0ELb0ELb0" /tmp/ab_minb5.log | head -3
