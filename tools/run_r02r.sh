# r02r: pass kernels with (re, im) pair exchanges: parity (pass variants, large-m fp64 pins,
# sharded emulation, config 5 full size vs the oracle) + A/B on config 5 vs the planar exchange
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pass_kernel or large_m or f64_bitwise or f32_rel or warp_kernel_small" > gpurun_out/r02r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02r_tests.txt
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q >> gpurun_out/r02r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02r_tests.txt
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config5" >> gpurun_out/r02r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02r_tests.txt
grep -E "passed|failed|rc=" gpurun_out/r02r_tests.txt
VARIANTS="planar||-DSFFT_PASS_PLANAR_X" CONFIGS="cfg5_n2p28_f32" ALGOS="dit dif" REPS=3 STEPS=20 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02r_ab.txt 2>&1
cat gpurun_out/r02r_ab.txt
