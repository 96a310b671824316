# r02k: bulk-store output variant of the warp kernel (A/B + its parity)
set -u
VARIANTS="obs|SFFT_TMAW=f64:10:7,3,1,1|" CONFIGS=cfg3_n1024_f64 ALGOS="dit dif" REPS=3 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02k_ab.txt 2>&1
cat gpurun_out/r02k_ab.txt
(cd /tmp/ab_obs && timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or (tma_kernel_many_tiles and f64) or (f64_bitwise and 10)") > gpurun_out/r02k_obs_tests.txt 2>&1
tail -2 gpurun_out/r02k_obs_tests.txt
