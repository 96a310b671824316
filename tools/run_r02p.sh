# r02p: shared slot ring for the fp64 N=1024 warp kernel (9/10/12 warps per SM) -- parity + A/B
set -u
VARIANTS="ring9|SFFT_TMAW=f64:10:9,3,1,1|;;ring10|SFFT_TMAW=f64:10:10,3,1,1|;;ring12|SFFT_TMAW=f64:10:12,3,1,1|" CONFIGS=cfg3_n1024_f64 ALGOS="dit dif" REPS=2 timeout 1800 bash tools/ab_build.sh > gpurun_out/r02p_ab.txt 2>&1
cat gpurun_out/r02p_ab.txt
for v in ring9 ring12; do
  (cd /tmp/ab_$v && timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or (tma_kernel_many_tiles and f64 and 10) or auto_batch_switch or (f64_bitwise and 10)") > gpurun_out/r02p_tests_$v.txt 2>&1
  tail -1 gpurun_out/r02p_tests_$v.txt
done
