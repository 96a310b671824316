# r02h: warp-per-signal fp64 N=1024 kernel: parity + A/B vs the radix-8 TMA kernel
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or tma_kernel_many_tiles or f64_bitwise or strided or graph or known" > gpurun_out/r02h_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02h_tests.txt
tail -3 gpurun_out/r02h_tests.txt
VARIANTS="old|SFFT_AUTO_OVERRIDE=f64:10:tma,3|;;hk0|SFFT_TMAW=f64:10:7,0|;;hk4|SFFT_TMAW=f64:10:7,4|;;w6|SFFT_TMAW=f64:10:6,3|" CONFIGS=cfg3_n1024_f64 ALGOS="dit dif" REPS=2 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02h_ab.txt 2>&1
cat gpurun_out/r02h_ab.txt
