# r02m: in-place TMA kernel for N=4096 fp32 (parity + A/B vs the LDG kernel)
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tma_kernel_many_tiles and f32 and 12" > gpurun_out/r02m_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02m_tests.txt
tail -2 gpurun_out/r02m_tests.txt
VARIANTS="xip|SFFT_AUTO_OVERRIDE=f32:12:tma,4|" CONFIGS=cfg4_n4096_f32 ALGOS="dit dif" REPS=3 timeout 1200 bash tools/ab_build.sh > gpurun_out/r02m_ab.txt 2>&1
cat gpurun_out/r02m_ab.txt
B="python bench.py --config cfg4_n4096_f32 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
(cd /tmp/ab_xip && $B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sfft -s 2 -c 1 -o $GRAFT_REPO_ROOT/gpurun_out/prof_r02m_cfg4_xip $B > $GRAFT_REPO_ROOT/gpurun_out/ncu_r02m.log 2>&1)
echo done
