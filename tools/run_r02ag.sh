# r02ag: pass kernels with 64-column tiles (256-byte runs, -DSFFT_PASS_TJ64, build/variants/tj64.so) vs the shipped 32-column tiles
set -u
OUT=gpurun_out/r02ag_sweep.jsonl
: > $OUT
for rep in 1 2 3; do
for A in dit dif; do
  P2_KERNEL=pass timeout 300 python tools/p2_sweep.py 28 f32 $A >> $OUT
  SFFT_B200_LIB=build/variants/tj64.so P2_KERNEL=pass timeout 300 python tools/p2_sweep.py 28 f32 $A >> $OUT
done
done
for M in 20 24 26; do
  P2_KERNEL=pass timeout 300 python tools/p2_sweep.py $M f32 dit >> $OUT
  SFFT_B200_LIB=build/variants/tj64.so P2_KERNEL=pass timeout 300 python tools/p2_sweep.py $M f32 dit >> $OUT
done
cat $OUT
SFFT_B200_LIB=build/variants/tj64.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -k "f32 or float32 or pass or large or dist" > gpurun_out/r02ag_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ag_tests.txt
tail -3 gpurun_out/r02ag_tests.txt
SFFT_B200_LIB=build/variants/tj64.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config5 and not fp64" > gpurun_out/r02ag_tests_full.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ag_tests_full.txt
tail -3 gpurun_out/r02ag_tests_full.txt
SFFT_B200_LIB=build/variants/tj64.so P2_KERNEL=pass timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfft_pass -c 4 -o gpurun_out/prof_r02ag_tj64 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02ag.log 2>&1
echo done
