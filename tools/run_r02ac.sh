# r02ac: pass2 with the cp.async landing-buffer pipeline (3 CTAs/SM) vs the direct-load build (build/variants/p2_direct.so) and the per-group schedule
set -u
timeout 1200 python -m pytest tests/test_gpu_pass2.py -x -q > gpurun_out/r02ac_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ac_tests.txt
tail -3 gpurun_out/r02ac_tests.txt
OUT=gpurun_out/r02ac_sweep.jsonl
: > $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
for F in 0 1; do
 for DS in "4 8" "6 16" "8 16" "12 16"; do
  set -- $DS
  SFFT_PASS2=1 SFFT_P2_FLAGS=$F SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f32 dit >> $OUT
 done
done
SFFT_B200_LIB=build/variants/p2_direct.so SFFT_PASS2=1 SFFT_P2_FLAGS=2 SFFT_P2_LAG=6 SFFT_P2_SLOTS=16 python tools/p2_sweep.py 28 f32 dit >> $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
SFFT_PASS2=1 SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 python tools/p2_sweep.py 28 f32 dif >> $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dif >> $OUT
for DS in "4 8" "8 16"; do
  set -- $DS
  SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
  SFFT_B200_LIB=build/variants/p2_direct.so SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
done
P2_KERNEL=pass python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
for M in 20 22 24 26; do
  python tools/p2_sweep.py $M f64 dit 10 >> $OUT
  SFFT_B200_LIB=build/variants/p2_direct.so python tools/p2_sweep.py $M f64 dit 10 >> $OUT
  P2_KERNEL=pass python tools/p2_sweep.py $M f64 dit 10 >> $OUT
  SFFT_PASS2=1 python tools/p2_sweep.py $M f32 dit 10 >> $OUT
  P2_KERNEL=pass python tools/p2_sweep.py $M f32 dit 10 >> $OUT
done
cat $OUT
SFFT_PASS2=1 SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02ac_pass2 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02ac.log 2>&1
tail -1 gpurun_out/ncu_r02ac.log
echo done
