# r02ab: pass2 with (re, im)-pair scratch, compile-time scratch strides, per-thread L2 prefetch
set -u
timeout 1200 python -m pytest tests/test_gpu_pass2.py -x -q > gpurun_out/r02ab_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ab_tests.txt
tail -3 gpurun_out/r02ab_tests.txt
OUT=gpurun_out/r02ab_sweep.jsonl
: > $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
for F in 0 2 3 6; do
 for DS in "4 8" "6 16" "8 16"; do
  set -- $DS
  SFFT_PASS2=1 SFFT_P2_FLAGS=$F SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f32 dit >> $OUT
 done
done
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
for F in 0 2; do
  SFFT_PASS2=1 SFFT_P2_FLAGS=$F SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 python tools/p2_sweep.py 28 f32 dif >> $OUT
  SFFT_P2_FLAGS=$F python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
  SFFT_P2_FLAGS=$F SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
  SFFT_P2_FLAGS=$F python tools/p2_sweep.py 24 f64 dit 10 >> $OUT
  SFFT_PASS2=1 SFFT_P2_FLAGS=$F python tools/p2_sweep.py 24 f32 dit 10 >> $OUT
done
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dif >> $OUT
P2_KERNEL=pass python tools/p2_sweep.py 24 f32 dit 10 >> $OUT
cat $OUT
SFFT_PASS2=1 SFFT_P2_FLAGS=2 SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02ab_pass2 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02ab.log 2>&1
tail -1 gpurun_out/ncu_r02ab.log
echo done
