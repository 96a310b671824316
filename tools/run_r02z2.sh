# r02z2: pass2 with look-ahead polling / relaxed counters: parity + ring sweep + ncu
set -u
timeout 900 python -m pytest tests/test_gpu_pass2.py -x -q > gpurun_out/r02z2_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02z2_tests.txt
tail -3 gpurun_out/r02z2_tests.txt
OUT=gpurun_out/r02z2_sweep.jsonl
: > $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
for DS in "2 4" "3 4" "4 8" "6 8" "8 16" "12 16"; do
  set -- $DS
  SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f32 dit >> $OUT
done
python tools/p2_sweep.py 28 f32 dif >> $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dif >> $OUT
python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
cat $OUT
ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02z2_pass2 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02z2.log 2>&1
tail -1 gpurun_out/ncu_r02z2.log
echo done
