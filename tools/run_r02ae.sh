# r02ae: pass2 completion signal deferred to the next tile's mid() (flags 9 / 11) vs at the tile boundary
set -u
OUT=gpurun_out/r02ae_sweep.jsonl
: > $OUT
for rep in 1 2; do
P2_KERNEL=pass timeout 300 python tools/p2_sweep.py 28 f32 dit >> $OUT
for F in 2 11 9 3; do
  SFFT_PASS2=1 SFFT_P2_FLAGS=$F timeout 300 python tools/p2_sweep.py 28 f32 dit >> $OUT
done
SFFT_PASS2=1 SFFT_P2_FLAGS=11 SFFT_P2_LAG=8 SFFT_P2_SLOTS=16 timeout 300 python tools/p2_sweep.py 28 f32 dit >> $OUT
SFFT_PASS2=1 SFFT_P2_FLAGS=11 SFFT_P2_LAG=4 SFFT_P2_SLOTS=8 timeout 300 python tools/p2_sweep.py 28 f32 dit >> $OUT
for F in 0 9; do
  SFFT_P2_FLAGS=$F timeout 300 python tools/p2_sweep.py 28 f64 dit 5 >> $OUT
done
done
cat $OUT
SFFT_PASS2=1 SFFT_P2_FLAGS=11 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02ae_pass2 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02ae.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pass2.py -x -q -k "knobs or plan_reports" > gpurun_out/r02ae_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ae_tests.txt
tail -3 gpurun_out/r02ae_tests.txt
echo done
