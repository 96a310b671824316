# r02z: pass2 ring geometry sweep + ncu of the fused launches (cfg5 m=28 fp32)
set -u
OUT=gpurun_out/r02z_sweep.jsonl
: > $OUT
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
for DS in "4 8" "8 12" "12 16" "16 20" "24 32" "30 32"; do
  set -- $DS
  SFFT_P2_LAG=$1 SFFT_P2_SLOTS=$2 python tools/p2_sweep.py 28 f32 dit >> $OUT
done
P2_KERNEL=pass python tools/p2_sweep.py 28 f32 dit >> $OUT
cat $OUT
ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02z_pass2 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02z.log 2>&1
SFFT_P2_LAG=16 SFFT_P2_SLOTS=20 ncu --set full --clock-control none --import-source on -k regex:pass2 -c 2 -o gpurun_out/prof_r02z_pass2_lag16 \
  python tools/p2_sweep.py 28 f32 dit 1 > gpurun_out/ncu_r02z_lag16.log 2>&1
tail -2 gpurun_out/ncu_r02z.log
echo done
