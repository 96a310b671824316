set -x
for C in cfg3_n1024_f32 cfg3_n1024_f64 cfg4_n4096_f32; do
  CMD="python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_$C.log 2>&1 || exit 1
done
for C in cfg3_n1024_f32 cfg3_n1024_f64 cfg4_n4096_f32; do
  CMD="python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
  ncu --set full --clock-control none --import-source on -k regex:sfft -s 1 -c 1 -o gpurun_out/prof_$C $CMD > gpurun_out/ncu_$C.log 2>&1
done
