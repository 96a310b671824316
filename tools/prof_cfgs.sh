# usage: bash tools/prof_cfgs.sh TAG cfg...   (ncu --set full of the top kernel per config)
TAG=$1; shift
# kernel-source hash of this capture (bench.py's roofline.traffic is only
# taken from a capture of the sources it runs)
python -c "import bench; print(bench.src_hash())" > gpurun_out/prof_${TAG}.srchash
for C in "$@"; do
  CMD="python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${TAG}_$C.log 2>&1 || { echo "plain run failed: $C"; exit 1; }
done
for C in "$@"; do
  CMD="python bench.py --config $C --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
  ncu --set full --clock-control none --import-source on -k regex:sfft -s 2 -c 1 -o gpurun_out/prof_${TAG}_$C $CMD > gpurun_out/ncu_${TAG}_$C.log 2>&1
done
