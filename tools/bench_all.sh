# usage: bash tools/bench_all.sh TAG  -- one bench line per BASELINE config + the reference arm
TAG=$1
for C in cfg1_n8_f64 cfg2_n64_f32 cfg3_n1024_f32 cfg3_n1024_f64 cfg4_n4096_f32 cfg5_n2p28_f32; do
  timeout 900 python bench.py --config $C --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_${TAG}_$C.json 2> gpurun_out/bench_${TAG}_$C.err || echo "FAILED $C"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_reference.json 2>&1 || echo "FAILED reference"
