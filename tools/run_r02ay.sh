# r02ay: cfg2 (N=64 fp32) TMA pipeline shapes in the settled power state (variants prebuilt, SFFT_B200_LIB)
set -u
OUT=gpurun_out/r02ay_ab.txt
: > $OUT
run() {  # name lib
  SFFT_B200_LIB=$2 python bench.py --config cfg2_n64_f32 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$1', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['parity'].get('pass'))" >> $OUT
}
CUR=paper_2504_07264_b200/libsplitfft_b200.so
for rep in 1 2 3; do
  run cur $CUR
  for v in s2t128 s1t128 s2t64 s2t128o1 s2t128m; do run $v build/variants/$v.so; done
done
cat $OUT
