# r02at: headline kernel L2 policies in the settled state: evict-first hint on the input bulk copies, write-back instead of streaming output stores
set -u
OUT=gpurun_out/r02at_ab.txt
: > $OUT
run() {  # name lib algo
  SFFT_B200_LIB=$2 python bench.py --algorithm $3 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$1', '$3', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['parity'].get('bitwise'))" >> $OUT
}
CUR=paper_2504_07264_b200/libsplitfft_b200.so
for rep in 1 2 3 4; do
  run cur $CUR dit
  for v in ef plain efplain; do run $v build/variants/$v.so dit; done
done
for rep in 1 2; do
  run cur $CUR dif
  for v in ef plain efplain; do run $v build/variants/$v.so dif; done
done
cat $OUT
