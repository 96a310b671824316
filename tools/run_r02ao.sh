# r02ao: headline kernel warp count / ring depth / prefetch re-swept in the settled power state
# (variants prebuilt in build/variants/*.so, selected with SFFT_B200_LIB)
set -u
OUT=gpurun_out/r02ao_ab.txt
: > $OUT
run() {  # name lib algo
  SFFT_B200_LIB=$2 python bench.py --algorithm $3 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$1', '$3', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['parity'].get('bitwise'))" >> $OUT
}
CUR=paper_2504_07264_b200/libsplitfft_b200.so
for rep in 1 2 3; do
  run cur $CUR dit
  for v in w10 w11 w12x1 w12x2 w9pf2 w9x3; do run $v build/variants/$v.so dit; done
done
for rep in 1 2; do
  run cur $CUR dif
  for v in w10 w12x1 w12x2; do run $v build/variants/$v.so dif; done
done
cat $OUT
