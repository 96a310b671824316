# r02ap: 10 warps (ring of 11 / 12 / 13 slots) vs the shipped 9 warps + 11 slots, settled power state, alternating
set -u
OUT=gpurun_out/r02ap_ab.txt
: > $OUT
run() {  # name lib algo
  SFFT_B200_LIB=$2 python bench.py --algorithm $3 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$1', '$3', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['parity'].get('bitwise'))" >> $OUT
}
CUR=paper_2504_07264_b200/libsplitfft_b200.so
for rep in 1 2 3 4 5; do
  for A in dit dif; do
    run cur $CUR $A
    for v in w10 w10x1 w10x3; do run $v build/variants/$v.so $A; done
  done
done
cat $OUT
