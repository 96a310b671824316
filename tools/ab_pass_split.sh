for i in 1 2; do
for SP in "" "8,7,7,6" "6,7,7,8" "7,7,8,6" "8,8,6,6" "7,7,6,8"; do
  SFFT_PASS_SPLIT=$SP python bench.py --config cfg5_n2p28_f32 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('split=$SP', round(d['ms_per_step'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done
done
