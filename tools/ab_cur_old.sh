set -e
o=/tmp/ab_old; rm -rf $o && cp -r "$GRAFT_REPO_ROOT" $o
rm -rf $o/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc $o/paper_2504_07264_b200/csrc
make -C $o/paper_2504_07264_b200/csrc -B -j16 > $o.log 2>&1
for C in ${CONFIGS:-cfg2_n64_f32 cfg3_n1024_f32 cfg3_n1024_f64 cfg4_n4096_f32}; do for i in 1 2; do
  python bench.py --config $C --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cur', '$C', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'))"
  (cd $o && python bench.py --config $C --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('old', '$C', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'))")
done; done
