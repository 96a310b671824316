# A/B on one box: current sources vs ab_old/csrc (previous commit) on the bench
# configs, plus the current build at forced register radices (RADIX="cfg:lr ...").
set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
build() {  # name srcdir
  d=/tmp/ab_$1; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
  if [ -n "$2" ]; then rm -rf $d/paper_2504_07264_b200/csrc && cp -r $2 $d/paper_2504_07264_b200/csrc; fi
  (cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu && make -B -j16 NVFLAGS="$NV") > $d.log 2>&1 || { tail -5 $d.log; exit 1; }
}
build cur ""
build old "$GRAFT_REPO_ROOT/ab_old/csrc"
run() {  # name config algo extra
  (cd /tmp/ab_$1 && python bench.py --config $2 --algorithm $3 $4 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$2', '$3', '$4', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
}
for i in $(seq ${REPS:-2}); do
  for C in ${CONFIGS:-cfg2_n64_f32}; do
    for A in ${ALGOS:-dit}; do
      run old $C $A ""
      run cur $C $A ""
    done
  done
  for cl in ${RADIX}; do
    C=${cl%%:*}; L=${cl#*:}
    for A in ${ALGOS:-dit}; do run cur $C $A "--radix-log $L"; done
  done
done
