# A/B of build variants on one box: VARIANTS="name=extra nvcc flags;..." (current sources),
# plus OLD from ab_old/csrc when present.  CONFIGS: bench configs.  Each bench twice, interleaved.
set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
DIRS=()
IFS=';' read -ra VS <<< "${VARIANTS:-cur=}"
for v in "${VS[@]}"; do
  name=${v%%=*}; flags=${v#*=}
  d=/tmp/ab_$name; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
  # a "ENV:K=V" word in the flags is exported for the generator instead of passed to nvcc
  envs=$(echo "$flags" | tr ' ' '\n' | grep '^ENV:' | sed 's/^ENV://' | tr '\n' ' ')
  nvf=$(echo "$flags" | tr ' ' '\n' | grep -v '^ENV:' | tr '\n' ' ')
  (cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu && env $envs make -B -j16 NVFLAGS="$NV $nvf") > $d.log 2>&1 || { tail -5 $d.log; exit 1; }
  DIRS+=("$name:$d")
done
if [ -d "$GRAFT_REPO_ROOT/ab_old/csrc" ] && [ -n "$WITH_OLD" ]; then
  d=/tmp/ab_old; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
  rm -rf $d/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc $d/paper_2504_07264_b200/csrc
  make -C $d/paper_2504_07264_b200/csrc -B -j16 > $d.log 2>&1 || { tail -5 $d.log; exit 1; }
  DIRS+=("old:$d")
fi
# ALGOS: "dit" (default) and/or "dif"
for C in ${CONFIGS:-cfg2_n64_f32}; do
 for A in ${ALGOS:-dit}; do
  for i in $(seq ${REPS:-2}); do
    for nd in "${DIRS[@]}"; do
      n=${nd%%:*}; d=${nd#*:}
      (cd $d && python bench.py --config $C --algorithm $A --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$n', '$C', '$A', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
    done
  done
 done
done
