# A/B of build variants on one box with per-run bench arguments.
# VARIANTS="name=extra nvcc flags;..." (ENV:K=V words go to the generator),
# RUNS="config:algorithm:extra bench args (commas for spaces);..."
set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
NAMES=()
IFS=';' read -ra VS <<< "${VARIANTS:-cur=}"
for v in "${VS[@]}"; do
  name=${v%%=*}; flags=${v#*=}
  d=/tmp/ab_$name; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
  envs=$(echo "$flags" | tr ' ' '\n' | grep '^ENV:' | sed 's/^ENV://' | tr '\n' ' ')
  nvf=$(echo "$flags" | tr ' ' '\n' | grep -v '^ENV:' | tr '\n' ' ')
  (cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu && env $envs make -B -j16 NVFLAGS="$NV $nvf") > $d.log 2>&1 || { tail -5 $d.log; exit 1; }
  NAMES+=("$name")
done
IFS=';' read -ra RS <<< "${RUNS:-cfg2_n64_f32:dit:}"
for i in $(seq ${REPS:-2}); do
  for r in "${RS[@]}"; do
    C=$(echo "$r" | cut -d: -f1); A=$(echo "$r" | cut -d: -f2); X=$(echo "$r" | cut -d: -f3- | tr ',' ' ')
    for n in "${NAMES[@]}"; do
      (cd /tmp/ab_$n && python bench.py --config $C --algorithm $A $X --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$n', '$C', '$A', '$X', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
    done
  done
done
