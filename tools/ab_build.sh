# A/B of build variants on one GPU box (run under gpurun from the repo root).
#   VARIANTS="name|ENV=.. ENV2=..|extra nvcc flags ;; name2|...|..."   (';;'-separated)
#   CONFIGS="cfg3_n1024_f64 ..."  ALGOS="dit dif"  REPS=2  STEPS=100
# Each variant is a copy of the tree rebuilt with the given generator
# environment (SFFT_TMA_OVERRIDE, SFFT_AUTO_OVERRIDE, ...) and nvcc flags;
# "cur" (the tree as shipped, prebuilt .so) is always included.
set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
ROOT=${GRAFT_REPO_ROOT:-$(pwd)}
names="cur"
while IFS= read -r v; do
  [ -z "$v" ] && continue
  name=${v%%|*}; rest=${v#*|}; envs=${rest%%|*}; flags=${rest#*|}
  d=/tmp/ab_$name; rm -rf $d && cp -r "$ROOT" $d
  (cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu sfft_small_tw.h && env $envs make -B -j32 NVFLAGS="$NV $flags") > $d.log 2>&1 || { echo "build $name failed"; tail -20 $d.log; exit 1; }
  names="$names $name"
done < <(echo "${VARIANTS:-}" | sed 's/;;/\n/g')
run() {  # dir name config algo
  (cd $1 && python bench.py --config $3 --algorithm $4 --steps ${STEPS:-100} --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$2', '$3', '$4', d['roofline'].get('kernel', ''), round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
}
for i in $(seq ${REPS:-2}); do
  for C in ${CONFIGS:-cfg3_n1024_f64}; do
    for A in ${ALGOS:-dit}; do
      for n in $names; do
        if [ $n = cur ]; then run "$ROOT" cur $C $A; else run /tmp/ab_$n $n $C $A; fi
      done
    done
  done
done
