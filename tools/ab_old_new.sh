# A/B: current kernels vs ab_old/csrc (previous sources), same box, cfg2 + cfg4 + cfg3f64 benches
set -e
rm -rf /tmp/repoOld && cp -r "$GRAFT_REPO_ROOT" /tmp/repoOld
rm -rf /tmp/repoOld/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc /tmp/repoOld/paper_2504_07264_b200/csrc
make -C /tmp/repoOld/paper_2504_07264_b200/csrc -B -j16 > /tmp/repoOld_build.log 2>&1 || { tail -20 /tmp/repoOld_build.log; exit 1; }
b() { (cd "$1" && python bench.py --config $2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$3', '$2', round(d['ms_per_step'],5), round(d['roofline']['frac'],4))"); }
for C in ${CONFIGS:-cfg2_n64_f32 cfg4_n4096_f32 cfg3_n1024_f32}; do
  for i in 1 2; do b "$GRAFT_REPO_ROOT" $C NEW; b /tmp/repoOld $C OLD; done
done
