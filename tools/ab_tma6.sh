# A/B of TMA configs for N=64 fp32 (cfg2): separate builds in /tmp, bench each twice
set -e
run() {  # $1 = dir
  (cd "$1" && python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$2', round(d['ms_per_step'],5), round(d['roofline']['frac'],4))")
}
for V in "3,256,3,2" "3,256,2,1" "3,256,3,1"; do
  D=/tmp/v_${V//,/_}
  rm -rf $D && cp -r "$GRAFT_REPO_ROOT" $D
  SFFT_TMA_OVERRIDE="f32:6:$V" make -C $D/paper_2504_07264_b200/csrc -B -j32 > $D.log 2>&1 || { echo "build $V failed"; tail -5 $D.log; continue; }
  run $D "$V"; run $D "$V"
done
