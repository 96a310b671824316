# ncu --set full on cfg2's kernel for the current build and ab_old (same box)
set -e
d=/tmp/ab_old; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
rm -rf $d/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc $d/paper_2504_07264_b200/csrc
make -C $d/paper_2504_07264_b200/csrc -B -j16 > $d.log 2>&1
C="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
$C > gpurun_out/abn_new_plain.log 2>&1
(cd $d && $C > "$GRAFT_REPO_ROOT"/gpurun_out/abn_old_plain.log 2>&1)
ncu --set full --import-source on --clock-control none -k regex:sfft -s 30 -c 1 -o gpurun_out/abn_new $C > gpurun_out/abn_new.log 2>&1
(cd $d && ncu --set full --import-source on --clock-control none -k regex:sfft -s 30 -c 1 -o "$GRAFT_REPO_ROOT"/gpurun_out/abn_old $C > "$GRAFT_REPO_ROOT"/gpurun_out/abn_old.log 2>&1)
