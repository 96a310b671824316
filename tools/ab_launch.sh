set -e
d=/tmp/ab_old; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
rm -rf $d/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc $d/paper_2504_07264_b200/csrc
make -C $d/paper_2504_07264_b200/csrc -B -j16 > $d.log 2>&1
for i in 1 2; do echo -n "new "; python tools/launch_probe.py; (cd $d && echo -n "old " && python tools/launch_probe.py); done
