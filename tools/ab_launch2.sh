set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
d=/tmp/ab_gen; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
make -C $d/paper_2504_07264_b200/csrc -B -j16 NVFLAGS="$NV -DSFFT_TMA_GENERIC_SMEM" > $d.log 2>&1
e=/tmp/ab_gens; rm -rf $e && cp -r "$GRAFT_REPO_ROOT" $e
make -C $e/paper_2504_07264_b200/csrc -B -j16 NVFLAGS="$NV -DSFFT_TMA_GENERIC_SMEM -DSFFT_TMA_SCALAR" > $e.log 2>&1
o=/tmp/ab_old; rm -rf $o && cp -r "$GRAFT_REPO_ROOT" $o
rm -rf $o/paper_2504_07264_b200/csrc && cp -r "$GRAFT_REPO_ROOT"/ab_old/csrc $o/paper_2504_07264_b200/csrc
make -C $o/paper_2504_07264_b200/csrc -B -j16 > $o.log 2>&1
for i in 1 2; do
  echo -n "new-lds-pack "; python tools/launch_probe.py
  (cd $d && echo -n "generic-pack " && python tools/launch_probe.py)
  (cd $e && echo -n "generic-scalar " && python tools/launch_probe.py)
  (cd $o && echo -n "old " && python tools/launch_probe.py)
done
