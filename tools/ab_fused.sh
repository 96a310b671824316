# A/B: fused/TMA kernels with / without up-front base factors (fp32)
set -e
rm -rf /tmp/repoB && cp -r "$GRAFT_REPO_ROOT" /tmp/repoB
make -C /tmp/repoB/paper_2504_07264_b200/csrc -B -j16 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -DSFFT_NO_FUSED_PRE" > /tmp/repoB_build.log 2>&1
python tools/tune.py --dtypes f32 --sizes 6,7,8,9,10,11,12 > gpurun_out/ab_A.log 2>&1
(cd /tmp/repoB && python tools/tune.py --dtypes f32 --sizes 6,7,8,9,10,11,12 > "$GRAFT_REPO_ROOT"/gpurun_out/ab_B.log 2>&1)
python tools/tune.py --dtypes f32 --sizes 6,7,8,9,10,11,12 > gpurun_out/ab_A2.log 2>&1
