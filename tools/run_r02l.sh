# r02l: X2 exchange vs planar across fp32 sizes (tune sweep on both builds), ncu of cfg4 with X2
set -u
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
d=/tmp/ab_nox2; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
(cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu sfft_small_tw.h && make -B -j32 NVFLAGS="$NV -DSFFT_FUSED_NO_X2") > /tmp/nox2.log 2>&1 || tail -5 /tmp/nox2.log
for A in dit dif; do
  python tools/tune.py --sizes 7,8,9,10,11,12 --dtypes f32 --algo $A > gpurun_out/r02l_tune_x2_$A.txt 2>&1
  (cd $d && python tools/tune.py --sizes 7,8,9,10,11,12 --dtypes f32 --algo $A) > gpurun_out/r02l_tune_nox2_$A.txt 2>&1
done
python tools/tune.py --sizes 10 --dtypes f64 --algo dit > gpurun_out/r02l_tune_f64_10_dit.txt 2>&1
B="python bench.py --config cfg4_n4096_f32 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_r02l_cfg4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sfft -s 2 -c 1 -o gpurun_out/prof_r02l_cfg4_x2 $B > gpurun_out/ncu_r02l_cfg4.log 2>&1
grep best gpurun_out/r02l_tune_*.txt
