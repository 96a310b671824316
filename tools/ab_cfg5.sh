# A/B: pass kernel with / without the up-front base factors (cfg5)
set -e
rm -rf /tmp/repoB && cp -r "$GRAFT_REPO_ROOT" /tmp/repoB
make -C /tmp/repoB/paper_2504_07264_b200/csrc -B -j16 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -DSFFT_NO_PASS_PRE" > /tmp/repoB_build.log 2>&1
for i in 1 2; do
  python bench.py --config cfg5_n2p28_f32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('A(pre)',d['ms_per_step'])"
  (cd /tmp/repoB && python bench.py --config cfg5_n2p28_f32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('B(nopre)',d['ms_per_step'])")
done
