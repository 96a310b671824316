set -e
NV="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr"
for v in "nopdl:-DSFFT_TMA_NO_PDL" "pdl:"; do
  name=${v%%:*}; flags=${v#*:}
  d=/tmp/ab_$name; rm -rf $d && cp -r "$GRAFT_REPO_ROOT" $d
  (cd $d/paper_2504_07264_b200/csrc && rm -f sfft_inst_*.cu && make -B -j16 NVFLAGS="$NV $flags") > $d.log 2>&1 || { tail -5 $d.log; exit 1; }
done
(cd /tmp/ab_pdl && timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "tma" > $GRAFT_REPO_ROOT/gpurun_out/pdl_parity.log 2>&1; echo rc=$? >> $GRAFT_REPO_ROOT/gpurun_out/pdl_parity.log)
for i in 1 2 3; do
  for se in 1 0; do
    for n in nopdl pdl; do
      (cd /tmp/ab_$n && SFFT_BENCH_STEP_EVENTS=$se python bench.py --config cfg2_n64_f32 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$n', 'step_events=$se', round(d['ms_per_step'],5), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))")
    done
  done
done
