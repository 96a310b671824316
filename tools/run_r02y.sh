# r02y: L2-fused group pairs (sfft_pass2) -- parity + cfg5 timing vs the per-group schedule
set -u
timeout 900 python -m pytest tests/test_gpu_pass2.py -x -q > gpurun_out/r02y_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02y_tests.txt
tail -5 gpurun_out/r02y_tests.txt
for v in 1 0 1 0; do
  SFFT_PASS2=$v timeout 300 python bench.py --config cfg5_n2p28_f32 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/r02y_cfg5_p2$v.json 2> gpurun_out/r02y_cfg5_p2$v.err
  python -c "import json;d=json.loads(open('gpurun_out/r02y_cfg5_p2$v.json').read().strip().splitlines()[-1]);print('p2=$v', d['ms_per_step'], d['roofline']['frac'], d['parity']['rel_l2_global'], d['clocks'])" || tail -5 gpurun_out/r02y_cfg5_p2$v.err
done
for A in dit dif; do
  timeout 300 python bench.py --config cfg5_n2p28_f32 --algorithm $A --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/r02y_cfg5_$A.json 2>&1
  tail -1 gpurun_out/r02y_cfg5_$A.json | cut -c1-300
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "large_m or pass_kernel_variants or (f64_bitwise and (20 or 22)) or (f32_rel and (20 or 22))" > gpurun_out/r02y_tests2.txt 2>&1; echo "rc=$?" >> gpurun_out/r02y_tests2.txt
tail -3 gpurun_out/r02y_tests2.txt
echo done
