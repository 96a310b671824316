# r02q: ring depth (extra slots) A/B for the fp64 N=1024 warp kernel, batch crossover re-sweep, parity
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or (tma_kernel_many_tiles and f64 and 10) or auto_batch_switch or (f64_bitwise and 10) or strided or graph" > gpurun_out/r02q_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02q_tests.txt
tail -2 gpurun_out/r02q_tests.txt
VARIANTS="xs2|SFFT_TMAW=f64:10:9,3,1,1,2|;;xs3|SFFT_TMAW=f64:10:9,3,1,1,3|;;w10xs2|SFFT_TMAW=f64:10:10,3,1,1,2|;;w8xs2|SFFT_TMAW=f64:10:8,3,1,1,2|" CONFIGS=cfg3_n1024_f64 ALGOS="dit dif" REPS=2 timeout 1800 bash tools/ab_build.sh > gpurun_out/r02q_ab.txt 2>&1
cat gpurun_out/r02q_ab.txt
for B in 28 29 30 31 32 33; do
  for A in dit dif; do
    python tools/tune.py --sizes 10 --dtypes f64 --algo $A --bytes $((1 << B)) 2>&1 | grep -v best | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if d.get('kernel') == 'tma': print('$A', d['batch'], d['lr'], round(d['GBs']))" >> gpurun_out/r02q_batch_sweep.txt
  done
done
cat gpurun_out/r02q_batch_sweep.txt
