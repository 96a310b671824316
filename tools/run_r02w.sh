# r02w: L2 prefetch-ahead in the slot ring (fp64 N=1024 headline, fp32 N=4096) -- A/B + parity
set -u
VARIANTS="pf9|SFFT_TMAW=f64:10:9,3,1,1,2,1,9|;;pf18|SFFT_TMAW=f64:10:9,3,1,1,2,1,18|" CONFIGS="cfg3_n1024_f64" ALGOS="dit dif" REPS=3 timeout 1500 bash tools/ab_build.sh > gpurun_out/r02w_ab.txt 2>&1
cat gpurun_out/r02w_ab.txt
(cd /tmp/ab_pf9 && timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "warp_kernel or (tma_kernel_many_tiles and f64 and 10)") > gpurun_out/r02w_tests.txt 2>&1
tail -1 gpurun_out/r02w_tests.txt
VARIANTS="pf4|SFFT_TMAW=f32:12:8,0,0,1,2,2,4|" CONFIGS="cfg4_n4096_f32" ALGOS="dit dif" REPS=3 timeout 1200 bash tools/ab_build.sh > gpurun_out/r02w_ab32.txt 2>&1
cat gpurun_out/r02w_ab32.txt
for B in 26 27 28 29; do
  for A in dit dif; do
    python tools/tune.py --sizes 12 --dtypes f32 --algo $A --bytes $((1 << B)) 2>&1 | grep -v best | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if (d.get('kernel'), d.get('lr')) in (('tma', 6), ('ldg', 4)) and not d.get('pre'): print('$A', d['batch'], d['kernel'], d['lr'], round(d['GBs']))" >> gpurun_out/r02w_batch_sweep32.txt
  done
done
cat gpurun_out/r02w_batch_sweep32.txt
