# r02n: fp64 N=1024 warp kernel vs radix-8 TMA kernel across batch sizes (crossover for kernel=auto)
set -u
for B in 28 29 30 31 32 33; do
  for A in dit dif; do
    python tools/tune.py --sizes 10 --dtypes f64 --algo $A --bytes $((1 << B)) 2>&1 | grep -v best | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if d.get('kernel') == 'tma': print('$A', d['batch'], d['lr'], round(d['GBs']))" >> gpurun_out/r02n_batch_sweep.txt
  done
done
cat gpurun_out/r02n_batch_sweep.txt
