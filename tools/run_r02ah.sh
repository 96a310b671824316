# r02ah: run-to-run spread of the default bench command's device-timed value on one box (8 back-to-back processes)
set -u
: > gpurun_out/r02ah_spread.txt
for i in 1 2 3 4 5 6 7 8; do
  python bench.py --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" >> gpurun_out/r02ah_spread.txt
done
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.mem,power.limit,power.draw,temperature.gpu --format=csv >> gpurun_out/r02ah_spread.txt
cat gpurun_out/r02ah_spread.txt
