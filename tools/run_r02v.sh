# r02v: fp32 N=4096 auto = signal-group kernel: batch crossover vs LDG, parity, e2e + PCIe on one box
set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "auto_batch or tma_kernel_many_tiles or f32_rel or every_radix or strided or graph or config4 or full_batch" > gpurun_out/r02v_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02v_tests.txt
tail -2 gpurun_out/r02v_tests.txt
for B in 26 27 28 29 30; do
  for A in dit dif; do
    python tools/tune.py --sizes 12 --dtypes f32 --algo $A --bytes $((1 << B)) 2>&1 | grep -v best | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    if (d.get('kernel'), d.get('lr')) in (('tma', 6), ('ldg', 4)) and not d.get('pre'): print('$A', d['batch'], d['kernel'], d['lr'], round(d['GBs']))" >> gpurun_out/r02v_batch_sweep.txt
  done
done
cat gpurun_out/r02v_batch_sweep.txt
python tools/pcie_probe.py > gpurun_out/r02v_pcie.txt 2>&1; tail -1 gpurun_out/r02v_pcie.txt
python bench.py --steps 20 > gpurun_out/r02v_default.json 2> gpurun_out/r02v_default.err
python bench.py --config cfg4_n4096_f32 --steps 20 > gpurun_out/r02v_cfg4.json 2> gpurun_out/r02v_cfg4.err
echo done
