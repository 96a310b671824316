# r02x: re-entry check of HEAD (ring kernel PF knob, group kernel): GPU tests, default bench, cfg4 bench
set -u
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit,temperature.gpu --format=csv > gpurun_out/r02x_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02x_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02x_gpu_tests.txt
tail -3 gpurun_out/r02x_gpu_tests.txt
python bench.py > gpurun_out/r02x_default.json 2> gpurun_out/r02x_default.err
python bench.py --config cfg4_n4096_f32 > gpurun_out/r02x_cfg4.json 2> gpurun_out/r02x_cfg4.err
python bench.py --config cfg5_n2p28_f32 --no-cpu-baseline > gpurun_out/r02x_cfg5.json 2> gpurun_out/r02x_cfg5.err
echo done
