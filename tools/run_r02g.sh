set -u
TAG=r02g
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
python bench.py > gpurun_out/${TAG}_default.json 2> gpurun_out/${TAG}_default.err
bash tools/prof_cfgs.sh $TAG cfg3_n1024_f64 cfg4_n4096_f32
echo done
