set -u
timeout 900 python -m pytest tests/test_gpu_edges.py -x -q > gpurun_out/r02ai_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r02ai_tests.txt
tail -30 gpurun_out/r02ai_tests.txt
