# r02af: driver-style check of the final tree: smoke(), the default bench command, the reference arm, a 2-rank spawn on one GPU
set -u
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02af_smoke.txt 2>&1; tail -2 gpurun_out/r02af_smoke.txt
python bench.py > gpurun_out/r02af_default.json 2> gpurun_out/r02af_default.err; tail -c 600 gpurun_out/r02af_default.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02af_reference.json 2>&1; tail -c 300 gpurun_out/r02af_reference.json
echo done
