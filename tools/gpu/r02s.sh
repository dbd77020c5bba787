set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02s_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r02s_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err; echo "bench rc $?"
tail -c 3000 gpurun_out/r02s_bench.json
tail -3 gpurun_out/r02s_bench.err
