set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 200 -c 8 -o gpurun_out/c3_step python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/prof_plain.log
