set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc $?"
cat gpurun_out/ref.json
timeout 600 python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/bench_short.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 50 -c 3 -o gpurun_out/c3_step_final python tools/prof_solve.py --config c3 --size 512 --iters 40 --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc $?"
