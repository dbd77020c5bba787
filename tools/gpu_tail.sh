set -x
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/pytest_step.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_step.log
for t in 0 1; do ADP_TAIL=$t timeout 300 python tools/step_ab.py --iters 300 --modes 1; done
timeout 600 python bench.py --no-extra --maid-steps 0 --no-cpu > gpurun_out/bench_tail.json 2> gpurun_out/bench_tail.err; echo "bench rc $?"
cat gpurun_out/bench_tail.json
