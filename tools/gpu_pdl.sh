set -x
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/pytest_step.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_step.log
for t in 0 1; do ADP_PDL=$t timeout 300 python tools/step_ab.py --iters 300 --modes 1; done
