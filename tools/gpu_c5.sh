timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py tests/test_gpu_k31.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/pytest_step.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_step.log
ADP_STEP=0 timeout 300 python tools/prof_solve.py --config c5 --size 4096 --iters 10 --reps 2
timeout 300 python tools/prof_solve.py --config c5 --size 4096 --iters 10 --reps 2
timeout 300 python tools/step_ab.py --iters 300 --modes 1
