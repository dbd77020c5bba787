timeout 600 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py tests/test_gpu_solvers.py -x -q -m gpu 2>&1 | tail -3
for d in 0 1 2 1 2; do
  echo "ADP_OVL=$d"; ADP_OVL=$d timeout 300 python tools/step_ab.py --modes 1 --iters 300 2>&1 | tail -1
done
