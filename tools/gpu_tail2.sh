timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py tests/test_gpu_solvers.py -m gpu -x -q > gpurun_out/pytest_step.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_step.log
for t in 0 1; do ADP_TAIL=$t timeout 300 python tools/step_ab.py --iters 300 --modes 1; done
ADP_TAIL=1 timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ADP_TAIL=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 60 --csv --log-file gpurun_out/ll1.csv python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/ncu_ll.log 2>&1; echo "ncu rc $?"
