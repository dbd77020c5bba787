set -x
timeout 600 python tools/step_ab.py > gpurun_out/r02n_step_ab.txt 2>&1; cat gpurun_out/r02n_step_ab.txt
ADP_STEP=1 timeout 300 python tools/step_ab.py --iters 30 --modes 1 > /dev/null 2>&1 && \
ADP_STEP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r02n_step_launches.csv python tools/step_ab.py --iters 30 --modes 1 > gpurun_out/r02n_ncu.log 2>&1; echo "ncu rc $?"
