set -x
ADP_STEP=1 timeout 300 python tools/step_ab.py --iters 30 --modes 1 > /dev/null 2>&1 && \
ADP_STEP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"step_(b|a|c)_kernel" -s 6 -c 3 -o gpurun_out/r02o_step python tools/step_ab.py --iters 30 --modes 1 > gpurun_out/r02o_ncu.log 2>&1; echo "ncu rc $?"
