set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"step_ca_kernel|step_b_kernel" -s 40 -c 2 -o gpurun_out/r02v_step python tools/prof_solve.py --config c3 --size 512 --iters 40 --reps 2 > gpurun_out/r02v_ncu.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/r02v_ncu.log
