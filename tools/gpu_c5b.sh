timeout 300 python tools/prof_solve.py --config c5 --size 4096 --iters 6 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 14 -c 2 -o gpurun_out/c5_step python tools/prof_solve.py --config c5 --size 4096 --iters 6 --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
