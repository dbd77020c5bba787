timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 40 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 50 -c 3 -o gpurun_out/c3_ca4 python tools/prof_solve.py --config c3 --size 512 --iters 40 --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
