set -x
timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_ -s 200 -c 8 -o gpurun_out/c3_step2 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/prof_plain.log
