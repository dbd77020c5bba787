for t in 0 1; do
ADP_TAIL=$t timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ADP_TAIL=$t timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 60 --csv --log-file gpurun_out/ll$t.csv python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/ncu_ll.log 2>&1; echo "ncu rc $?"
done
