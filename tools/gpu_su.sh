for su in 5 1; do echo "ADP_SU=$su"; ADP_SU=$su timeout 300 python tools/step_ab.py --iters 300 --modes 1; done
for su in 1; do
ADP_SU=$su timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ADP_SU=$su timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 40 --csv --log-file gpurun_out/ll_su$su.csv python tools/prof_solve.py --config c3 --size 512 --iters 60 --reps 2 > gpurun_out/ncu_ll.log 2>&1; echo "ncu rc $?"
done
