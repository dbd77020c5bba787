timeout 200 python tools/prof_solve.py --config c2 --size 256 --iters 1200 --reps 3
ADP_STEP=1 ADP_RW=4 timeout 200 python tools/prof_solve.py --config c2 --size 256 --iters 1200 --reps 3
ADP_STEP=1 ADP_RW=4 ADP_TAIL=0 timeout 200 python tools/prof_solve.py --config c2 --size 256 --iters 1200 --reps 3
