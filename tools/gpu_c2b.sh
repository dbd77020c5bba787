timeout 200 python tools/prof_solve.py --config c2 --size 256 --iters 1200 --reps 4
ADP_TMA=0 timeout 200 python tools/prof_solve.py --config c2 --size 256 --iters 1200 --reps 3
python tools/phase_trace.py 2>&1 | tail -14
