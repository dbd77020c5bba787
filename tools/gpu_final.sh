set -x
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu1 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_solve_kernel -s 1 -c 1 -o gpurun_out/c2_solve_final python tools/prof_solve.py --iters 1200 > gpurun_out/ncu_full_final.log 2>&1; echo "ncu2 rc $?"
