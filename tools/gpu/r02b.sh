# round-2 bench re-anchor on c3: default bench, reference arm, launch list, ncu of one c3 step
set -x
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err; echo "ref rc $?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02b_short.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02b_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 1200 > gpurun_out/r02b_c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_solve_kernel -s 1 -c 1 -o gpurun_out/r02b_c3_solve python tools/prof_solve.py --config c3 --size 512 --iters 1200 > gpurun_out/r02b_ncu_c3.log 2>&1; echo "ncu2 rc $?"
