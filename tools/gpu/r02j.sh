# round 2 consolidated measurement: GPU suite, smoke, default bench, reference arm, c5/c2 lines,
# launch list and one ncu --set full capture of the c3 solve kernel
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02j_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r02j_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; echo "smoke rc $?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02j_ref.json 2> gpurun_out/r02j_ref.err; echo "ref rc $?"
timeout 900 python bench.py --workload c5 --steps 3 --warmup 1 > gpurun_out/r02j_c5.json 2> gpurun_out/r02j_c5.err; echo "c5 rc $?"
timeout 900 python bench.py --workload c2 --steps 20 --warmup 5 --no-extra --maid-steps 0 > gpurun_out/r02j_c2.json 2> gpurun_out/r02j_c2.err; echo "c2 rc $?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02j_short.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02j_launches.csv python bench.py --steps 2 --warmup 1 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02j_ncu_launch.log 2>&1; echo "ncu1 rc $?"
timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 1200 > gpurun_out/r02j_c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_solve_kernel -s 1 -c 1 -o gpurun_out/r02j_c3_solve python tools/prof_solve.py --config c3 --size 512 --iters 1200 > gpurun_out/r02j_ncu_c3.log 2>&1; echo "ncu2 rc $?"
