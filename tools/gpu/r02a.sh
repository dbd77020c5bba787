set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r02a_pytest_gpu.log
timeout 300 python tools/prof_solve.py --config c3 --size 512 --iters 200 > gpurun_out/r02a_c3_plain.log 2>&1; echo "plain rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_solve_kernel -s 1 -c 1 -o gpurun_out/r02a_c3_solve python tools/prof_solve.py --config c3 --size 512 --iters 200 > gpurun_out/r02a_ncu_c3.log 2>&1; echo "ncu rc $?"
