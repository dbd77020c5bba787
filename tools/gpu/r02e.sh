# slab hypergradient / MAID tests; c3 and c2 phase traces
set -x
timeout 1500 python -m pytest tests/test_gpu_slab_hyper.py -x -q -rA > gpurun_out/r02e_slab.log 2>&1; echo "slab rc $?"
tail -15 gpurun_out/r02e_slab.log
timeout 300 python tools/phase_trace.py --config c3 --size 512 > gpurun_out/r02e_phase_c3.txt 2>&1; echo "phase rc $?"
cat gpurun_out/r02e_phase_c3.txt
