# round 2: slab hypergradient / MAID tests, then the whole GPU suite
set -x
timeout 1500 python -m pytest tests/test_gpu_slab_hyper.py tests/test_gpu_slabs.py -x -q -rA > gpurun_out/r02d_slab.log 2>&1; echo "slab rc $?"
tail -30 gpurun_out/r02d_slab.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02d_pytest_gpu.log 2>&1; echo "all gpu rc $?"
tail -15 gpurun_out/r02d_pytest_gpu.log
