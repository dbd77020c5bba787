set -x
timeout 600 python -m pytest tests/test_gpu_dense_large.py -q -x > gpurun_out/r02h_dense.log 2>&1; echo "dense rc $?"
tail -15 gpurun_out/r02h_dense.log
timeout 900 python tools/sweep_c3.py > gpurun_out/r02h_sweep_pipe1.txt 2>&1; echo "sweep1 rc $?"
cat gpurun_out/r02h_sweep_pipe1.txt
ADP_PIPE=0 timeout 900 python tools/sweep_c3.py > gpurun_out/r02h_sweep_pipe0.txt 2>&1; echo "sweep0 rc $?"
cat gpurun_out/r02h_sweep_pipe0.txt
