# pipelined RW=4 stages: parity tests, phase trace, A/B bench
set -x
timeout 1200 python -m pytest tests/test_gpu_lockstep.py tests/test_gpu_k31.py tests/test_gpu_solvers.py tests/test_gpu_primitives.py tests/test_gpu_fused.py -x -q > gpurun_out/r02g_pytest.log 2>&1; echo "tests rc $?"
tail -4 gpurun_out/r02g_pytest.log
timeout 300 python tools/phase_trace.py --config c3 --size 512 > gpurun_out/r02g_phase_c3.txt 2>&1; echo "phase rc $?"
cat gpurun_out/r02g_phase_c3.txt
ADP_PIPE=0 timeout 600 python bench.py --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02g_bench_pipe0.json 2>&1; echo "b0 rc $?"
timeout 600 python bench.py --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02g_bench_pipe1.json 2>&1; echo "b1 rc $?"
python - <<'PY'
import json
for f in ("gpurun_out/r02g_bench_pipe0.json", "gpurun_out/r02g_bench_pipe1.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"])
PY
