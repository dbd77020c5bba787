# TMA c2 kernel: parity tests, A/B bench; c5 side lines after the cache fix
set -x
timeout 1200 python -m pytest tests/test_gpu_lockstep.py tests/test_gpu_solvers.py tests/test_gpu_primitives.py tests/test_gpu_fused.py tests/test_gpu_fft.py -x -q > gpurun_out/r02k_pytest.log 2>&1; echo "tests rc $?"
tail -4 gpurun_out/r02k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
ADP_TMA=0 timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02k_c2_tma0.json 2>&1; echo "c2 tma0 rc $?"
timeout 600 python bench.py --workload c2 --steps 20 --warmup 5 --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02k_c2_tma1.json 2>&1; echo "c2 tma1 rc $?"
timeout 300 python tools/phase_trace.py --config c2 > gpurun_out/r02k_phase_c2.txt 2>&1; cat gpurun_out/r02k_phase_c2.txt | head -4
timeout 900 python bench.py --steps 5 --warmup 3 --maid-steps 0 --no-cpu > gpurun_out/r02k_bench.json 2>&1; echo "bench rc $?"
python - <<'PY'
import json
for f in ("gpurun_out/r02k_c2_tma0.json", "gpurun_out/r02k_c2_tma1.json", "gpurun_out/r02k_bench.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], d["ms_per_step"], d["e2e"]["value"])
d = json.loads(open("gpurun_out/r02k_bench.json").read().strip().splitlines()[-1])
c = d["configs"]
print("c5", c["c5"]["value"], c["c5"]["ms_per_solve"], "fft", c["c5_fft"]["value"], c["c5_fft"]["stencil_ms"])
PY
