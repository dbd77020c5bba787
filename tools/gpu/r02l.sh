set -x
timeout 900 python -m pytest tests/test_gpu_step.py -x -q -rA > gpurun_out/r02l_step.log 2>&1; echo "step rc $?"
tail -20 gpurun_out/r02l_step.log
ADP_STEP=0 timeout 600 python bench.py --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02l_bench_step0.json 2>&1; echo "b0 rc $?"
ADP_STEP=1 timeout 600 python bench.py --no-extra --maid-steps 0 --no-cpu > gpurun_out/r02l_bench_step1.json 2>&1; echo "b1 rc $?"
python - <<'PY'
import json
for f in ("gpurun_out/r02l_bench_step0.json", "gpurun_out/r02l_bench_step1.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["e2e"]["value"])
    except Exception as e:
        print(f, "failed", e)
PY
tail -5 gpurun_out/r02l_bench_step1.json
