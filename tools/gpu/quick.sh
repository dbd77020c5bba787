# quick A/B: step-path parity tests + c3 main line only.  usage: bash tools/gpu/quick.sh TAG
set -x
T=${1:-q}
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_lockstep.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extra --maid-steps 0 --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc $?"
python - <<PY
import json
d = json.loads(open("gpurun_out/${T}_bench.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("c3", round(d["value"],4), "ms/step", round(d["ms_per_step"],2), "e2e", round(d["e2e"]["value"],4), "launches", d["gpu_launches"])
print("dominant", r["kernel"], round(r["achieved"],3), round(r["frac"],4), "launch_ms", round(r["launch_ms"],4), "whole", round(r["whole_step"]["frac"],4), d["clocks"])
PY
tail -2 gpurun_out/${T}_bench.err
