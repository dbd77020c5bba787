# A/B over an environment knob: bash tools/gpu/ab_env.sh TAG VAR v1 v2 ...
# per value: the step-path parity tests + the c3 main line (no side lines)
T=$1; V=$2; shift 2
for val in "$@"; do
  export $V=$val
  timeout 600 python -m pytest tests/test_gpu_step.py -m gpu -q -x > gpurun_out/${T}_${val}_pytest.log 2>&1; echo "$V=$val pytest rc $? $(tail -1 gpurun_out/${T}_${val}_pytest.log)"
  timeout 600 python bench.py --steps 5 --warmup 3 --no-extra --maid-steps 0 --no-cpu > gpurun_out/${T}_${val}_bench.json 2> gpurun_out/${T}_${val}_bench.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/${T}_${val}_bench.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("$V=$val c3", round(d["value"],4), "ms/step", round(d["ms_per_step"],2), "e2e", round(d["e2e"]["value"],4), "dominant", r["kernel"], round(r["frac"],4), "launch_ms", round(r["launch_ms"],4), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
