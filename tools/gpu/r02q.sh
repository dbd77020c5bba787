set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02q_pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r02q_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err; echo "bench rc $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r02q_bench.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("c3", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "launches", d["gpu_launches"])
print("roof", r["kernel"], r["achieved"], r["frac"], r["launch_ms"], r["kernel_share_of_step"], r["whole_step"]["frac"], r["strict_ceiling"])
print("maid", d["maid"]["c1"]["value"], d["maid"]["c2"]["value"])
c = d["configs"]
print("c2", c["c2"]["value"], "c4", c["c4"]["value"], "c5", c["c5"]["value"], "fft", c["c5_fft"]["value"])
print("modes", d["other_modes"])
PY
tail -3 gpurun_out/r02q_bench.err
