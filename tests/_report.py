"""Measured parity values (first divergence, error magnitudes, band
statistics) appended to gpurun_out/parity_report.jsonl when that directory
exists (the GPU box run), so the numbers behind each tolerance are kept."""
import json
import os

_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


def report(test: str, **values):
    if not os.path.isdir(_DIR):
        return
    with open(os.path.join(_DIR, "parity_report.jsonl"), "a") as f:
        f.write(json.dumps({"test": test, **{k: (float(v) if hasattr(v, "__float__") and not isinstance(v, (int, bool))
                                                 else v) for k, v in values.items()}}) + "\n")
