"""conftest for the reference-suite conformance run (tools/ref_suite/stage.py):
`adp` and `adp.<module>` resolve to the B200 drop-in, so the
reference's unchanged tests exercise the CUDA path.  The device must be present:
there is no CPU fallback."""
import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_09758_b200 as _b200  # noqa: E402

_MODULES = ("operators", "regularizers", "lower_solvers", "hypergradient", "maid", "problems", "baselines",
            "metrics_io")
for _name in _MODULES:
    sys.modules[f"adp.{_name}"] = getattr(_b200, _name) if hasattr(_b200, _name) else importlib.import_module(
        f"paper_2502_09758_b200.{_name}")
_pkg = types.ModuleType("adp")
_pkg.__path__ = []
_pkg.__dict__.update({k: v for k, v in vars(_b200).items() if not k.startswith("__")})
for _name in _MODULES:
    setattr(_pkg, _name, sys.modules[f"adp.{_name}"])
sys.modules["adp"] = _pkg

# the reference's verify module, loaded as adp.verify so its relative imports bind the drop-in
_here = os.path.dirname(os.path.abspath(__file__))
_spec = importlib.util.spec_from_file_location("adp.verify", os.path.join(_here, "ref_verify.py"))
_verify = importlib.util.module_from_spec(_spec)
_verify.__package__ = "adp"
sys.modules["adp.verify"] = _verify
_spec.loader.exec_module(_verify)
_pkg.verify = _verify
_b200.set_precision("float64", "strict")
