"""Stage the reference's OWN unit tests and verify suites for a conformance run
against the drop-in.

    python tools/ref_suite/stage.py          # in the build container (needs /root/reference)

Copies /root/reference/pkg/tests/test_{operators,regularizers,lower_solvers,
hypergradient,maid,problems,baselines,metrics_io}.py and
/root/reference/pkg/src/adp/verify.py UNCHANGED into ref_suite_run/ (git-ignored,
NOT gpurun-ignored, so it travels to the GPU box for one run and is deleted
afterwards; no reference source enters the repository history), next to
tools/ref_suite/conftest_alias.py (our own) as conftest.py.  The alias conftest
points `adp` and `adp.<module>` at paper_2502_09758_b200 before the tests
import anything, so the reference's tests call the B200 path.

Run on the GPU box:  python -m pytest ref_suite_run -q -p no:cacheprovider
"""
import os
import shutil

REF = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(ROOT, "ref_suite_run")
MODULES = ("operators", "regularizers", "lower_solvers", "hypergradient", "maid", "problems", "baselines",
           "metrics_io")

if __name__ == "__main__":
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    for m in MODULES:
        shutil.copy(os.path.join(REF, "tests", f"test_{m}.py"), OUT)
    shutil.copy(os.path.join(REF, "src", "adp", "verify.py"), os.path.join(OUT, "ref_verify.py"))
    shutil.copy(os.path.join(HERE, "conftest_alias.py"), os.path.join(OUT, "conftest.py"))
    shutil.copy(os.path.join(HERE, "test_verify_suites.py"), OUT)
    print("staged", sorted(os.listdir(OUT)))
