# round 2: new parity tests, c1 tolerance report, reference-suite conformance run
set -x
rm -f gpurun_out/parity_report.jsonl
timeout 1500 python -m pytest tests/test_gpu_k31.py tests/test_gpu_maid2d_p4.py tests/test_gpu_solvers.py -q -rA > gpurun_out/r02c_pytest_new.log 2>&1; echo "new tests rc $?"
tail -5 gpurun_out/r02c_pytest_new.log
timeout 1800 python -m pytest ref_suite_run -q -p no:cacheprovider -rf --durations=15 > gpurun_out/r02c_ref_suite.log 2>&1; echo "ref suite rc $?"
tail -30 gpurun_out/r02c_ref_suite.log
