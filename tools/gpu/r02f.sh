# compute-sanitizer memcheck on small invocations of every kernel family
set -x
timeout 600 python tools/sanitize_case.py > gpurun_out/r02f_plain.log 2>&1; echo "plain rc $?"
tail -3 gpurun_out/r02f_plain.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_case.py > gpurun_out/r02f_memcheck.log 2>&1; echo "memcheck rc $?"
tail -8 gpurun_out/r02f_memcheck.log
