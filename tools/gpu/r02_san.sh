timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02_memcheck.log
