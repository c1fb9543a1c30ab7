timeout 2400 bash tools/debug_checks.sh > gpurun_out/r02_debug_checks.log 2>&1; echo "rc=$?" >> gpurun_out/r02_debug_checks.log
