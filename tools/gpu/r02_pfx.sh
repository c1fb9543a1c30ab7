python -m pytest tests/test_gpu_gvns.py tests/test_gpu_pins.py tests/test_gpu_api.py -q -x 2>&1 | tail -4 > gpurun_out/r02_pfx_tests.log
for lib in base new; do
  if [ $lib = base ]; then export REMLOT_B200_LIB=paper_1704_05132_b200/_lib/libremlot_b200_base.so; else unset REMLOT_B200_LIB; fi
  for w in "2 400" "2 20000" "128 200" "1024 40"; do echo -n "$lib " >> gpurun_out/r02_pfx_rate.log; python tools/profile_gvns.py $w >> gpurun_out/r02_pfx_rate.log 2>&1; done
done
unset REMLOT_B200_LIB
timeout 600 python tools/tail_probe.py c4 > gpurun_out/r02_tail.log 2>&1
timeout 600 python tools/tail_probe.py c3 >> gpurun_out/r02_tail.log 2>&1
