python tools/lpt_probe.py > gpurun_out/r02_lpt.log 2>&1
for w in 4 6 8 10; do RL_LANE_WARPS_PER_SM=$w python tools/ab_vnd.py c3 0 >> gpurun_out/r02_lpt.log 2>&1; echo "warps/SM $w" >> gpurun_out/r02_lpt.log; done
