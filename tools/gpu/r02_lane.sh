python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/r02_lane_tests.log
for r in 2 4 8 12; do RL_LANE_REFILL=$r python tools/ab_vnd.py c3 0 >> gpurun_out/r02_lane_ab.log 2>&1; echo "refill $r" >> gpurun_out/r02_lane_ab.log; done
python tools/ab_vnd.py c3 32 >> gpurun_out/r02_lane_ab.log 2>&1
REMLOT_B200_LIB=$PWD/paper_1704_05132_b200/_lib/libremlot_b200_walkstats.so python tools/lane_stats.py c3 > gpurun_out/r02_lanestats.log 2>&1
