out=paper_1704_05132_b200/_lib/libremlot_b200_walkstats.so
REMLOT_B200_LIB=$PWD/$out python tools/lane_stats.py c3 > gpurun_out/r02_lanestats.log 2>&1
