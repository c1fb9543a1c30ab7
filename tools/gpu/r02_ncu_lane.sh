ncu --set full --clock-control none --import-source on -k regex:k_vnd_lane -c 1 -o gpurun_out/r02_lane_c3b python tools/profile_vnd.py c3 > gpurun_out/ncu_lane.log 2>&1
python tools/product_work.py c3 > gpurun_out/product_work.log 2>&1
