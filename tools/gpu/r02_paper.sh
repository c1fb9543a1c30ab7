python tools/paper_scale.py gpu 8 60 > gpurun_out/r02_paper_scale.log 2>&1
