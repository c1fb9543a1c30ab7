for v in 0 8; do for w in "2 400" "2 20000" "128 200"; do echo "variant $v" >> gpurun_out/r02_gv_skip.log; RL_VARIANT=$v python tools/profile_gvns.py $w >> gpurun_out/r02_gv_skip.log 2>&1; done; done
