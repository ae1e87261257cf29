CMVG_BUILD_TIMING=1 python tools/create_time.py 24 > gpurun_out/bt_c2.json 2> gpurun_out/bt_c2.log
CMVG_BUILD_TIMING=1 python tools/c4_diag.py 25 3968 > gpurun_out/bt_c4.log 2>&1
