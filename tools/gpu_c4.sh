mkdir -p gpurun_out
CMVG_BUILD_TIMING=1 python tools/c4_diag.py 25 3968 > gpurun_out/c4_r2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:bvf_ python tools/c4_diag.py 25 3968 > gpurun_out/c4_launch_r2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 -o gpurun_out/prof_c4_r2 python tools/c4_diag.py 25 3968 > gpurun_out/ncu_c4_r2.log 2>&1
