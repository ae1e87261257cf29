mkdir -p gpurun_out
T=$1
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/c4_diag.py 24 3968 > gpurun_out/c4_launch_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 -o gpurun_out/prof_c4_$T python tools/c4_diag.py 24 3968 > gpurun_out/ncu_c4_$T.log 2>&1
