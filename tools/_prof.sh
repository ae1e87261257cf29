set -x
mkdir -p gpurun_out
T=$1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 -o gpurun_out/prof_c4_$T python tools/c4_diag.py 24 3968 > gpurun_out/ncu_c4_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 -o gpurun_out/prof_c2_$T python tools/ab_gather.py --rounds 1 --reps 3 paper_1708_07271_b200/libcmvg.so > gpurun_out/ncu_c2_$T.log 2>&1
