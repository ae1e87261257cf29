#!/bin/bash
# GPU-box recipe (run under gpurun): one ncu --set full capture each of the
# scatter (C2), the multi-vector product (BV-F kernel) (C5 shape at n = 2^24) and the fused
# PageRank step (C3, n = 2^26), after each plain command exited 0.
set -e
mkdir -p gpurun_out
TAG=${1:-r1}
python tools/ab_gather.py --form scatter --rounds 1 paper_1708_07271_b200/libcmvg.so > gpurun_out/others_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvt_scatter_kernel -s 3 -c 1 \
    -o gpurun_out/prof_scatter_$TAG python tools/ab_gather.py --form scatter --rounds 1 --reps 2 paper_1708_07271_b200/libcmvg.so >> gpurun_out/others_$TAG.log 2>&1
python tools/mm_diag.py 24 16 >> gpurun_out/others_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_matmat_kernel -s 2 -c 1 \
    -o gpurun_out/prof_matmat_$TAG python tools/mm_diag.py 24 16 >> gpurun_out/others_$TAG.log 2>&1
python tools/pr_diag.py 26 20 >> gpurun_out/others_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 4 -c 1 \
    --graph-profiling node -o gpurun_out/prof_pagerank_$TAG python tools/pr_diag.py 26 5 >> gpurun_out/others_$TAG.log 2>&1
echo done $TAG
