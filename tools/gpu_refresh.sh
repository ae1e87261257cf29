#!/bin/bash
# GPU-box recipe (run under gpurun): bench line, reference arm, launch list of
# the same command, one ncu --set full capture of the gather kernel.  Each
# profiler pass runs only after the plain command exited 0.
set -e
mkdir -p gpurun_out
TAG=${1:-r2}
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log
python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --no-csr --no-pagerank --no-parity --c4-log2 0 \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 \
    -o gpurun_out/prof_gather_$TAG python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --no-csr \
    --no-pagerank --no-parity --c4-log2 0 > gpurun_out/ncu_full_$TAG.log 2>&1
echo refreshed $TAG
