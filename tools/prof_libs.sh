# ncu --set full of the gather kernel for each library (dev tool, GPU box)
mkdir -p gpurun_out
for lib in "$@"; do
  t=$(basename $lib .so)
  CMVG_LIBRARY=$PWD/$lib ncu --set full --import-source on --clock-control none -k regex:bvf_gather_kernel -s 3 -c 1 \
    -o gpurun_out/prof_$t python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-clocks --no-csr --no-pagerank --no-parity \
    > gpurun_out/ncu_$t.log 2>&1
done
