ncu --set full --clock-control none --import-source on -k regex:bvf_matmat_kernel -s 2 -c 1 -o gpurun_out/mm_bvf3 -f python tools/mm_diag.py 24 16 > gpurun_out/mmncu.log 2>&1
