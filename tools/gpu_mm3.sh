timeout 900 python -m pytest tests/test_gpu_scatter_matmat.py -q -x -k "matmat" > gpurun_out/mm3c.log 2>&1
for a in 0 37 74 148 296; do echo ahead=$a >> gpurun_out/mm3c.log; CMVG_MM_AHEAD=$a python tools/mm_diag.py 24 16 >> gpurun_out/mm3c.log 2>&1; done
python tools/mm_diag.py 27 16 >> gpurun_out/mm3c.log 2>&1
