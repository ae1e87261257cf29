timeout 900 python -m pytest tests/test_gpu_scatter_matmat.py -q -x -k "matmat" > gpurun_out/mm3d.log 2>&1
python tools/mm_diag.py 24 16 >> gpurun_out/mm3d.log 2>&1
python tools/mm_diag.py 24 16 >> gpurun_out/mm3d.log 2>&1
python tools/mm_diag.py 27 16 >> gpurun_out/mm3d.log 2>&1
