for lib in _ab/libmm64.so _ab/libmm32.so; do CMVG_LIBRARY=$PWD/$lib python tools/mm_diag.py 25 16; done > gpurun_out/ab_mm.log 2>&1
for lib in _ab/libmm64.so _ab/libmm32.so; do CMVG_LIBRARY=$PWD/$lib python tools/mm_diag.py 27 16; done >> gpurun_out/ab_mm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scatter_matmat.py tests/test_gpu_fullsize.py -q -k "matmat or c5" >> gpurun_out/ab_mm.log 2>&1
