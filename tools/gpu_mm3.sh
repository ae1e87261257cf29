timeout 900 python -m pytest tests/test_gpu_scatter_matmat.py tests/test_gpu_device_build.py -q -x > gpurun_out/mm3e.log 2>&1
python tools/mm_diag.py 24 16 >> gpurun_out/mm3e.log 2>&1
python tools/mm_diag.py 27 16 >> gpurun_out/mm3e.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-pagerank --no-csr >> gpurun_out/mm3e.log 2>&1
