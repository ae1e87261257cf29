timeout 900 python -m pytest tests/test_gpu_gather.py -q -x -k "host or pageable" > gpurun_out/host14.log 2>&1
python bench.py --no-cpu-baseline --no-pagerank --no-csr > gpurun_out/bench14.json 2> gpurun_out/bench14.log
