mkdir -p gpurun_out
python tools/c4_diag.py 24 3968 > gpurun_out/c4d_3.log 2>&1
python tools/c4_diag.py 24 2048 >> gpurun_out/c4d_3.log 2>&1
python tools/ab_gather.py --rounds 1 --dtype f32 paper_1708_07271_b200/libcmvg.so >> gpurun_out/c4d_3.log 2>&1
python -m pytest tests/test_gpu_gather.py tests/test_bvf_layout.py -x -q >> gpurun_out/c4d_3.log 2>&1
