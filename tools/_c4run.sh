set -x
mkdir -p gpurun_out
python tools/c4_diag.py 24 3968 > gpurun_out/c4d_2.log 2>&1
python tools/c4_diag.py 24 1536 >> gpurun_out/c4d_2.log 2>&1
python tools/c4_diag.py 24 2048 >> gpurun_out/c4d_2.log 2>&1
python tools/ab_gather.py --rounds 1 paper_1708_07271_b200/libcmvg.so >> gpurun_out/c4d_2.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_c4_2.log 2>&1
