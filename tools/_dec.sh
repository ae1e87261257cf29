mkdir -p gpurun_out
python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/dec_2.log 2>&1
python tools/decode_diag.py 24 2 >> gpurun_out/dec_2.log 2>&1
CMVG_DECODE_CAP=48000 python tools/decode_diag.py 24 2 >> gpurun_out/dec_2.log 2>&1
python tools/decode_diag.py 24 4 >> gpurun_out/dec_2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:bv_ python tools/decode_diag.py 24 2 > gpurun_out/dec_ncu2.log 2>&1
