mkdir -p gpurun_out
python tools/decode_diag.py 24 2 > gpurun_out/dec_r2.log 2>&1
python tools/decode_diag.py 25 4 >> gpurun_out/dec_r2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:bv_ python tools/decode_diag.py 24 2 > gpurun_out/dec_ncu_r2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bv_decode_tiles -s 1 -c 1 -o gpurun_out/prof_dec_r2 python tools/decode_diag.py 24 2 > gpurun_out/dec_ncufull_r2.log 2>&1
