mkdir -p gpurun_out/r2y
timeout 300 python tools/kpp_check.py > gpurun_out/r2y/kpp_check.log 2>&1
timeout 300 python tools/km_split.py 5 2 > gpurun_out/r2y/km_c5.log 2>&1
timeout 300 python tools/km_split.py 4 2 > gpurun_out/r2y/km_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_kpp_update_map -s 290 -c 20 --log-file gpurun_out/r2y/upd.csv python tools/km_split.py 5 1 > gpurun_out/r2y/upd.log 2>&1
