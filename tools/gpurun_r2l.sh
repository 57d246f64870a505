mkdir -p gpurun_out/r2l
timeout 300 python tools/kpp_check.py > gpurun_out/r2l/kpp_check.log 2>&1
SC_KPP_STATS=1 timeout 300 python tools/km_split.py 5 1 > gpurun_out/r2l/km_c5.log 2>&1
timeout 300 python tools/km_split.py 4 2 > gpurun_out/r2l/km_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 140 --log-file gpurun_out/r2l/kpp_c5.csv python tools/km_split.py 5 1 > gpurun_out/r2l/kpp_c5.log 2>&1
