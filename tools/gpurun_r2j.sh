mkdir -p gpurun_out/r2j
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 140 --log-file gpurun_out/r2j/band_launches.csv python tools/kpp_band.py 1e6 100 1e-9 > gpurun_out/r2j/band_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 140 --log-file gpurun_out/r2j/kpp_c5.csv python tools/km_split.py 5 1 > gpurun_out/r2j/kpp_c5.log 2>&1
