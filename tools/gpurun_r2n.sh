mkdir -p gpurun_out/r2n
./tools/lat_bench > gpurun_out/r2n/lat.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2n/launches_c3.csv python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2n/launches_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kpp_update_map -s 10 -c 1 -o gpurun_out/r2n/upd_c5 python tools/km_split.py 5 1 > gpurun_out/r2n/upd_ncu.log 2>&1
