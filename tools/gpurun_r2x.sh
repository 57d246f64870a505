mkdir -p gpurun_out/r2x
timeout 300 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2x/multi.log 2>&1; echo "exit $?" >> gpurun_out/r2x/multi.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kpp_update_map -s 300 -c 1 -o gpurun_out/r2x/upd_c5 python tools/km_split.py 5 1 > gpurun_out/r2x/upd_ncu.log 2>&1
