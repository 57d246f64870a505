mkdir -p gpurun_out/r2m
timeout 300 python tools/kpp_check.py > gpurun_out/r2m/kpp_check.log 2>&1
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py tests/test_gpu_kmeans_fused.py tests/test_gpu_seqsum.py tests/test_gpu_metrics.py tests/test_gpu_block.py -q -x > gpurun_out/r2m/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2m/tests.log
for c in 2 4 5; do timeout 300 python tools/km_split.py $c 2 >> gpurun_out/r2m/km_split.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 140 --log-file gpurun_out/r2m/kpp_c5.csv python tools/km_split.py 5 1 > gpurun_out/r2m/kpp_c5.log 2>&1
