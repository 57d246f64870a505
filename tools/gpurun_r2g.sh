mkdir -p gpurun_out/r2g
timeout 300 python tools/kpp_check.py > gpurun_out/r2g/kpp_check.log 2>&1; echo "exit $?" >> gpurun_out/r2g/kpp_check.log
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py tests/test_gpu_kmeans_fused.py tests/test_gpu_kmeans_fast.py -q -x > gpurun_out/r2g/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2g/tests.log
timeout 120 python tools/c1_timing.py > gpurun_out/r2g/c1_timing.log 2>&1
for c in 2 4 5; do timeout 300 python tools/km_split.py $c 2 >> gpurun_out/r2g/km_split.log 2>&1; done
