mkdir -p gpurun_out/r2i
for sc in 1e-9 1e-6; do timeout 120 python tools/kpp_band.py 1e6 100 $sc >> gpurun_out/r2i/band.log 2>&1; done
for sc in 1e-9 1e-3; do timeout 300 python tools/kpp_band.py 2e5 50 $sc check >> gpurun_out/r2i/band.log 2>&1; done
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py tests/test_gpu_kmeans_fused.py tests/test_gpu_seqsum.py tests/test_gpu_metrics.py -q -x > gpurun_out/r2i/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2i/tests.log
for c in 2 4 5; do timeout 300 python tools/km_split.py $c 1 >> gpurun_out/r2i/km_split.log 2>&1; done
