mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py tests/test_gpu_kmeans_fused.py tests/test_gpu_seqsum.py tests/test_gpu_metrics.py tests/test_gpu_block.py -q -x > gpurun_out/r2f/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2f/tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "config3 or config4" > gpurun_out/r2f/fullsize.log 2>&1; echo "exit $?" >> gpurun_out/r2f/fullsize.log
for c in 2 4 5; do timeout 600 python tools/km_split.py $c 2 >> gpurun_out/r2f/km_split.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/launches_c3.csv python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2f/launches_c3.log 2>&1
