mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_kmeans_pp.py tests/test_gpu_parity.py tests/test_gpu_seqsum.py -q -x > gpurun_out/r2p/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2p/tests.log
for c in 2 5; do timeout 300 python tools/km_split.py $c 2 >> gpurun_out/r2p/km_split.log 2>&1; done
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_rw_wide -s 2 -c 1 -o gpurun_out/r2p/wide_c3 python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2p/ncu_wide.log 2>&1
