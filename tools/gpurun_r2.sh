set -x
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_kmeans_fused.py tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py -q -x > gpurun_out/r2/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2/tests.log
for c in 2 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/r2/bench_c$c.json 2> gpurun_out/r2/bench_c$c.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rw_step -c 1 -o gpurun_out/r2/spmv_c3 python tools/prof_spmv.py 2 --cfg 3 > gpurun_out/r2/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rw_step -c 1 -o gpurun_out/r2/spmv_c4 python tools/prof_spmv.py 2 --cfg 4 > gpurun_out/r2/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rw_step -c 1 -o gpurun_out/r2/spmv_c5 python tools/prof_spmv.py 2 --cfg 5 > gpurun_out/r2/ncu_c5.log 2>&1
ls -la gpurun_out/r2
