mkdir -p gpurun_out/r2q
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shards.py tests/test_gpu_panels.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/r2q/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2q/tests.log
timeout 600 python bench.py --config 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2q/bench_c3.json 2> gpurun_out/r2q/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2q/launches_c3_warm.csv python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2q/launches_c3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k config3 > gpurun_out/r2q/fullsize.log 2>&1; echo "exit $?" >> gpurun_out/r2q/fullsize.log
