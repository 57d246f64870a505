set -x
mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/r2b/multi.log 2>&1; echo "exit $?" >> gpurun_out/r2b/multi.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/r2b/gpu_all.log 2>&1; echo "exit $?" >> gpurun_out/r2b/gpu_all.log
timeout 900 python bench.py --config 5 > gpurun_out/r2b/bench_c5.json 2> gpurun_out/r2b/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b/launches_c3.csv python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2b/launches_c3.log 2>&1
