mkdir -p gpurun_out/r2o
timeout 600 python bench.py --config 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2o/bench_c3.json 2> gpurun_out/r2o/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r2o/launches_c3_warm.csv python tools/prof_spmv.py 3 --cfg 3 > gpurun_out/r2o/launches_c3.log 2>&1
timeout 900 python bench.py --config 2 --devices 0,0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2o/bench_c2_2shards.json 2> gpurun_out/r2o/bench_c2_2shards.err
timeout 900 python bench.py --config 5 --devices 0,0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r2o/bench_c5_2shards.json 2> gpurun_out/r2o/bench_c5_2shards.err
