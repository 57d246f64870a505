mkdir -p gpurun_out/r2u
timeout 300 python -m pytest tests/test_gpu_host_numerics.py -q > gpurun_out/r2u/host_numerics.log 2>&1; echo "exit $?" >> gpurun_out/r2u/host_numerics.log
for c in 3 4 5; do timeout 1200 python bench.py --config $c > gpurun_out/r2u/bench_c$c.json 2> gpurun_out/r2u/bench_c$c.err; done
