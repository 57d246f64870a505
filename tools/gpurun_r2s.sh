mkdir -p gpurun_out/r2s
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2s/gpu_all.log 2>&1; echo "exit $?" >> gpurun_out/r2s/gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2s/bench_c2.json 2> gpurun_out/r2s/bench_c2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2s/bench_ref.json 2> gpurun_out/r2s/bench_ref.err
