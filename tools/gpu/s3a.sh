set -x
mkdir -p gpurun_out/s3a
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s3a/tests.log 2>&1; echo "exit $?" >> gpurun_out/s3a/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a/smoke.log 2>&1; echo "exit $?" >> gpurun_out/s3a/smoke.log
timeout 600 python bench.py > gpurun_out/s3a/bench_c2.json 2> gpurun_out/s3a/bench_c2.err
tail -3 gpurun_out/s3a/tests.log
