mkdir -p gpurun_out/s3c
O=gpurun_out/s3c
timeout 900 python -m pytest tests/test_gpu_upload.py tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_shards.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
timeout 600 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
SC_STAGE_OFF=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_c2_nostage.json 2> $O/bench_c2_nostage.err
timeout 300 python tools/step_time.py 3 > $O/c3.log 2>&1
timeout 300 python tools/step_time.py 4 > $O/c4.log 2>&1
tail -2 $O/tests.log
