mkdir -p gpurun_out/r2w
timeout 300 python -m pytest tests/test_gpu_shards.py -q -k device_csr > gpurun_out/r2w/shard_test.log 2>&1; echo "exit $?" >> gpurun_out/r2w/shard_test.log
for t in 4096 8192 16384; do SC_CS_TILE=$t SC_KMEANS_PROFILE=1 timeout 300 python tools/km_split.py 4 1 2>&1 | grep -v "^\[kpp\]\|fused" | tail -3 >> gpurun_out/r2w/km_c4_tiles.log; echo "tile $t" >> gpurun_out/r2w/km_c4_tiles.log; done
SC_CS_TILE=16384 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kmeans_sorted.py -q -x > gpurun_out/r2w/tests16k.log 2>&1; echo "exit $?" >> gpurun_out/r2w/tests16k.log
