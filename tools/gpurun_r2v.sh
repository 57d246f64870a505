mkdir -p gpurun_out/r2v
timeout 600 python -m pytest tests/test_gpu_shards.py tests/test_gpu_multi.py tests/test_gpu_panels.py -q -x > gpurun_out/r2v/tests.log 2>&1; echo "exit $?" >> gpurun_out/r2v/tests.log
for c in 3 5; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --sharded --config $c --steps 5 --warmup 3 > gpurun_out/r2v/strong_c$c.json 2> gpurun_out/r2v/strong_c$c.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 1 --sharded > gpurun_out/r2v/weak_c2.json 2> gpurun_out/r2v/weak_c2.err
