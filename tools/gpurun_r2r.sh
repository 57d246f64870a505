mkdir -p gpurun_out/r2r
timeout 600 python tools/c4_delta_probe.py 4 > gpurun_out/r2r/c4_delta.log 2>&1
SC_KMEANS_PROFILE=1 timeout 300 python tools/km_split.py 4 1 > gpurun_out/r2r/km_c4_prof.log 2>&1
SC_KMEANS_PROFILE=1 timeout 300 python tools/km_split.py 3 1 > gpurun_out/r2r/km_c3_prof.log 2>&1
