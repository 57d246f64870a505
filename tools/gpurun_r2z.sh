mkdir -p gpurun_out/r2z
for c in 5 3 4; do for h in 0 16 17 20; do SC_FAR_HINT=$h timeout 300 python tools/step_time.py $c >> gpurun_out/r2z/far.log 2>&1; done; done
