mkdir -p gpurun_out/r2t
SC_KMEANS_PROFILE=1 timeout 300 python tools/km_split.py 2 2 > gpurun_out/r2t/km_c2_prof.log 2>&1
timeout 120 python -c "
import time,sys
t=time.perf_counter()
import __graft_entry__ as g
g.smoke()
print('smoke wall', time.perf_counter()-t)
" > gpurun_out/r2t/smoke.log 2>&1
CUDA_MODULE_LOADING=LAZY timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t/smoke_lazy.log 2>&1
