mkdir -p gpurun_out/r2d
timeout 300 python tools/c1_timing.py > gpurun_out/r2d/c1_timing.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rw_wide -c 1 -o gpurun_out/r2d/wide_c3 python tools/prof_spmv.py 2 --cfg 3 > gpurun_out/r2d/ncu_wide.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 200 --log-file gpurun_out/r2d/kpp_c5.csv python tools/km_split.py 5 1 > gpurun_out/r2d/kpp_c5.log 2>&1
python - > gpurun_out/r2d/c3_degrees.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2310_10939_b200.generate import config_device_csr
with config_device_csr(3) as d:
    g = d.download().graph
deg = np.diff(g.row_offsets)
print("max deg", deg.max(), "rows>256", (deg > 256).sum(), "entries in rows>256", deg[deg > 256].sum(), "nnz", g.nnz)
print("top degrees", np.sort(deg)[-20:])
PY
