mkdir -p gpurun_out/r2h
for sc in 1e-9 1e-6 1e-3 1e-1; do timeout 120 python tools/kpp_band.py 1e6 100 $sc >> gpurun_out/r2h/band.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_kpp|k_seq" -c 140 --log-file gpurun_out/r2h/band_launches.csv python tools/kpp_band.py 1e6 100 1e-9 > gpurun_out/r2h/band_ncu.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_seq_compose -s 40 -c 1 -o gpurun_out/r2h/compose_band python tools/kpp_band.py 1e6 100 1e-9 > gpurun_out/r2h/compose_ncu.log 2>&1
