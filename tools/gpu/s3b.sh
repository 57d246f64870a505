mkdir -p gpurun_out/s3b
O=gpurun_out/s3b
for c in 3 4; do
  timeout 300 python tools/step_time.py $c > $O/base_c$c.log 2>&1
  for v in w5 w6 w6u6; do SC_LIB_PATH=tools/variants/$v/libsc_b200.so timeout 300 python tools/step_time.py $c > $O/${v}_c$c.log 2>&1; done
done
timeout 400 python tools/step_time.py 5 > $O/base_c5.log 2>&1
SC_LIB_PATH=tools/variants/u8/libsc_b200.so timeout 400 python tools/step_time.py 5 > $O/u8_c5.log 2>&1
timeout 300 python tools/km_split.py 2 3 > $O/km_c2.log 2>&1
timeout 300 python tools/e2e_breakdown.py 2 3 > $O/e2e_c2.log 2>&1
grep -h "per-step" $O/*.log
