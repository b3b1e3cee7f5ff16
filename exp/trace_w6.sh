# device pipeline trace of the W6 experiment build (profiles/r02_cnn_schemes.md), c5
PNPULA_WSLOTS=6 PNPULA_LIB=paper_2511_00870_b200/libpnpula_w6trace.so PNPULA_CNN_TRACE=gpurun_out/trace_w6 \
  timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace_w6.log 2>&1
echo "trace rc=$?"; ls -la gpurun_out/trace_w6*
