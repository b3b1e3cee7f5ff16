# Device pipeline trace of the first CNN evaluation (CTA 0, its first work unit), c5: the
# -DPNPULA_TRACE=1 build (libpnpula_trace.so, built here); analyse with tools_trace.py
PNPULA_LIB=paper_2511_00870_b200/libpnpula_trace.so PNPULA_CNN_TRACE=gpurun_out/trace_c5 \
  timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace_c5.log 2>&1
echo "trace rc=$?"; ls -la gpurun_out/trace_c5*
