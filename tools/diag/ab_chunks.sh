for lib in libhdpstereo libhdp_c12 libhdp_c14; do
  echo "== $lib" >> gpurun_out/abc.log
  HDP_LIB=$PWD/paper_1509_08197_b200/$lib.so python tools/trace_c5.py 5 2>&1 | grep -A6 "^rep 2" | grep -E "aggregate|full" >> gpurun_out/abc.log
  HDP_LIB=$PWD/paper_1509_08197_b200/$lib.so python tools/trace_c5.py 2 2>&1 | grep -A6 "^rep 2" | grep -E "aggregate|full" >> gpurun_out/abc.log
done
