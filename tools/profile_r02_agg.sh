# ncu --set full of every aggregation launch of two C5 calls and two C2 calls
# (tools/ncu_call_summary.py picks one complete call); CSV only (size limit)
python tools/trace_full.py 5 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' \
    -c 200 -o /tmp/agg_c5 -f python tools/trace_full.py 5 2 > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/agg_c5.ncu-rep --page raw --csv > gpurun_out/r02_agg_c5_raw.csv 2>&1
python tools/trace_full.py 2 2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' \
    -c 200 -o /tmp/agg_c2 -f python tools/trace_full.py 2 2 > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/agg_c2.ncu-rep --page raw --csv > gpurun_out/r02_agg_c2_raw.csv 2>&1
