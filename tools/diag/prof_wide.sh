python tools/trace_c5.py 5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:'k_wide|k_keys' --csv --log-file gpurun_out/wide_launches.csv python tools/trace_c5.py 5 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_wide_up$|k_wide_upEN|k_wide_up\b' -s 14 -c 1 -o /tmp/wup -f python tools/trace_c5.py 5 > gpurun_out/ncu2.log 2>&1
ncu -i /tmp/wup.ncu-rep --page details > gpurun_out/wup_details.txt 2>&1
ncu -i /tmp/wup.ncu-rep --page source --csv > gpurun_out/wup_src.csv 2>&1
