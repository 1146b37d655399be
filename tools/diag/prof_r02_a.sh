# Round-2 profile A: ncu --set full of the HDP prior / HDPF kernels (C4, 8 pairs)
# and of one C5 aggregation call; reports reduced to CSV on the box.
set -x
python tools/stage_times.py --config 4 --batch 8 --levels 5 --size-class full --skip-dense --reps 1 > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_prior|k_grp' -c 4 -o /tmp/hdp_c4 -f python tools/stage_times.py --config 4 --batch 8 --levels 5 --size-class full --skip-dense --reps 1 > gpurun_out/ncu_c4.log 2>&1
ncu -i /tmp/hdp_c4.ncu-rep --page raw --csv > gpurun_out/hdp_c4_raw.csv 2>&1
ncu -i /tmp/hdp_c4.ncu-rep --page source --csv > gpurun_out/hdp_c4_source.csv 2>&1
python tools/trace_full.py 5 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' -s 60 -c 60 -o /tmp/agg_c5 -f python tools/trace_full.py 5 2 > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/agg_c5.ncu-rep --page raw --csv > gpurun_out/agg_c5_raw.csv 2>&1
ls -la /tmp/*.ncu-rep gpurun_out
