# Round-2 profile set (run under gpurun; outputs in gpurun_out/, copied to profiles/):
#  1. launch list of the headline bench command (C5, device time per launch)
#  2. ncu --set full of one C5 and one C2 aggregation call (DRAM traffic per call)
#  3. ncu --set full of the HDPF kernel (C2 level 0) and the prior (C4 level 0)
set -x
python bench.py --steps 2 --warmup 1 --legs none --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_c5.csv \
    python bench.py --steps 2 --warmup 1 --legs none --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/trace_full.py 5 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish|k_fill_cols' \
    -s 60 -c 60 -o /tmp/agg_c5 -f python tools/trace_full.py 5 2 > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/agg_c5.ncu-rep --page raw --csv > gpurun_out/r02_agg_c5_raw.csv 2>&1
python tools/trace_full.py 2 3 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish|k_fill_cols' \
    -s 80 -c 80 -o /tmp/agg_c2 -f python tools/trace_full.py 2 3 > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/agg_c2.ncu-rep --page raw --csv > gpurun_out/r02_agg_c2_raw.csv 2>&1
python tools/stage_times.py --config 2 --skip-dense --reps 1 > gpurun_out/plain_hdp.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_grp' -s 2 -c 1 -o /tmp/grp -f \
    python tools/stage_times.py --config 2 --skip-dense --reps 1 > gpurun_out/ncu_grp.log 2>&1
ncu -i /tmp/grp.ncu-rep --page details > gpurun_out/r02_grp_details.txt 2>&1
python tools/prior_one.py 0 > gpurun_out/plain_prior.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_prior' -s 1 -c 1 -o /tmp/prior0 -f python tools/prior_one.py 0 > gpurun_out/ncu_prior.log 2>&1
ncu -i /tmp/prior0.ncu-rep --page details > gpurun_out/r02_prior_c4l0_details.txt 2>&1
ls -la gpurun_out
