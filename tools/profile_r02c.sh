# Round-2 (final) profile set, run under gpurun; summaries are copied to profiles/ (r02c_*):
#  1. launch list (device time per launch) of the headline bench command (C5)
#  2. ncu --set full of one C5 and one C2 hdp_aggregate_wta call (DRAM traffic per call ->
#     profiles/r02_traffic_{c5,c2}.json, the bench's roofline.traffic)
#  3. ncu --set full of the prior (C4 level 0: byte-record filter; level 1: f32 records)
set -x
python bench.py --steps 2 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_bench_c5.csv \
    python bench.py --steps 2 --warmup 3 --legs none --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/trace_full.py 5 2 > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_pack_rec8|k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' \
    -c 200 -o /tmp/agg_c5 -f python tools/trace_full.py 5 2 > gpurun_out/ncu_c5.log 2>&1
ncu -i /tmp/agg_c5.ncu-rep --page raw --csv > gpurun_out/r02c_agg_c5_raw.csv 2>&1
python tools/trace_full.py 2 2 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none -k regex:'k_pack_rec8|k_ecost|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' \
    -c 200 -o /tmp/agg_c2 -f python tools/trace_full.py 2 2 > gpurun_out/ncu_c2.log 2>&1
ncu -i /tmp/agg_c2.ncu-rep --page raw --csv > gpurun_out/r02c_agg_c2_raw.csv 2>&1
for lv in 0 1; do
python tools/prior_one.py $lv > gpurun_out/plain_prior.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_prior' -s 1 -c 1 -o gpurun_out/r02c_prior_l$lv -f python tools/prior_one.py $lv > gpurun_out/ncu_prior.log 2>&1
ncu -i gpurun_out/r02c_prior_l$lv.ncu-rep --page details > gpurun_out/r02c_prior_c4l${lv}_details.txt 2>&1
python tools/ncu_stalls.py gpurun_out/r02c_prior_l$lv.ncu-rep 12 > gpurun_out/r02c_prior_c4l${lv}_stalls.txt 2>&1
done
ls -la gpurun_out
