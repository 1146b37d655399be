# Round profile: bench line, bench launch list, full ncu capture of one
# aggregation call (C2 dense).  Outputs in gpurun_out/ (copy to profiles/).
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:'k_ecost_range|k_up_chunk|k_down_chunk|k_seg_up|k_seg_down|k_keys_finish' \
    -o gpurun_out/agg_full_c2 -f python tools/trace_full.py 2 1 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_launches.py gpurun_out/agg_full_c2.ncu-rep > gpurun_out/agg_full_c2.txt 2>&1
python tools/ncu_traffic.py gpurun_out/agg_full_c2.ncu-rep > gpurun_out/aggregate_traffic.json 2>&1
