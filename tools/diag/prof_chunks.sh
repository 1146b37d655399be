# ncu --set full (with source) of the largest launch of each aggregation kernel at C5 (second call)
set -x
python tools/trace_full.py 5 2 > gpurun_out/plain_c5.log 2>&1
for k in "k_up_chunk:16" "k_down_chunk:16" "k_seg_up:15" "k_seg_down:15"; do
  n=${k%%:*}; s=${k#*:}
  ncu --set full --import-source on --clock-control none -k regex:"$n\b" -s $s -c 1 -o gpurun_out/$n -f \
      python tools/trace_full.py 5 2 > gpurun_out/ncu_$n.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
