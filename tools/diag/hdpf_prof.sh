HDP_LIB=$PWD/paper_1509_08197_b200/libhdp_prof.so python tools/stage_times.py --config 2 --skip-dense --reps 1 > gpurun_out/hdpf_prof.log 2>&1
HDP_LIB=$PWD/paper_1509_08197_b200/libhdp_prof.so python tools/stage_times.py --config 4 --batch 8 --levels 5 --size-class full --skip-dense --reps 1 >> gpurun_out/hdpf_prof.log 2>&1
python tools/stage_times.py --config 2 --skip-dense --reps 2 > gpurun_out/st_c2.log 2>&1
