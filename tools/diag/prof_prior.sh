python tools/prior_one.py > gpurun_out/plain.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:'k_prior' -s 1 -c 1 -o /tmp/prior -f python tools/prior_one.py > gpurun_out/ncu.log 2>&1
ncu -i /tmp/prior.ncu-rep --page raw --csv > gpurun_out/prior_raw.csv 2>&1
ncu -i /tmp/prior.ncu-rep --page source --csv > gpurun_out/prior_src.csv 2>&1
ncu -i /tmp/prior.ncu-rep --page details > gpurun_out/prior_details.txt 2>&1
