python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "wide or c5 or dense" > gpurun_out/t.log 2>&1
HDP_WIDE_MIN=64 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_gpu_configs.py -q -p no:cacheprovider -k "dense or baseline or c2_every" >> gpurun_out/t.log 2>&1
python tools/trace_c5.py 5 > gpurun_out/tr_new.log 2>&1
HDP_WIDE_MIN=0 python tools/trace_c5.py 5 > gpurun_out/tr_old.log 2>&1
HDP_WIDE_MIN=64 python tools/trace_c5.py 2 > gpurun_out/tr_new2.log 2>&1
HDP_WIDE_MIN=0 python tools/trace_c5.py 2 > gpurun_out/tr_old2.log 2>&1
python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "giant" >> gpurun_out/t.log 2>&1
python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "giant" >> gpurun_out/t.log 2>&1
