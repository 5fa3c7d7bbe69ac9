mkdir -p gpurun_out
python -m pytest tests/test_multitensor_gpu.py tests/test_chunked_psgd_gpu.py tests/test_edge_cases_gpu.py tests/test_distributed_gpu.py tests/test_fullsize_gpu.py -q -m gpu -x > gpurun_out/pt17.log 2>&1
python tools/sweep.py --only powersgd --warmup 3 > gpurun_out/sweep17.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gpt2m6_launches.csv python tools/prof_scheme.py psgd_gpt2m 0 8 2 > /dev/null 2>&1
