mkdir -p gpurun_out
python -m pytest tests/test_dense_topk_gpu.py tests/test_edge_cases_gpu.py tests/test_distributed_gpu.py tests/test_multitensor_gpu.py tests/test_payloads.py tests/test_fullsize_gpu.py -q -m gpu -x > gpurun_out/pt18.log 2>&1
python tools/sweep.py --only topk_,powersgd_r4_gpt2m > gpurun_out/sweep18.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk10_launches.csv python tools/prof_scheme.py topk 110000000 8 3 > /dev/null 2>&1
