mkdir -p gpurun_out
python -m pytest tests/test_dense_topk_gpu.py tests/test_edge_cases_gpu.py tests/test_chunked_psgd_gpu.py tests/test_distributed_gpu.py tests/test_payloads.py -q -m gpu -x > gpurun_out/pt7.log 2>&1
python tools/sweep.py --only topk > gpurun_out/sweep7.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk7_launches.csv python tools/prof_scheme.py topk 110000000 8 14 > /dev/null 2>&1
