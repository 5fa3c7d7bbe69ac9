mkdir -p gpurun_out
python -m pytest tests/test_dense_topk_gpu.py tests/test_chunked_psgd_gpu.py tests/test_multitensor_gpu.py tests/test_distributed_gpu.py tests/test_edge_cases_gpu.py tests/test_ddp_gpu.py -q -m gpu -x > gpurun_out/pt15.log 2>&1
python tools/sweep.py --only dense,topkc,powersgd_r4_cfg4 --warmup 3 > gpurun_out/sweep15.log 2>&1
