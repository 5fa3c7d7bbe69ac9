mkdir -p gpurun_out
python -m pytest tests/test_multitensor_gpu.py tests/test_chunked_psgd_gpu.py tests/test_edge_cases_gpu.py tests/test_distributed_gpu.py tests/test_fullsize_gpu.py -q -m gpu -x > gpurun_out/pt14.log 2>&1
python tools/sweep.py --only powersgd --warmup 2 > gpurun_out/sweep14.log 2>&1
for v in h8 h16; do GRADCOMP_B200_LIB=build/$v/lib.so python tools/sweep.py --only topk_ > gpurun_out/sweep14_$v.log 2>&1; done
python tools/sweep.py --only topk_ > gpurun_out/sweep14_h4.log 2>&1
