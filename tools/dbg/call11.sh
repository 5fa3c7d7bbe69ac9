mkdir -p gpurun_out
bash tools/dbg/ab.sh head build/v0/lib.so new paper_2407_01378_b200/libgradcomp_b200.so > gpurun_out/ab3.txt 2>&1
GRADCOMP_B200_LIB=build/v0/lib.so python tools/sweep.py --only topk_ > gpurun_out/sweep8_head.log 2>&1
python tools/sweep.py --only topk_ > gpurun_out/sweep8_new.log 2>&1
python -m pytest tests/test_dense_topk_gpu.py tests/test_thc_gpu.py tests/test_edge_cases_gpu.py -q -m gpu -x > gpurun_out/pt8.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk8_launches.csv python tools/prof_scheme.py topk 110000000 8 14 > /dev/null 2>&1
