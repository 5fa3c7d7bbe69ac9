mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk9_launches.csv python tools/prof_scheme.py topk 110000000 8 4 > /dev/null 2>&1
python tools/sweep.py --only topk_ > gpurun_out/sweep9.log 2>&1
GRADCOMP_B200_LIB=build/s3/lib.so python tools/sweep.py --only powersgd_r4_cfg4 --warmup 2 > gpurun_out/sweep9_s3.log 2>&1
python tools/sweep.py --only powersgd_r4_cfg4 --warmup 2 > gpurun_out/sweep9_s2.log 2>&1
python -m pytest tests/test_dense_topk_gpu.py -q -m gpu -x > gpurun_out/pt9.log 2>&1
