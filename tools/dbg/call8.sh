mkdir -p /tmp/prof gpurun_out
python -m pytest tests/test_chunked_psgd_gpu.py tests/test_multitensor_gpu.py tests/test_edge_cases_gpu.py tests/test_ddp_gpu.py -q -m gpu -x > gpurun_out/pt5.log 2>&1
python tools/sweep.py --only powersgd > gpurun_out/sweep5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/topk5_launches.csv python tools/prof_scheme.py topk 110000000 8 14 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:thc_fused -c 1 -o /tmp/prof/thc_one -f python tools/prof_thc.py 25557032 8 1 1 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/prof/thc_one.ncu-rep > gpurun_out/thc_full2.txt 2>&1
cp /tmp/prof/thc_one.ncu-rep gpurun_out/thc_one2.ncu-rep
