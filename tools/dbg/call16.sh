mkdir -p gpurun_out /tmp/prof
python -m pytest tests/test_multitensor_gpu.py tests/test_chunked_psgd_gpu.py tests/test_edge_cases_gpu.py tests/test_distributed_gpu.py -q -m gpu -x > gpurun_out/pt13.log 2>&1
python tools/sweep.py --only powersgd --warmup 2 > gpurun_out/sweep13.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gpt2m4_launches.csv python tools/prof_scheme.py psgd_gpt2m 0 8 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:thc_fused -c 1 -o /tmp/prof/thc_one -f python tools/prof_thc.py 25557032 8 1 1 > /dev/null 2>&1
FN=ILi10ELb1E TOP=40 python tools/ncu_lines.py /tmp/prof/thc_one.ncu-rep paper_2407_01378_b200/libgradcomp_b200.so paper_2407_01378_b200/csrc/gc_thc_fused.cu thc_fused > gpurun_out/thc_lines3.txt 2>&1
