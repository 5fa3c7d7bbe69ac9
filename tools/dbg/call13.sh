mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gpt2m_launches.csv python tools/prof_scheme.py psgd_gpt2m 0 8 2 > gpurun_out/gpt2m.log 2>&1
python -m pytest tests/test_dense_topk_gpu.py -q -m gpu -x > gpurun_out/pt10.log 2>&1
