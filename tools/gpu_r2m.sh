# round-2 call m: per-rank THC K2 at four CTAs per SM
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_nccl_gpu.py tests/test_baseline_scale_gpu.py tests/test_distributed_gpu.py -q -k "rotated or thc or quant or per_rank" > gpurun_out/m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/m_tests.log
timeout 300 python tools/time_rank.py --scheme thc --steps 10 > gpurun_out/m_rank_thc.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/m_rank_thc_launches.csv python tools/time_rank.py --scheme thc --steps 1 > /dev/null 2>&1
