# round-2 call i: float4 TMA MtP
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py tests/test_chunked_psgd_gpu.py tests/test_baseline_scale_gpu.py -q -k "psgd or powersgd or mtp or deferred" > gpurun_out/i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/i_tests.log
timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/i_rank_psgd.jsonl 2>&1
GC_PSGD_MTP=cores timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/i_rank_psgd_cores.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/i_rank_psgd_launches.csv python tools/time_rank.py --scheme psgd --steps 1 > /dev/null 2>&1
