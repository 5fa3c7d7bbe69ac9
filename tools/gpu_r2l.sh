# round-2 call l: batched TMA fix, DivN in the fused estimate
mkdir -p gpurun_out
timeout 300 python tools/dbg_batched.py > gpurun_out/l_dbg.txt 2>&1
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py tests/test_multitensor_gpu.py tests/test_thc_gpu.py tests/test_fullsize_gpu.py -q > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log
timeout 300 python tools/time_rank.py --scheme psgd_gpt2 --steps 10 > gpurun_out/l_rank_gpt2.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/l_rank_gpt2_launches.csv python tools/time_rank.py --scheme psgd_gpt2 --steps 1 > /dev/null 2>&1
bash tools/ab_thc.sh prev build/libgc_prev.so new paper_2407_01378_b200/libgradcomp_b200.so > gpurun_out/l_ab.txt 2>&1
