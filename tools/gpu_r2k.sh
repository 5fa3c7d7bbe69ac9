# round-2 call k: batched TMA + deferred PowerSGD (GPT-2-medium), THC fused source-level capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py tests/test_multitensor_gpu.py tests/test_baseline_scale_gpu.py -q -k "psgd or powersgd or deferred or mtp or gpt2 or multitensor" > gpurun_out/k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k_tests.log
timeout 300 python tools/time_rank.py --scheme psgd_gpt2 --steps 10 > gpurun_out/k_rank_gpt2.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/k_rank_gpt2_launches.csv python tools/time_rank.py --scheme psgd_gpt2 --steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:thc_fused_kernel -s 1 -c 1 \
   -o gpurun_out/k_thc_fused -f python tools/prof_thc.py 25557032 8 1 2 > gpurun_out/k_ncu_fused.log 2>&1
