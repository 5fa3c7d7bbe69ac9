mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "psgd or multitensor" > gpurun_out/c3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c3_tests.log
timeout 300 python tools/time_rank.py --segs 1000000 > gpurun_out/c3_rank.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_rank_launches.csv python tools/time_rank.py --segs 1000000 --steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rank_quant_kernel -s 2 -c 1 -o gpurun_out/c3_rank_quant python tools/time_rank.py --segs 1000000 --steps 2 > gpurun_out/c3_ncu_rank.log 2>&1
FUSED_ONLY=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:thc_fused_kernel -s 3 -c 1 -o gpurun_out/c3_thc_fused python tools/time_thc.py > gpurun_out/c3_ncu_fused.log 2>&1
