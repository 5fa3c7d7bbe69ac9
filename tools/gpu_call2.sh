mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "nccl or distributed or ddp or per_rank" > gpurun_out/c2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c2_tests.log
timeout 600 python tools/time_rank.py > gpurun_out/c2_rank_350m.jsonl 2> gpurun_out/c2_rank.err
timeout 600 python tools/time_rank.py --d 25557032 --n 8 --segs 512,1024,4096,100000 > gpurun_out/c2_rank_cfg2.jsonl 2>> gpurun_out/c2_rank.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c2_rank_launches.csv python tools/time_rank.py --segs 4096 --steps 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rank_quant_kernel -s 20 -c 1 -o gpurun_out/c2_rank_quant python tools/time_rank.py --segs 100000 --steps 2 > gpurun_out/c2_ncu.log 2>&1
