# round-2 call e: microbenchmarks (LCG immediates, TMA streaming shapes), deferred tests, K3/signs
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lcg_imm tools/ubench/lcg_imm.cu && timeout 120 /tmp/lcg_imm > gpurun_out/e_lcg_imm.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_stream tools/ubench/tma_stream.cu && timeout 300 /tmp/tma_stream > gpurun_out/e_tma_stream.txt 2>&1
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py -q > gpurun_out/e_deferred.log 2>&1; echo "rc=$?" >> gpurun_out/e_deferred.log
timeout 300 python tools/time_rank.py --scheme thc --steps 10 >> gpurun_out/e_rank.jsonl 2>> gpurun_out/e_rank.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/e_rank_thc_launches.csv python tools/time_rank.py --scheme thc --steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rank_decode_kernel -s 1 -c 1 \
   -o gpurun_out/e_rank_decode -f python tools/time_rank.py --scheme thc --steps 1 > gpurun_out/e_ncu_dec.log 2>&1
