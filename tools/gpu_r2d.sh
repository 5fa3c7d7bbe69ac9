# round-2 call d: 5-stage TMA MQ, bar kernels, K3 table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py -q > gpurun_out/d_deferred.log 2>&1; echo "rc=$?" >> gpurun_out/d_deferred.log
timeout 1500 python -m pytest tests -m gpu -q -k "psgd or powersgd or dense or fp16 or nccl or distributed or thc" > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
for s in psgd fp16 thc; do
  timeout 300 python tools/time_rank.py --scheme $s --steps 10 >> gpurun_out/d_rank.jsonl 2>> gpurun_out/d_rank.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/d_rank_${s}_launches.csv python tools/time_rank.py --scheme $s --steps 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mq_tma_kernel -s 2 -c 1 \
   -o gpurun_out/d_mq_tma -f python tools/time_rank.py --scheme psgd --steps 1 > gpurun_out/d_ncu_mq.log 2>&1
