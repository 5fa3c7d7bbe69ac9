# round-2 call c: TMA / deferred-EF PowerSGD and the Cholesky orthonormalization
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py -q -x > gpurun_out/c_deferred.log 2>&1; echo "rc=$?" >> gpurun_out/c_deferred.log
timeout 1500 python -m pytest tests -m gpu -q -k "psgd or powersgd or multitensor or nccl or distributed or ddp or baseline_scale" > gpurun_out/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c_tests.log
for s in psgd psgd_gpt2 thc; do
  timeout 300 python tools/time_rank.py --scheme $s --steps 10 >> gpurun_out/c_rank.jsonl 2>> gpurun_out/c_rank.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/c_rank_${s}_launches.csv python tools/time_rank.py --scheme $s --steps 1 > /dev/null 2>&1
done
timeout 300 python tools/sweep.py --help > /dev/null 2>&1
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
