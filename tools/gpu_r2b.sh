# round-2 call b: fixed PowerSGD tests, per-rank launch lists, THC fused source-level capture, sanitizers
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "psgd or powersgd or multitensor" > gpurun_out/b_psgd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b_psgd_tests.log
for s in thc psgd psgd_gpt2 fp16; do
  timeout 300 python tools/time_rank.py --scheme $s --steps 10 >> gpurun_out/b_rank.jsonl 2>> gpurun_out/b_rank.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/b_rank_${s}_launches.csv python tools/time_rank.py --scheme $s --steps 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:thc_fused_kernel -s 1 -c 1 \
   -o gpurun_out/b_thc_fused -f python tools/prof_thc.py 25557032 8 1 2 > gpurun_out/b_ncu_fused.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/b_san_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/b_san_${tool}.log
done
