mkdir -p gpurun_out
o=gpurun_out/p1
for s in psgd_gpt2 psgd_gpt2_dist psgd fp16 thc; do
  timeout 300 python tools/time_rank.py --scheme $s --steps 10 >> ${o}_rank.jsonl 2>> ${o}_rank.err
done
for s in psgd_gpt2 psgd_gpt2_dist; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file ${o}_rank_${s}_launches.csv python tools/time_rank.py --scheme $s --steps 1 > /dev/null 2>&1
done
cat ${o}_rank.jsonl
