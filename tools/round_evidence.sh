# round-end evidence on one B200 (run under gpurun; outputs in gpurun_out/r02e_*): full GPU tests, smoke,
# bench (both arms), launch list of the bench, ncu full capture of the bench kernel (roofline traffic),
# per-rank launch lists at d = 350M, ncu summaries of the PowerSGD TMA kernels, sweeps (fresh synthetic
# rounds; cfg5 size sweep), reference tests through both seams, sanitizers.
# `bash tools/collect_profiles.sh` (here) turns them into profiles/r02_*.
o=gpurun_out/r02e
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > ${o}_smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf > ${o}_pytest.log 2>&1; echo "rc=$?" >> ${o}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${o}_smoke.log 2>&1; echo "rc=$?" >> ${o}_smoke.log
timeout 900 python bench.py > ${o}_bench.json 2> ${o}_bench.err
timeout 900 python bench.py --impl reference > ${o}_bench_ref.json 2> ${o}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-north-star > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:thc_fused_kernel -s 1 -c 1 \
  -o ${o}_thc_fused -f python tools/prof_thc.py 25557032 8 1 2 > /dev/null 2>&1
for s in thc psgd psgd_gpt2 psgd_gpt2_dist fp16; do
  timeout 300 python tools/time_rank.py --scheme $s --steps 10 >> ${o}_rank.jsonl 2>> ${o}_rank.err
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file ${o}_rank_${s}_launches.csv python tools/time_rank.py --scheme $s --steps 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mq_tma_kernel|mtp_tma_kernel|decode_vec" \
  -s 5 -c 3 -o ${o}_psgd_tma -f python tools/time_rank.py --scheme psgd --steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mtp_umma_kernel" -s 1 -c 1 \
  -o ${o}_mtp_umma -f python tools/time_rank.py --scheme psgd --rank 8 --steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mq_async_kernel|mtp_async_kernel|mtp_tma_kernel" \
  -s 3 -c 3 -o ${o}_psgd_async -f python tools/time_rank.py --scheme psgd_gpt2 --steps 1 > /dev/null 2>&1
timeout 120 ./build/ubench/umma_rate > ${o}_umma_rate.jsonl 2>&1
timeout 120 ./build/ubench/unaligned_stream > ${o}_unaligned_stream.jsonl 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"rank_quant|rank_ranges|rank_decode" -s 3 -c 3 \
  -o ${o}_thc_rank -f python tools/time_rank.py --scheme thc --steps 1 > /dev/null 2>&1
if [ -z "$GC_EVIDENCE_QUICK" ]; then
timeout 1500 python tools/sweep.py --synthetic --warmup 3 --steps 8 > ${o}_sweep_synthetic.jsonl 2> ${o}_sweep.err
timeout 1500 python tools/sweep.py --dims 1048576,4194304,16777216,67108864,268435456,1000000000 --warmup 3 --steps 5 \
  > ${o}_sweep_dims.jsonl 2>> ${o}_sweep.err
timeout 900 python tools/sweep.py --nmse 5 --dims 4194304 > ${o}_nmse_sweep.txt 2>> ${o}_sweep.err
timeout 900 bash tools/run_reference_tests.sh run ${o}_ref_tests_seam.txt
timeout 900 bash tools/run_reference_tests.sh run-core ${o}_ref_tests_core.txt
fi
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > ${o}_san_${tool}.txt 2>&1
  echo "rc=$?" >> ${o}_san_${tool}.txt
done
echo done > ${o}_done
