# round-2 call g: TMA mtp, ctypes core through the reference's tests, synthetic stream, fresh-round TopK sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_psgd_deferred_gpu.py tests/test_synthetic_gpu.py tests/test_chunked_psgd_gpu.py tests/test_multitensor_gpu.py -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 900 bash tools/run_reference_tests.sh run-core gpurun_out/g_ref_core.log
timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/g_rank_psgd.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/g_rank_psgd_launches.csv python tools/time_rank.py --scheme psgd --steps 1 > /dev/null 2>&1
timeout 1200 python tools/sweep.py --synthetic --warmup 3 --steps 8 --only topk,topkc > gpurun_out/g_sweep_synth.jsonl 2> gpurun_out/g_sweep_synth.err
timeout 600 python tools/sweep.py --nmse 5 --dims 4194304 > gpurun_out/g_nmse.txt 2> gpurun_out/g_nmse.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"mq_tma_kernel|mtp_tma_kernel" -s 4 -c 2 \
   -o gpurun_out/g_psgd_tma -f python tools/time_rank.py --scheme psgd --steps 1 > gpurun_out/g_ncu.log 2>&1
