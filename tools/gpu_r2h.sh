# round-2 call h: distributed wire parity (2/3/4 ranks), collective check, synthetic, bench both arms
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_distributed_gpu.py tests/test_collective_check_gpu.py tests/test_synthetic_gpu.py tests/test_nccl_gpu.py -q -rf > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/h_rank_psgd.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/h_bench_ref.json 2> gpurun_out/h_bench_ref.err
