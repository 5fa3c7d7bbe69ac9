# round-2 GPU check: new parity / NCCL / DDP tests, bench (both modes), then the full GPU suite
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt 2>&1
nproc > gpurun_out/c1_nproc.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "baseline_scale or nccl or ddp or distributed_nmse or fp16_bar_saturates or multitensor" > gpurun_out/c1_new.log 2>&1; echo "rc=$?" >> gpurun_out/c1_new.log
timeout 900 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 600 python bench.py --workers 1 --distributed --no-north-star --no-cpu-baseline > gpurun_out/c1_bench_w1.json 2> gpurun_out/c1_bench_w1.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c1_all.log 2>&1; echo "rc=$?" >> gpurun_out/c1_all.log
