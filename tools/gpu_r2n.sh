# round-2 call n: multi-rank bench path (2 gloo ranks sharing the GPU), then the round-end evidence
mkdir -p gpurun_out
GC_BENCH_ONE_DEVICE=1 GC_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/n_bench_2ranks.json 2> gpurun_out/n_bench_2ranks.err
bash tools/round_evidence.sh
