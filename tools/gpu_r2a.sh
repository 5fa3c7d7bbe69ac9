# round-2 re-entry check: full GPU suite, smoke, bench (default + per-rank mode)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
nproc > gpurun_out/a_nproc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/a_smoke.log
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout 2700 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/a_all.log 2>&1; echo "rc=$?" >> gpurun_out/a_all.log
timeout 400 python tools/time_rank.py > gpurun_out/a_rank_350m.jsonl 2> gpurun_out/a_rank.err
