# round-end evidence on one B200 (run under gpurun): full GPU tests, smoke, bench (both arms), sweep, launch list,
# per-scheme ncu (tools/profile_all.sh); then `bash tools/collect_profiles.sh` here copies the summaries to profiles/
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python tools/sweep.py > gpurun_out/final_sweep.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_bench_launches.csv python bench.py --steps 3 --warmup 3 > /dev/null 2>&1
NCU_COUNT=40 bash tools/profile_all.sh r01f thc topk topkc psgd dense16 > /dev/null 2>&1
echo done > gpurun_out/final_done
