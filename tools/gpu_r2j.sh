# round-2 call j: THC fused-kernel A/B (HEAD vs loop counters + bit transpose vs + immediate LCG multiplier)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_thc_gpu.py tests/test_fullsize_gpu.py tests/test_baseline_scale_gpu.py -q -k "thc or rotated or quant" > gpurun_out/j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/j_tests.log
GRADCOMP_B200_LIB=$PWD/build/libgc_imm.so timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke_imm.log 2>&1; echo "rc=$?" >> gpurun_out/j_smoke_imm.log
for rep in 1 2; do
  bash tools/ab_thc.sh old build/libgc_old.so new paper_2407_01378_b200/libgradcomp_b200.so imm build/libgc_imm.so >> gpurun_out/j_ab.txt 2>&1
done
for v in old imm; do
  lib=build/libgc_$v.so
  GRADCOMP_B200_LIB=$PWD/$lib timeout 300 python tools/time_rank.py --scheme thc --steps 10 >> gpurun_out/j_rank_$v.jsonl 2>&1
done
timeout 300 python tools/time_rank.py --scheme thc --steps 10 >> gpurun_out/j_rank_new.jsonl 2>&1
