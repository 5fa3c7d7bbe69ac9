#!/bin/bash
# Copy the round-end evidence from gpurun_out/ (tools/dbg/final.sh on the B200) into profiles/.
# usage: bash tools/collect_profiles.sh [round-tag] [run-tag]
r=${1:-r01}; t=${2:-r01f}; o=gpurun_out; p=profiles
mkdir -p $p
python -c "import json,sys; print(json.dumps(json.loads(open('$o/final_bench.json').read().strip().splitlines()[-1]), indent=1))" > $p/${r}_bench.json
python -c "import json,sys; print(json.dumps(json.loads(open('$o/final_bench_ref.json').read().strip().splitlines()[-1]), indent=1))" > $p/${r}_bench_reference.json
cp $o/final_sweep.log $p/${r}_sweep.jsonl
cp $o/final_bench_launches.csv $p/${r}_bench_launches.csv
{ echo "ncu --metrics gpu__time_duration.sum --clock-control none  python bench.py --steps 3 --warmup 3 (cold-cache, serialised launches)";
  python tools/launch_summary.py $o/final_bench_launches.csv; } > $p/${r}_bench_launch_summary.txt
for s in thc topk topkc psgd dense16; do
  [ -f $o/${t}_${s}_full.txt ] && cp $o/${t}_${s}_full.txt $p/${r}_${s}_ncu_full.txt
  [ -f $o/${t}_${s}_launches.csv ] && { echo "ncu launch list: tools/profile_all.sh $s"; python tools/launch_summary.py $o/${t}_${s}_launches.csv; } > $p/${r}_${s}_launch_summary.txt
done
[ -f $o/${t}_thc_lines.txt ] && cp $o/${t}_thc_lines.txt $p/${r}_thc_fused_lines.txt
tail -3 $o/final_pytest.log > $p/${r}_pytest_gpu_tail.txt
ls -la $p
