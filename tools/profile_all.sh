#!/bin/bash
# Per-scheme ncu evidence (run under gpurun on ONE GPU): a launch list (device time per
# launch, cold-cache, serialised) and one `--set full` capture of every kernel of one round,
# summarised on the box (tools/ncu_summary.py) so only text comes back.
# usage: bash tools/profile_all.sh [tag] [schemes...]
#   -> gpurun_out/<tag>_<scheme>_launches.csv, gpurun_out/<tag>_<scheme>_full.txt
tag=${1:-r01}; shift
schemes=${@:-thc topk topkc psgd dense16}
out=gpurun_out
mkdir -p $out /tmp/prof
run() {  # name, cmd...
  local name=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $out/${tag}_${name}_launches.csv "$@" > /dev/null 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -c ${NCU_COUNT:-40} \
      -o /tmp/prof/${tag}_${name}_full -f "$@" > /tmp/prof/${tag}_${name}_full.log 2>&1
  python tools/ncu_summary.py /tmp/prof/${tag}_${name}_full.ncu-rep > $out/${tag}_${name}_full.txt 2>&1
}
lines() {  # name, kernel regex, source file, cmd...  -> per-source-line shares of one launch
  local name=$1 kre=$2 src=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 \
      -o /tmp/prof/${tag}_${name}_one -f "$@" > /dev/null 2>&1
  FN=${FN:-} python tools/ncu_lines.py /tmp/prof/${tag}_${name}_one.ncu-rep paper_2407_01378_b200/libgradcomp_b200.so \
      $src $kre > $out/${tag}_${name}_lines.txt 2>&1
}
for s in $schemes; do
  case $s in
    thc)     run thc     python tools/prof_thc.py ${THC_D:-25557032} 8 1 1
             FN=${FN:-ILi10ELb1E} lines thc thc_fused paper_2407_01378_b200/csrc/gc_thc_fused.cu python tools/prof_thc.py 25557032 8 1 1 ;;
    topk)    run topk    python tools/prof_scheme.py topk 110000000 8 1 ;;
    topkc)   run topkc   python tools/prof_scheme.py topkc 110000000 8 1 ;;
    psgd)    run psgd    python tools/prof_scheme.py psgd 350000000 8 1 ;;
    dense16) run dense16 python tools/prof_scheme.py dense16 25557032 8 1 ;;
  esac
done
echo profile_all done
