mkdir -p /tmp/prof gpurun_out
python tools/dbg/payload_dbg.py > gpurun_out/dbg.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:thc_fused -c 1 -o /tmp/prof/thc_one -f python tools/prof_thc.py 25557032 8 1 1 > /dev/null 2>&1
FN=ILi10ELb1E TOP=60 python tools/ncu_lines.py /tmp/prof/thc_one.ncu-rep paper_2407_01378_b200/libgradcomp_b200.so paper_2407_01378_b200/csrc/gc_thc_fused.cu thc_fused > gpurun_out/thc_lines.txt 2>&1
python tools/ncu_summary.py /tmp/prof/thc_one.ncu-rep > gpurun_out/thc_full.txt 2>&1
cp /tmp/prof/thc_one.ncu-rep gpurun_out/
