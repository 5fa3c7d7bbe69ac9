# Round-end evidence on the B200 with the summaries made on the box: the raw ncu reports are too
# large to travel back (gpurun merges <= 64 MiB of gpurun_out/), so collect_profiles.sh runs there
# and only profiles/ text + traffic.json come back in gpurun_out/prof/.
# usage (under gpurun): GC_EVIDENCE_QUICK=1 bash tools/round_evidence_remote.sh
bash tools/round_evidence.sh
bash tools/collect_profiles.sh > gpurun_out/collect.log 2>&1
mkdir -p gpurun_out/prof
cp profiles/r02_* profiles/traffic.json gpurun_out/prof/
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
