# round-2 call f: warp-specialised TMA MQ (paired refills vs not), reference tests through the B200 seam, full suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_psgd_deferred_gpu.py tests/test_chunked_psgd_gpu.py -q -x > gpurun_out/f_psgd.log 2>&1; echo "rc=$?" >> gpurun_out/f_psgd.log
timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/f_rank_psgd_pair.jsonl 2>&1
GRADCOMP_B200_LIB=$PWD/build/libgc_np.so timeout 300 python tools/time_rank.py --scheme psgd --steps 10 > gpurun_out/f_rank_psgd_nopair.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/f_rank_psgd_launches.csv python tools/time_rank.py --scheme psgd --steps 1 > /dev/null 2>&1
timeout 900 bash tools/run_reference_tests.sh run gpurun_out/f_ref_tests.log
timeout 2700 python -m pytest tests -m gpu -q -rf > gpurun_out/f_all.log 2>&1; echo "rc=$?" >> gpurun_out/f_all.log
