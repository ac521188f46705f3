export NBB_GPU_LIB=tune_tmp/libnbb_bulkst.so
timeout 600 python tools/time_pass.py 120 1,4,8 > gpurun_out/time_bulkst.jsonl 2>&1; echo "time rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_multi.py -x -q -m gpu -k "trajectory or c5 or multi_matches or rules_pass" > gpurun_out/gputests_bulkst.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_bulkst.log
