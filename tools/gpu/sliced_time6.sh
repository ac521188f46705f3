timeout 600 python tools/time_pass.py 120 1,4,6,8 > gpurun_out/time_tma.jsonl 2>&1; echo "tma rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "trajectory or c5" > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.log
