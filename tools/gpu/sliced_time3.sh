nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python tools/time_pass.py 120 1,2,4,6,8 > gpurun_out/time_sliced.jsonl 2>&1; echo "time rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "trajectory" > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.log
