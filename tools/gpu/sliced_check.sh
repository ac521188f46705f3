# tile-sliced pass kernel: timing vs the warp-per-tile kernel + GPU tests
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python tools/time_pass.py 240 1,2,4,6,8 > gpurun_out/time_sliced.jsonl 2>&1; echo "sliced rc=$?"
NBB_PASS_IMPL=warp timeout 600 python tools/time_pass.py 240 1,2,4 > gpurun_out/time_warp.jsonl 2>&1; echo "warp rc=$?"
timeout 1800 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_shard.py -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gputests.log
