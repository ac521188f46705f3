# K-step pass kernel: timing (two register budgets) + full-size parity + all GPU tests
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python tools/time_pass.py > gpurun_out/time_pass_minb3.jsonl 2>&1; echo "time3 rc=$?"
NBB_GPU_LIB=tune_tmp/libnbb_minb2.so timeout 600 python tools/time_pass.py > gpurun_out/time_pass_minb2.jsonl 2>&1; echo "time2 rc=$?"
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gputests.log
