# session-start baseline: all GPU tests + the driver's bench command
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -i "model name"; nproc
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.log
