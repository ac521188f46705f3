set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
free -g; nproc; lscpu | grep -i "model name"
python tests/golden/make_golden_c3.py gpurun_out/c3_r16.json > gpurun_out/golden_c3.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/fullsize.log 2>&1
tail -5 gpurun_out/fullsize.log
