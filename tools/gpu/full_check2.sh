nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python tools/time_pass.py 120 1,2,4,6,8 > gpurun_out/time_sliced.jsonl 2>&1; echo "time rc=$?"
timeout 2700 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --gpus 1 --steps 200 --warmup 5 --no-extras --no-cpu > gpurun_out/bench200.log 2> gpurun_out/bench200.err; echo "bench200 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-extras > gpurun_out/bench_2ranks.log 2> gpurun_out/bench_2ranks.err; echo "bench2 rc=$?"
K=120 timeout 900 python tools/p2p_overhead.py > gpurun_out/p2p_overhead_r2.json 2> gpurun_out/p2p_overhead.err; echo "p2p model rc=$?"
