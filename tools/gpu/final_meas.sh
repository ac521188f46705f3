nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2700 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --gpus 1 --steps 200 --warmup 5 --no-extras --no-cpu > gpurun_out/bench200.log 2> gpurun_out/bench200.err; echo "bench200 rc=$?"
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 20 --warmup 5 --no-extras --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ca_compact_sliced -s 2 -c 1 -o gpurun_out/ncu_r2_sliced_k8 -f python tools/profile_pass.py 8 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
K=120 timeout 900 python tools/p2p_overhead.py > gpurun_out/p2p_overhead_r2.json 2> gpurun_out/p2p_overhead.err; echo "p2p model rc=$?"
timeout 600 python tools/time_pass.py 240 1,2,4,6,8 > gpurun_out/time_sliced.jsonl 2>&1; echo "time rc=$?"
