#!/bin/bash
# round-2 final evidence: GPU suite, smoke, bench (K = 200 default, K = 20), one-GPU multi-GPU model,
# ncu of the headline pass, launch list, reference arm
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 20 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
python tools/p2p_overhead.py > gpurun_out/p2p_overhead.json 2> gpurun_out/p2p_overhead.err
ncu --set full --clock-control none --import-source on -k regex:ca_compact_cluster -s 1 -c 1 \
    -o gpurun_out/ncu_cluster_k8_final python tools/profile_pass.py 8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 16 --warmup 3 --no-cpu --no-extras --no-e2e > gpurun_out/ncu_launch.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gputests.log
