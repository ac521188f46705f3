#!/bin/bash
# end-of-round check: GPU suite, smoke, bench (default K = 200, and K = 20), reference arm
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests_exit=$? >> gpurun_out/gputests.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 20 > gpurun_out/bench_k20.json 2> gpurun_out/bench_k20.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gputests.log; cat gpurun_out/smoke.log
