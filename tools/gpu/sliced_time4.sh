timeout 600 python tools/time_pass.py 120 1,4,8 > gpurun_out/time_sliced.jsonl 2>&1; echo "time rc=$?"
