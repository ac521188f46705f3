timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "run_dev_embedded" > gpurun_out/gputests_emb.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests_emb.log
