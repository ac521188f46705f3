#!/bin/bash
# cluster walk incl. the multi-GPU (P2P / workers / NCCL) paths: timing variants, then the GPU tests of those paths
bash tools/gpu/cl_time.sh > gpurun_out/cl_time.log 2>&1
python -m pytest tests/test_gpu_shard.py tests/test_gpu_multi.py tests/test_gpu_comm.py tests/test_gpu_fullsize.py -x -q > gpurun_out/p2p_tests.log 2>&1
echo tests_exit=$? >> gpurun_out/p2p_tests.log
tail -3 gpurun_out/p2p_tests.log
