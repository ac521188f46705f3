#!/bin/bash
timeout 900 python tools/cluster_check.py 24 > gpurun_out/cluster_check.log 2>&1; echo rc=$? >> gpurun_out/cluster_check.log
python tools/time_cluster.py default > gpurun_out/cl_time.log 2>&1
R=17 python tools/time_cluster.py default_r17 >> gpurun_out/cl_time.log 2>&1
python -m pytest tests/test_gpu_fullsize.py tests/test_capi.py tests/test_gpu_shard.py tests/test_gpu_multi.py tests/test_gpu_comm.py -x -q > gpurun_out/k12_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/k12_tests.log
tail -2 gpurun_out/k12_tests.log; tail -2 gpurun_out/cluster_check.log
