#!/bin/bash
timeout 900 python tools/cluster_check.py 24 > gpurun_out/cluster_check.log 2>&1; echo rc=$? >> gpurun_out/cluster_check.log
NBB_CL_CHAIN=0 python tools/time_cluster.py nochain > gpurun_out/cl_time.log 2>&1
python tools/time_cluster.py chain >> gpurun_out/cl_time.log 2>&1
R=17 python tools/time_cluster.py chain_r17 >> gpurun_out/cl_time.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_fullsize.py -q -x > gpurun_out/chain_tests.log 2>&1; echo tests_exit=$? >> gpurun_out/chain_tests.log
tail -2 gpurun_out/chain_tests.log; tail -2 gpurun_out/cluster_check.log
