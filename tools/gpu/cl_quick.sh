#!/bin/bash
timeout 900 python tools/cluster_check.py 24 > gpurun_out/cluster_check.log 2>&1; echo rc=$? >> gpurun_out/cluster_check.log
python tools/time_cluster.py default > gpurun_out/cl_time.log 2>&1
tail -2 gpurun_out/cluster_check.log
