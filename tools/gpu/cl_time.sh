#!/bin/bash
# time the default library and every tune/lib_*.so with tools/time_cluster.py
python tools/time_cluster.py default
for f in tune/lib_*.so; do [ -f "$f" ] && NBB_GPU_LIB=$f python tools/time_cluster.py $(basename $f .so); done
