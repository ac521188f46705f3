for v in p2m5 p2m6 p2m7; do
  NBB_GPU_LIB=tune_tmp/libnbb_$v.so timeout 600 python tools/time_pass.py 120 1,4,6,8 > gpurun_out/time_$v.jsonl 2>&1; echo "$v rc=$?"
done
