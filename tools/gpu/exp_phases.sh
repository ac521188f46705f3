for v in nohalo nostore nohalo_nostore; do
  NBB_GPU_LIB=tune_tmp/libnbb_$v.so timeout 600 python tools/time_pass.py 60 1,8 > gpurun_out/exp_$v.jsonl 2>&1; echo "$v rc=$?"
done
