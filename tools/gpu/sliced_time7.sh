for v in ldg ldg_m4 tma_m4; do
  NBB_GPU_LIB=tune_tmp/libnbb_$v.so timeout 600 python tools/time_pass.py 120 1,8 > gpurun_out/time_$v.jsonl 2>&1; echo "$v rc=$?"
done
