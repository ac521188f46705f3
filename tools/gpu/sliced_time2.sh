nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for v in default sl5 sl3; do
  if [ $v = default ]; then L=""; else L="tune_tmp/libnbb_$v.so"; fi
  NBB_GPU_LIB=$L timeout 600 python tools/time_pass.py 120 1,4,8 > gpurun_out/time_$v.jsonl 2>&1; echo "$v rc=$?"
done
