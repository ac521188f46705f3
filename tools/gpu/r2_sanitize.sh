for tool in memcheck racecheck synccheck; do
  SAN_R=9 timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done
timeout 900 python tools/parity_sweep.py 600 > gpurun_out/parity_sweep_r2.json 2> gpurun_out/parity_sweep_r2.err; echo "sweep rc=$?"; tail -c 600 gpurun_out/parity_sweep_r2.json
