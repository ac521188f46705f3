for K in 1 8; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ca_compact_sliced -s 1 -c 1 -o gpurun_out/ncu_sliced_k$K -f python tools/profile_pass.py $K > gpurun_out/ncu_k$K.log 2>&1; echo "ncu K=$K rc=$?"
done
