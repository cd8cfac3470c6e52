ncu --set full --clock-control none --import-source on -k regex:"tc_layer_kernel" -s 1 -c 1 -o gpurun_out/tc_fwd python scripts/profile_iter.py --steps 1 > gpurun_out/ncu_tc.log 2>&1; echo full=$?
