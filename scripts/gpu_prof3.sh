python scripts/profile_iter.py --steps 1 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ray_backward|wavefront_kernel|loss_bins|siren_fwd_kernel|siren_dgrad|siren_wgrad_kernel" -s 0 -c 8 -o gpurun_out/iter_full3 python scripts/profile_iter.py --steps 1 > gpurun_out/ncu_f3.log 2>&1; echo full=$?
