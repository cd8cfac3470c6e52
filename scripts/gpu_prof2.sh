python scripts/profile_iter.py --steps 1 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ray_backward|wavefront_kernel|loss_grad|siren_fwd_kernel" -s 0 -c 4 -o gpurun_out/iter_full2 python scripts/profile_iter.py --steps 1 > gpurun_out/ncu_f2.log 2>&1; echo full=$?
