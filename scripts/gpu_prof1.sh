python scripts/profile_iter.py --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iter_launches.csv python scripts/profile_iter.py --steps 2 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"siren_fwd_kernel|siren_dgrad|siren_wgrad|ray_backward|wavefront_kernel|loss_grad" -s 20 -c 6 -o gpurun_out/iter_full python scripts/profile_iter.py --steps 2 > gpurun_out/ncu_f.log 2>&1; echo full=$?
cat gpurun_out/prof_plain.log | tail -3
