python scripts/profile_iter.py --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python scripts/profile_iter.py --steps 1 > gpurun_out/ncu_l.log 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"tc_" -s 0 -c 9 -o gpurun_out/tc_full python scripts/profile_iter.py --steps 1 > gpurun_out/ncu_f.log 2>&1; echo full=$?
tail -3 gpurun_out/prof_plain.log
