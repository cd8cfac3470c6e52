for e in 0 1 2 4; do
  if [ $e = 0 ]; then L=""; else L="PACT_LIB=build/exp/libpact_exp$e.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"tc_|siren|reduce" \
    --log-file gpurun_out/exp$e.csv python scripts/profile_iter.py --steps 1 > /dev/null 2>&1; echo exp$e=$?
done
