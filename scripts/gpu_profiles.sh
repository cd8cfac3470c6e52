# Round profiles: bench launch list + full captures of the hot kernels.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err; echo bench_plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1; echo launches=$?
python scripts/profile_iter.py --steps 1 > gpurun_out/iter_plain.log 2>&1; echo iter_plain=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"ray_backward_plan|wavefront_plan|siren_chain_fwd|tc_bwd|loss_bins|loss_nyquist" -s 0 -c 8 \
    -o gpurun_out/iter_full python scripts/profile_iter.py --steps 1 > gpurun_out/iter_full.log 2>&1; echo full=$?
ncu --set full --clock-control none --import-source on -k regex:das_stack -c 1 \
    -o gpurun_out/das_full python scripts/profile_iter.py --steps 1 > gpurun_out/das_full.log 2>&1; echo das=$?
