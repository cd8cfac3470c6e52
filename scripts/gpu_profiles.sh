#!/bin/bash
# Round profiles (profiles/<tag>_*, PROFILE_TAG): GPU tests, the bench line, the bench launch
# list, full captures of the cfg3 hot kernels, the DAS, and cfg5.  Every ncu
# command runs after the same command exited 0 without ncu.  The .ncu-rep
# files are exported to CSV on the box (raw metrics + source hot spots) and
# removed, so what comes back stays under gpurun's 64 MiB.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export_rep() {  # $1 = report basename
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  gzip -f gpurun_out/$1_raw.csv gpurun_out/$1_details.csv
  rm -f gpurun_out/$1.ncu-rep
}
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest.log
timeout 900 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err; echo "bench rc=$?" >> gpurun_out/p_bench.err
python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg5 > gpurun_out/p_bench_plain.json 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/p_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-cfg5 > gpurun_out/p_launches.log 2>&1; echo launches=$?
python scripts/profile_iter.py --steps 1 > gpurun_out/p_iter.log 2>&1; echo iter=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"ray_backward_plan|cell_gather|side_gather|wavefront_plan|siren_chain|tc_bwd|loss_reg|loss_finish|patch_fft64|fix_to_grad|ray_bound|reduce_segments" -s 0 -c 15 \
    -o gpurun_out/p_iter_full python scripts/profile_iter.py --steps 1 > gpurun_out/p_iter_full.log 2>&1; echo full=$?
for k in ray_backward_plan cell_gather side_gather wavefront_plan loss_reg siren_chain_pair patch_fft64; do
  python scripts/src_hot.py gpurun_out/p_iter_full.ncu-rep $k 30 > gpurun_out/p_hot_$k.txt 2>&1
done
export_rep p_iter_full
ncu --set full --clock-control none --import-source on -k regex:das_stack -c 1 \
    -o gpurun_out/p_das_full python scripts/profile_iter.py --steps 1 > gpurun_out/p_das_full.log 2>&1; echo das=$?
export_rep p_das_full
timeout 900 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/p_iter_cfg5.log 2>&1; echo cfg5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/p_cfg5_launches.csv \
    python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/p_cfg5_launches.log 2>&1; echo cfg5_launches=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"das_stack|tc_wide|siren_top|siren_first|wavefront_plan|cell_gather|side_gather|loss_reg|patch_fft" -c 12 \
    -o gpurun_out/p_cfg5_full python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/p_cfg5_full.log 2>&1; echo cfg5_full=$?
export_rep p_cfg5_full
python scripts/traffic_json.py gpurun_out/p_traffic.json gpurun_out/p_iter_full_raw.csv.gz \
    gpurun_out/p_das_full_raw.csv.gz gpurun_out/p_cfg5_full_raw.csv.gz "$PROFILE_TAG" > gpurun_out/p_traffic.log 2>&1
gzip -f gpurun_out/p_launches.csv gpurun_out/p_cfg5_launches.csv
du -sh gpurun_out
