#!/bin/bash
# round-2 pass f: register radix-4 FFT (P=64), fixed-point fold, DAS row band, phase split, cfg5 bench line
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/r02f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02f_iter.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"patch_fft|patch_ifft|fix_to_grad|border_fold|ray_bound|loss_finish|loss_nyq" -c 8 \
    -o gpurun_out/r02f_k python scripts/profile_iter.py --steps 1 > gpurun_out/r02f_ncu.log 2>&1
PACT_FFT_SMEM=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"patch_fft" -c 2 --csv \
    python scripts/profile_iter.py --steps 1 > gpurun_out/r02f_fft_old.csv 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
echo "bench rc=$?" >> gpurun_out/r02f_bench.err
