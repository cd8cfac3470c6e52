#!/bin/bash
# round-2 pass d: Nyquist finish split into a warp-per-angle gather; RED throughput probe
cd $GRAFT_REPO_ROOT
./build/red_rate > gpurun_out/r02d_red.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -k "composed or nf_small or cfg2 or bench_configs or dropin or cli" > gpurun_out/r02d_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02d_iter.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"loss_" -s 0 -c 3 \
    -o gpurun_out/r02d_loss python scripts/profile_iter.py --steps 1 > gpurun_out/r02d_loss_ncu.log 2>&1
