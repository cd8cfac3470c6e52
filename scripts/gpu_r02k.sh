#!/bin/bash
# round-2 pass k: tiled interior ray adjoint (shared fixed-point windows)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "nf_small or cfg2 or bench_configs or composed or partition or dropin or cli" > gpurun_out/r02k_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02k_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02k_iter.log 2>&1
PACT_RAY_TILES=0 python scripts/profile_iter.py --steps 2 > gpurun_out/r02k_iter_notile.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02k_iter_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ray_backward" -c 2 \
    -o gpurun_out/r02k_k python scripts/profile_iter.py --steps 1 > gpurun_out/r02k_ncu.log 2>&1
python scripts/src_hot.py gpurun_out/r02k_k.ncu-rep ray_backward_tile 25 > gpurun_out/r02k_hot.txt 2>&1
ncu -i gpurun_out/r02k_k.ncu-rep --page raw --csv > gpurun_out/r02k_raw.csv 2>&1; rm -f gpurun_out/r02k_k.ncu-rep
