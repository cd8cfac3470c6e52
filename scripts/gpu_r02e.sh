#!/bin/bash
# round-2 pass e: fixed-point (int64) ray adjoint; loss slot finish; full tests + timings + ncu
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/r02e_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02e_iter.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02e_iter_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ray_backward_plan|loss_|ray_bound|fix_to_grad" -s 0 -c 6 \
    -o gpurun_out/r02e_k python scripts/profile_iter.py --steps 1 > gpurun_out/r02e_ncu.log 2>&1
