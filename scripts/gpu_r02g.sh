#!/bin/bash
# round-2 pass g: border-line adjoint in shared fixed-point slots
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/r02g_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02g_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02g_iter.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02g_iter_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ray_backward|ray_bound|fix_to_grad|border_fold" -c 5 \
    -o gpurun_out/r02g_k python scripts/profile_iter.py --steps 1 > gpurun_out/r02g_ncu.log 2>&1
