#!/bin/bash
# round-2 pass h: persistent register loss kernel A with prefetch; finish with 8 partials
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "nf_small or cfg2 or bench_configs or composed or partition" > gpurun_out/r02h_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02h_iter.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02h_iter_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"loss_" -c 3 \
    -o gpurun_out/r02h_k python scripts/profile_iter.py --steps 1 > gpurun_out/r02h_ncu.log 2>&1
