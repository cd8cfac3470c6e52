#!/bin/bash
# round-2 pass j: fp32 fixed-point scaling alone; loss table loads ahead of the spectra
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "nf_small or cfg2 or bench_configs" > gpurun_out/r02j_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02j_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02j_iter.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02j_iter_cfg5.log 2>&1
