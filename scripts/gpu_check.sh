#!/bin/bash
# Round-end style check on one B200: the GPU suite, cfg3/cfg5 stage times, the bench line.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/check_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check_pytest.log
python scripts/profile_iter.py --steps 1 > gpurun_out/check_iter.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/check_iter_cfg5.log 2>&1
timeout 900 python bench.py > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err
