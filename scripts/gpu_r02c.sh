#!/bin/bash
# round-2 pass c: tests after the smem opt-in fix; register-resident loss kernel A (timing, ncu)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=10 > gpurun_out/r02c_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02c_iter.log 2>&1
PACT_LOSS_STAGED=1 python scripts/profile_iter.py --steps 2 > gpurun_out/r02c_iter_staged.log 2>&1
timeout 600 python scripts/profile_iter.py --steps 1 --cfg cfg5 > gpurun_out/r02c_iter_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"loss_reg|loss_nyquist" -s 0 -c 2 \
    -o gpurun_out/r02c_loss python scripts/profile_iter.py --steps 1 > gpurun_out/r02c_loss_ncu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
echo "bench rc=$?" >> gpurun_out/r02c_bench.err
