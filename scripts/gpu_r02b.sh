#!/bin/bash
# round-2 pass b: composed path + drop-in ports, bench with the cpu_baseline leg, reference arm (short)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/r02b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
echo "bench rc=$?" >> gpurun_out/r02b_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err
echo "ref rc=$?" >> gpurun_out/r02b_ref.err
nproc > gpurun_out/r02b_nproc.txt; lscpu | head -20 >> gpurun_out/r02b_nproc.txt
