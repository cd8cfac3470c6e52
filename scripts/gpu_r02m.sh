#!/bin/bash
# round-2 pass l: DAS with 4x4 half-warp pixel blocks for LDS.64
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "das or bench_configs or cfg2 or nf_small or partition" > gpurun_out/r02m_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02m_pytest.log
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
ncu --set full --clock-control none -k regex:das_stack -c 1 -o gpurun_out/r02m_das python scripts/profile_iter.py --steps 1 > gpurun_out/r02m_ncu.log 2>&1
ncu -i gpurun_out/r02m_das.ncu-rep --page raw --csv > gpurun_out/r02m_das_raw.csv 2>&1; rm -f gpurun_out/r02m_das.ncu-rep
