#!/bin/bash
# round-2 pass l: DAS with interleaved (x, dx) window entries (LDS.64 per tap)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "das or bench_configs or cfg2 or nf_small or partition" > gpurun_out/r02l_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02l_pytest.log
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
ncu --set full --clock-control none -k regex:das_stack -c 1 -o gpurun_out/r02l_das python scripts/profile_iter.py --steps 1 > gpurun_out/r02l_ncu.log 2>&1
ncu -i gpurun_out/r02l_das.ncu-rep --page raw --csv > gpurun_out/r02l_das_raw.csv 2>&1; rm -f gpurun_out/r02l_das.ncu-rep
