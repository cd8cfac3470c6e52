#!/bin/bash
# round-2 pass n: DAS staging without per-entry division; SIREN gradient reduction 32 x 8
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rA -k "das or bench_configs or cfg2 or nf_small or siren or partition" > gpurun_out/r02n_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02n_pytest.log
python scripts/profile_iter.py --steps 2 > gpurun_out/r02n_iter.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"reduce_segments|das_stack" -c 3 --csv python scripts/profile_iter.py --steps 1 > gpurun_out/r02n_k.csv 2>&1
