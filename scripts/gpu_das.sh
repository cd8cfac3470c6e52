python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench_rc=$?
cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:das_stack -s 3 -c 1 -o gpurun_out/das_full4 python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu4.log 2>&1; echo ncu=$?
