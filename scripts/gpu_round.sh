set -x
python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench_rc=$?
cat gpurun_out/bench5.json; tail -5 gpurun_out/bench5.err
