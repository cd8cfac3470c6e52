# bench A/B of ray-kernel build variants in build/rx (value only, no CPU arm)
for e in base "$@"; do
  if [ $e = base ]; then L=""; else L="PACT_LIB=build/rx/lib_$e.so"; fi
  env $L python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$e', round(d['value'],1), round(d['e2e']['value'],1))"
  echo "$e $(env $L python scripts/profile_iter.py --steps 2 2>&1 | grep stages | tail -1)"
done
