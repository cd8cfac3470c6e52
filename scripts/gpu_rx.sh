# A/B of ray-kernel build variants in build/rx (stage times of one cfg3 frame)
for e in base "$@"; do
  if [ $e = base ]; then L=""; else L="PACT_LIB=build/rx/lib_$e.so"; fi
  echo "$e $(env $L python scripts/profile_iter.py --steps 2 2>&1 | grep stages | tail -1)"
done
