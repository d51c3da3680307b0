#!/bin/bash
# A/B of the main build against variants over the config set that exercises
# every kernel path: tools/ab_all.sh variant...
for v in main "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="paper_1605_00854_b200/variants/libpbn_b200_$v.so"; fi
  for spec in "c2 20000 0" "c5 10000 0.0001" "c5 10000 0.001" "c1 100000 0" "c4 2000 0"; do
    set -- $spec
    extra=""; [ "$3" != 0 ] && extra="--p $3"
    PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config $1 --sim-steps $2 --steps 3 $extra > gpurun_out/aba_$v.json 2>/dev/null
    echo "$v $1 p=$3 $(python tools/bench_summary.py gpurun_out/aba_$v.json | cut -c 28-60)"
  done
  PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config c3 --steps 3 > gpurun_out/aba_$v.json 2>/dev/null
  echo "$v c3 $(python tools/bench_summary.py gpurun_out/aba_$v.json | cut -c 28-60)"
done
