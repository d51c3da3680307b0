#!/bin/bash
# A/B timing of compile-time variants on the GPU box: tools/ab.sh CONFIG STREAM [variant ...]
# (variant "main" = the default build). One bench line per variant into gpurun_out/ab_*.json.
cfg=$1; stream=$2; shift 2
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="paper_1605_00854_b200/variants/libpbn_b200_$v.so"; fi
  PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config $cfg --stream $stream --sim-steps ${SIM_STEPS:-20000} \
    > gpurun_out/ab_${cfg}_${stream}_$v.json 2> gpurun_out/ab_${cfg}_${stream}_$v.err
  echo "$v $(python tools/bench_summary.py gpurun_out/ab_${cfg}_${stream}_$v.json | cut -c 1-90)"
done
