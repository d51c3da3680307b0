#!/bin/bash
# A/B of build variants over the sub-warp workloads (and c1/c3 with LANE=1):
# tools/ab_pf.sh variant...   (main = the default build)
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="paper_1605_00854_b200/variants/libpbn_b200_$v.so"; fi
  for spec in "c2 20000 0 u53" "c2 20000 0 u32" "c5 10000 0.1 u53" "c5 10000 0.001 u53" "c5 10000 0.0001 u53" "c4 2000 0 u53" ${LANE:+"c1 100000 0 u53"}; do
    set -- $spec
    extra=""; [ "$3" != 0 ] && extra="--p $3"
    PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config $1 --stream $4 --sim-steps $2 --steps 3 $extra > gpurun_out/abp_$v.json 2>/dev/null
    echo "$v $1 p=$3 $4 $(python tools/bench_summary.py gpurun_out/abp_$v.json | cut -c 28-60)"
  done
  if [ -n "$LANE" ]; then
    PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config c3 --steps 3 > gpurun_out/abp_$v.json 2>/dev/null
    echo "$v c3 $(python tools/bench_summary.py gpurun_out/abp_$v.json | cut -c 28-60)"
  fi
done
