#!/bin/bash
# A/B of build variants on the lane-kernel workloads: tools/lane_ab.sh variant...
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib="paper_1605_00854_b200/variants/libpbn_b200_$v.so"; fi
  PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config c1 --sim-steps 100000 --steps 3 > gpurun_out/abl_$v.json 2>/dev/null
  echo "$v c1 $(python tools/bench_summary.py gpurun_out/abl_$v.json | cut -c 28-60)"
  PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config c3 --steps 3 > gpurun_out/abl_$v.json 2>/dev/null
  echo "$v c3 $(python tools/bench_summary.py gpurun_out/abl_$v.json | cut -c 28-60)"
done
