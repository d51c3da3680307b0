#!/bin/bash
# LPT sweep of one config: tools/lpt_sweep.sh CONFIG SIM_STEPS [lpt ...]
cfg=$1; ss=$2; shift 2
for l in "$@"; do
  python bench.py --no-cpu-baseline --config $cfg --sim-steps $ss --steps 3 --lpt $l > gpurun_out/lpt_${cfg}_$l.json 2> gpurun_out/lpt_${cfg}_$l.err
  echo "lpt=$l $(python tools/bench_summary.py gpurun_out/lpt_${cfg}_$l.json | cut -c 1-150)"
done
