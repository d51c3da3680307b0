#!/bin/bash
# The reference's acceptance profiles (acceptance.cpp:199-216) on the device:
# grouped / Method_reduction / Method_old steppers, each with the reference's CPU
# stepper of the same method beside it -> gpurun_out/acceptance.jsonl
: > gpurun_out/acceptance.jsonl
for c in acc_sparse acc_dense; do for m in grouped reduction old; do
  python bench.py --config $c --method $m --steps 3 >> gpurun_out/acceptance.jsonl 2>> gpurun_out/acceptance.err
done; done
python - <<'PY'
import json
for l in open('gpurun_out/acceptance.jsonl'):
    d = json.loads(l)
    print(d['config']['workload'][:10], d['config']['method'], d['config']['n_kept'], '%.3e' % d['trajectory_steps_per_s'],
          '%.3e' % d['cpu_baseline']['trajectory_steps_per_s'], d['config']['engine']['kernel'])
PY
