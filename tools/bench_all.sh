#!/bin/bash
# Round bench lines (run on the GPU box): headline c2 (with CPU baseline and
# the reference arm), then the other BASELINE configs as bench lines with
# bounded simulation lengths. Output: gpurun_out/all_*.json(l)
set -u
o=gpurun_out
python bench.py > $o/all_default.json 2> $o/all_default.err
python bench.py --impl reference > $o/all_ref.json 2> $o/all_ref.err
python bench.py --no-cpu-baseline --stream u32 > $o/all_c2_u32.json 2>> $o/all_default.err
python bench.py --no-cpu-baseline --config c1 --steps 3 > $o/all_c1.json 2>> $o/all_default.err
python bench.py --no-cpu-baseline --config c4 --sim-steps 2000 > $o/all_c4.json 2>> $o/all_default.err
: > $o/all_c5_sweep.jsonl
for p in 0.1 0.01 0.001 0.0001; do
  python bench.py --no-cpu-baseline --config c5 --p $p --sim-steps 10000 --steps 2 >> $o/all_c5_sweep.jsonl 2>> $o/all_default.err
done
python bench.py --config c3 > $o/all_c3.json 2>> $o/all_default.err
python tools/bench_summary.py $o/all_default.json $o/all_ref.json $o/all_c2_u32.json $o/all_c1.json $o/all_c4.json $o/all_c5_sweep.jsonl $o/all_c3.json | cut -c 1-150
