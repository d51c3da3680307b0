#!/bin/bash
# Round bench lines (run on the GPU box): headline c2 (with CPU baseline and
# the reference arm), then every BASELINE config at its stated shape where a
# bench step stays under ~30 s (c4 at 1e5 steps; the c5 sweep at 1e5 of its
# 1e6 steps per bench step), each with its reference CPU line.
# Output: gpurun_out/all_*.json(l)
set -u
o=gpurun_out
python bench.py > $o/all_default.json 2> $o/all_default.err
python bench.py --impl reference > $o/all_ref.json 2> $o/all_ref.err
python bench.py --no-cpu-baseline --stream u32 > $o/all_c2_u32.json 2>> $o/all_default.err
python bench.py --config c1 --steps 3 > $o/all_c1.json 2>> $o/all_default.err
python bench.py --impl reference --config c1 --steps 3 > $o/all_c1_ref.json 2>> $o/all_default.err
python bench.py --config c4 --steps 2 --cpu-seconds 8 > $o/all_c4.json 2>> $o/all_default.err
python bench.py --impl reference --config c4 --steps 2 > $o/all_c4_ref.json 2>> $o/all_default.err
: > $o/all_c5_sweep.jsonl
for p in 0.1 0.01 0.001 0.0001; do
  python bench.py --config c5 --p $p --sim-steps 100000 --steps 2 --cpu-seconds 6 >> $o/all_c5_sweep.jsonl 2>> $o/all_default.err
done
python bench.py --config c3 > $o/all_c3.json 2>> $o/all_default.err
python bench.py --impl reference --config c3 --steps 2 > $o/all_c3_ref.json 2>> $o/all_default.err
python tools/bench_summary.py $o/all_default.json $o/all_ref.json $o/all_c2_u32.json $o/all_c1.json $o/all_c1_ref.json $o/all_c4.json $o/all_c4_ref.json $o/all_c5_sweep.jsonl $o/all_c3.json $o/all_c3_ref.json | cut -c 1-170
