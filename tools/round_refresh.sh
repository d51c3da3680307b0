#!/bin/bash
# Re-measure after a kernel change: GPU tests, the bench lines the change touches
# (c2 headline + U32, c4, c5 sweep) and the c2 / c4 ncu summaries.
set -u
o=gpurun_out
python -m pytest tests -m gpu -x -q > $o/art_gputest.log 2>&1; echo "pytest rc=$?" >> $o/art_gputest.log
tail -2 $o/art_gputest.log
python bench.py > $o/all_default.json 2> $o/all_default.err
python bench.py --no-cpu-baseline --stream u32 > $o/all_c2_u32.json 2>> $o/all_default.err
python bench.py --config c4 --steps 2 --cpu-seconds 8 > $o/all_c4.json 2>> $o/all_default.err
: > $o/all_c5_sweep.jsonl
for p in 0.1 0.01 0.001 0.0001; do
  python bench.py --config c5 --p $p --sim-steps 100000 --steps 2 --cpu-seconds 6 >> $o/all_c5_sweep.jsonl 2>> $o/all_default.err
done
python tools/bench_summary.py $o/all_default.json $o/all_c2_u32.json $o/all_c4.json $o/all_c5_sweep.jsonl | cut -c 1-100
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/art_launches_raw.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $o/art_ncu_bench.log 2>&1
bash tools/ncu_capture.sh art_c2_u53 c2 2000 u53
bash tools/ncu_capture.sh art_c4_u53 c4 300 u53
