#!/bin/bash
# Round-end evidence on one GPU box: the GPU test log, every bench line
# (tools/bench_all.sh), the ncu launch list of the bench command and one
# --set full capture per bench kernel (c2 U53/U32, c4, c1, c3, c5 p = 0.1 / 1e-3).
# Output: gpurun_out/ (copy what is to be judged into profiles/).
set -u
o=gpurun_out
python -m pytest tests -m gpu -x -q > $o/art_gputest.log 2>&1; echo "pytest rc=$?" >> $o/art_gputest.log
tail -2 $o/art_gputest.log
bash tools/bench_all.sh
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/art_launches_raw.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $o/art_ncu_bench.log 2>&1
bash tools/ncu_capture.sh art_c2_u53 c2 2000 u53
bash tools/ncu_capture.sh art_c2_u32 c2 2000 u32
bash tools/ncu_capture.sh art_c4_u53 c4 300 u53
bash tools/ncu_capture.sh art_c1_u53 c1 2000 u53 0 - 131072
bash tools/ncu_capture.sh art_c3_u53 c3 2000 u53 0 - 65536
bash tools/ncu_capture.sh art_c5_p1e-1_u53 c5 2000 u53 0 0.1 32768
bash tools/ncu_capture.sh art_c5_p1e-3_u53 c5 1000 u53 0 0.001 32768
