#!/bin/bash
# On the GPU box: one ncu --set full capture of the ensemble kernel of a
# profile_launch.py command, summarised into gpurun_out/<name>.txt (the report
# itself stays in /tmp unless KEEP_REP=1): tools/ncu_capture.sh name args...
name=$1; shift
python profile_launch.py "$@" > /dev/null || exit 1
ncu --set full --clock-control none --import-source on -c 1 -k regex:'pbn_(ensemble|lane)' -o /tmp/$name python profile_launch.py "$@" > /tmp/$name.log 2>&1
python tools/ncu_summary.py /tmp/$name.ncu-rep > gpurun_out/$name.txt 2>&1
python tools/ncu_lines.py /tmp/$name.ncu-rep >> gpurun_out/$name.txt 2>/dev/null
[ -n "$KEEP_REP" ] && cp /tmp/$name.ncu-rep gpurun_out/
ls -la /tmp/$name.ncu-rep
