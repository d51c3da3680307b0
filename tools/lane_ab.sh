for v in main scan q8 q8t31 q4t31; do
  if [ "$v" = main ]; then lib=""; else lib="paper_1605_00854_b200/variants/libpbn_b200_$v.so"; fi
  PBN_B200_LIB=$lib python bench.py --no-cpu-baseline --config c1 --sim-steps 100000 --steps 3 > gpurun_out/abl_$v.json 2>/dev/null
  echo "$v c1 $(python tools/bench_summary.py gpurun_out/abl_$v.json | cut -c 28-60)"
done
bash tools/ncu_capture.sh s5_c1_queue c1 2000 u53 0 - 131072
