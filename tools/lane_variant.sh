#!/bin/bash
# Quick A/B build of the lane kernel alone: tools/lane_variant.sh NAME "-DFLAG=.. ..."
# -> paper_1605_00854_b200/variants/libpbn_b200_NAME.so (main build's other objects)
cd "$(dirname "$0")/../paper_1605_00854_b200" || exit 1
name=$1; flags=$2
mkdir -p variants/$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr $flags -c csrc/device/lane_ensemble.cu -o variants/$name/lane_ensemble.o || exit 1
objs=$(ls build/host/*.o build/capi.o build/group.o build/device/ensemble.o build/device/ensemble_script.o build/device/pool.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o variants/libpbn_b200_$name.so $objs variants/$name/lane_ensemble.o -lpthread -ldl
