#!/bin/bash
# Experiment build of libitq3 with one source file (any csrc/*.cu) replaced and/or extra nvcc flags:
#   tools/ab_build_src.sh NAME SRC.cu OBJ [NVCC FLAGS...]  ->  exp_libs/libitq3_NAME.so
# OBJ = the object it replaces (e.g. mmq), SRC.cu compiled from csrc/ (so its includes resolve).
set -e
name=$1; src=$2; obj=$3; shift 3
mkdir -p exp_libs/obj_$name
cp "$src" paper_2603_27914_b200/csrc/.exp_$name.cu
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
     --expt-relaxed-constexpr "$@" -c paper_2603_27914_b200/csrc/.exp_$name.cu -o exp_libs/obj_$name/$obj.o \
     2> exp_libs/obj_$name/ptxas.log || { cat exp_libs/obj_$name/ptxas.log; rm -f paper_2603_27914_b200/csrc/.exp_$name.cu; exit 1; }
rm -f paper_2603_27914_b200/csrc/.exp_$name.cu
objs=$(ls build/*.o | grep -v "/$obj.o\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp_libs/libitq3_$name.so exp_libs/obj_$name/$obj.o $objs -lcudart
