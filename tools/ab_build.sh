#!/bin/bash
# Experiment build of libitq3 with an alternative chain.cu and/or extra nvcc flags:
#   tools/ab_build.sh NAME CHAIN_CU [NVCC FLAGS...]  ->  exp_libs/libitq3_NAME.so
# (select it at run time with ITQ3_LIB=exp_libs/libitq3_NAME.so; tools/chain_decomp.py times it)
set -e
name=$1; src=$2; shift 2
mkdir -p exp_libs/obj_$name
cp "$src" paper_2603_27914_b200/csrc/.chain_exp_$name.cu
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
     --expt-relaxed-constexpr "$@" -c paper_2603_27914_b200/csrc/.chain_exp_$name.cu -o exp_libs/obj_$name/chain.o \
     2> exp_libs/obj_$name/ptxas.log || { cat exp_libs/obj_$name/ptxas.log; rm -f paper_2603_27914_b200/csrc/.chain_exp_$name.cu; exit 1; }
rm -f paper_2603_27914_b200/csrc/.chain_exp_$name.cu
objs=$(ls build/*.o | grep -v '/chain.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp_libs/libitq3_$name.so exp_libs/obj_$name/chain.o $objs -lcudart
grep -A3 "chain_kernel" exp_libs/obj_$name/ptxas.log | grep -E "registers|spill" | sed -n 3,4p
