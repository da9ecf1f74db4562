#!/bin/bash
# One-file variant build for A/B timing of the 3-D p=4 kernels:
#   tools/var_d3p4.sh NAME "-DFLAG=1 ..."  ->  var/NAME.so (other objects from build/obj)
set -e
name=$1; flags=$2
mkdir -p var build/var
nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -diag-suppress 177 $flags -c paper_1204_1533_b200/csrc/cuda/inst_${3:-d3_p4}.cu -o build/var/d3p4_$name.o
objs=$(ls build/obj/cuda/*.o | grep -v inst_${3:-d3_p4})
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o var/$name.so $objs build/var/d3p4_$name.o -lcudart
