#!/bin/bash
# Debug build with GDT_IPF_TRACE (phase clocks of the IPF kernels) into
# paper_2506_00976_b200/csrc/_trace/; select it with GRIDOT_B200_LIB.
set -e
cd "$(dirname "$0")/../paper_2506_00976_b200/csrc"
mkdir -p _trace
NV="/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -DGDT_IPF_TRACE"
objs=""
for f in grid_kernels cbar primal entropic; do $NV --fmad=false -c $f.cu -o _trace/$f.o & objs="$objs _trace/$f.o"; done
for f in cbar_fast cbar_diag ctransform ctransform_pruned probes; do $NV -c $f.cu -o _trace/$f.o & objs="$objs _trace/$f.o"; done
g++ -O3 -std=c++17 -fPIC -ffp-contract=off -fno-fast-math -pthread -c simplex.cpp -o _trace/simplex.o
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o _trace/libgridot_b200.so $objs _trace/simplex.o -lpthread
echo built _trace/libgridot_b200.so
