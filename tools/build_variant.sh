#!/bin/bash
# Build an experimental variant of libs5gpu.so with extra nvcc flags into
# paper_1403_2056_b200/_lib/var_<NAME>.so (select it with S5G_LIB=...).
# usage: bash tools/build_variant.sh NAME "-DMED_VMAX_CFG=31 ..."
NAME=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -Xcompiler -fopenmp -lgomp -I include $@ -o paper_1403_2056_b200/_lib/var_${NAME}.so \
    paper_1403_2056_b200/csrc/s5g.cu 2>&1 | grep -E "error" -A3
ls -la paper_1403_2056_b200/_lib/var_${NAME}.so
